set -u
O=gpurun_out
T=r02vp
timeout 2400 python -m pytest tests -m gpu -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?" >> $O/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_ref.json 2> $O/${T}_ref.err
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-interp --no-mu"
$B > $O/${T}_b_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv $B > $O/${T}_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dse_pairs_kernel -s 3 -c 1 -o $O/${T}_pairs $B > $O/${T}_ncu_pairs.log 2>&1
python scripts/interp_probe.py search 3 > $O/${T}_ip.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/${T}_interp_search python scripts/interp_probe.py search 3 > $O/${T}_ncu_interp.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/${T}_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_ncu_smoke.log 2>&1; echo "ncu rc=$?" >> $O/${T}_ncu_smoke.log
echo done
