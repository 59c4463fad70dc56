set -u
O=gpurun_out
T=r02vy
timeout 2400 python -m pytest tests -m gpu -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?" >> $O/${T}_bench.err
timeout 600 python bench.py --impl reference > $O/${T}_ref.json 2> $O/${T}_ref.err; echo "ref rc=$?" >> $O/${T}_ref.err
python scripts/interp_probe.py search 3 > $O/${T}_ip.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/${T}_interp_search python scripts/interp_probe.py search 3 > $O/${T}_ncu_interp.log 2>&1
echo done
