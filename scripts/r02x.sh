set -u
O=gpurun_out
T=r02x
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-interp --no-mu"
$B > $O/${T}_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv $B > $O/${T}_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dse_pairs_kernel -s 3 -c 1 -o $O/${T}_pairs $B > $O/${T}_ncu_pairs.log 2>&1
python scripts/interp_probe.py direct 3 > $O/${T}_interp_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/${T}_interp_direct python scripts/interp_probe.py direct 3 > $O/${T}_ncu_interp1.log 2>&1
python scripts/interp_probe.py cubic_direct 3 > $O/${T}_interp_plain2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/${T}_interp_cubic python scripts/interp_probe.py cubic_direct 3 > $O/${T}_ncu_interp2.log 2>&1
python scripts/interp_sweep.py > $O/${T}_interp_sweep.log 2>&1
echo done
