#!/bin/bash
# Round profile capture under gpurun: plain runs first, then ncu on the same
# command lines (B200_PROFILING.md).  Outputs to gpurun_out/prof_<tag>_*.
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-interp --no-mu"
$B > $O/${TAG}_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv $B > $O/${TAG}_launches.log 2>&1
$B > $O/${TAG}_bench_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dse_pairs_kernel -s 3 -c 1 -o $O/${TAG}_sweep_pairs $B > $O/${TAG}_ncu_sweep.log 2>&1
BE="python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-interp --no-mu --arith exact"
$BE > $O/${TAG}_bench_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dse_solve_kernel -s 3 -c 1 -o $O/${TAG}_sweep_exact $BE > $O/${TAG}_ncu_sweep_exact.log 2>&1
python scripts/interp_probe.py direct 3 > $O/${TAG}_interp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:interp_batch -s 1 -c 1 -o $O/${TAG}_interp_direct python scripts/interp_probe.py direct 3 > $O/${TAG}_ncu_interp.log 2>&1
python scripts/mu_step_probe.py bcb 3 > $O/${TAG}_mu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mu_solve_kernel -s 3 -c 1 -o $O/${TAG}_mu $(echo python scripts/mu_step_probe.py bcb 3) > $O/${TAG}_ncu_mu.log 2>&1
echo "profile round ${TAG} done"
