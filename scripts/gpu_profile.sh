#!/bin/bash
# Profiling recipe run under gpurun (B200_PROFILING.md): plain run first, then
# ncu on the same command line.  Usage: scripts/gpu_profile.sh <arith> <tag>
set -u
ARITH=${1:-exact}
TAG=${2:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-tts --no-interp --no-cpu --arith $ARITH"
$CMD > $OUT/plain_${ARITH}_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${ARITH}_${TAG}.csv $CMD > $OUT/ncu_launch_${ARITH}_${TAG}.log 2>&1
$CMD > $OUT/plain2_${ARITH}_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dse_solve_kernel -s 3 -c 1 -o $OUT/prof_${ARITH}_${TAG} $CMD > $OUT/ncu_full_${ARITH}_${TAG}.log 2>&1
echo "profile ${ARITH} ${TAG} done rc=$?"
