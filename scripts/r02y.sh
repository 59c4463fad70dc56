set -u
O=gpurun_out
for v in base q4 q4s3 q2s6 base q4; do DSE_LIB=build/ab_$v.so python scripts/interp_sweep.py | sed "s/^/$v /" >> $O/r02y.log 2>&1; done
DSE_LIB=build/ab_q4.so DSE_INTERP_FAST=1 python scripts/interp_sweep.py | sed "s/^/q4fast /" >> $O/r02y.log 2>&1
DSE_LIB=build/ab_q4.so DSE_INTERP_REP=3 python scripts/interp_sweep.py | sed "s/^/q4r3 /" >> $O/r02y.log 2>&1
echo done
