set -u
O=gpurun_out
for r in 1 2; do for v in new t2; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py exact | sed "s/^/$v /" >> $O/r02bv.log 2>&1; done; done
echo done
