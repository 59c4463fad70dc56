set -u
O=gpurun_out
for r in 1 2; do for a in pairs exact fast; do for v in prev base; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py $a | sed "s/^/$v /" >> $O/r02bi.log 2>&1; done; done; done
echo done
