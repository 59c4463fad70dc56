set -u
O=gpurun_out
for i in 1 2; do
python scripts/interp_sweep.py | sed "s/^/s3 /" >> $O/r02bz.log 2>&1
DSE_LIB=build/ab_s2.so python scripts/interp_sweep.py | sed "s/^/s2 /" >> $O/r02bz.log 2>&1
done
echo done
