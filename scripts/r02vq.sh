set -u
O=gpurun_out
for a in exact fast; do
for t in 256 512; do
echo -n "threads=$t " >> $O/r02vq.log
DSE_THREADS=$t python scripts/exact_time.py $a >> $O/r02vq.log 2>&1
done; done
echo done
