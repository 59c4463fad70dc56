set -u
O=gpurun_out
for i in 1 2; do
bash scripts/ab_pairs.sh build/ab_q0.so build/ab_q1.so build/ab_q3.so build/ab_q4.so build/ab_q8.so >> $O/r02vr_ab.log 2>&1
done
echo done
