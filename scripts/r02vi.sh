set -u
O=gpurun_out
for i in 1 2; do
bash scripts/ab_pairs.sh paper_2012_03667_b200/libdse_b200.so build/ab_nl0.so build/ab_nl1.so build/ab_nl1u6.so build/ab_nl1u8.so >> $O/r02vi_ab.log 2>&1
done
echo done
