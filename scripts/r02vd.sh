set -u
O=gpurun_out
for i in 1 2; do
bash scripts/ab_pairs.sh paper_2012_03667_b200/libdse_b200.so build/ab_t320m2u4.so build/ab_t320m2u2.so build/ab_t320m2u3.so build/ab_t384m2u4.so build/ab_t352m2u4.so build/ab_t288m2u4.so build/ab_t640m1u4.so build/ab_t704m1u4.so build/ab_t768m1u4.so build/ab_t576m1u4.so build/ab_t640m1u8.so >> $O/r02vd_ab.log 2>&1
done
echo done
