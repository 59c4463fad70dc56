set -u
O=gpurun_out
for i in 1 2; do
bash scripts/ab_pairs.sh paper_2012_03667_b200/libdse_b200.so build/ab_p640u5.so build/ab_p640u6.so build/ab_p512u6.so build/ab_p512u12.so build/ab_p512u16.so >> $O/r02vn_ab.log 2>&1
done
echo done
