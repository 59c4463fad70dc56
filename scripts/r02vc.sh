set -u
O=gpurun_out
for i in 1 2; do
bash scripts/ab_pairs.sh paper_2012_03667_b200/libdse_b200.so build/ab_t192m3u8.so build/ab_t192m3u6.so build/ab_t320m2u8.so build/ab_t320m2u6.so build/ab_t320m2u4.so build/ab_t160m4u8.so build/ab_t224m3u6.so build/ab_t128m4u8.so >> $O/r02vc_ab.log 2>&1
done
echo done
