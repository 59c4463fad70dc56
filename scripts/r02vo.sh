set -u
O=gpurun_out
bash scripts/ab_mu.sh paper_2012_03667_b200/libdse_b200.so build/ab_mu320m2u8.so build/ab_mu320m2u4.so build/ab_mu640m1u4.so build/ab_mu640m1u8.so build/ab_mu512m1u8.so > $O/r02vo_ab.log 2>&1
echo done
