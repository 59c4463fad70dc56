set -u
O=gpurun_out
for i in 1 2; do
for v in ws_s256u8 ws_s512u8 ws_s1024u8 ws_s2048u8 ws_s512u6 ws_s512u4 ws_s512u12; do
DSE_PAIRS_WS=1 timeout 300 bash scripts/ab_pairs.sh build/ab_$v.so >> $O/r02vu_ab.log 2>&1
done; done
echo done
