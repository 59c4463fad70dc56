set -u
O=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-interp --no-mu"
for v in nl1 wf640u4; do
DSE_LIB=build/ab_$v.so $B > $O/r02vk_plain_$v.log 2>&1 && DSE_LIB=build/ab_$v.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:dse_pairs_kernel -s 3 -c 1 -o $O/r02vk_$v $B > $O/r02vk_ncu_$v.log 2>&1
done
echo done
