set -u
O=gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-tts --no-interp --no-mu"
$B > $O/r02vj_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dse_pairs_kernel -s 3 -c 1 -o $O/r02vj_pairs $B > $O/r02vj_ncu.log 2>&1
echo done
