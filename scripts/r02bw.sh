set -u
O=gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > $O/r02bw_bench.json 2> $O/r02bw_bench.err; echo "bench rc=$?" >> $O/r02bw_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r02bw_ref.json 2> $O/r02bw_ref.err; echo "ref rc=$?" >> $O/r02bw_ref.err
echo done
