set -u
O=gpurun_out
timeout 900 python bench.py > $O/r02wc_bench.json 2> $O/r02wc_bench.err; echo "bench rc=$?" >> $O/r02wc_bench.err
timeout 600 python bench.py --impl reference > $O/r02wc_ref.json 2> $O/r02wc_ref.err; echo "ref rc=$?" >> $O/r02wc_ref.err
echo done
