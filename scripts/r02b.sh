set -u
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02b_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/r02b_bench.json 2> $O/r02b_bench.err; echo "bench rc=$?" >> $O/r02b_bench.err
echo done
