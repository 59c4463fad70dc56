set -u
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r02an_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02an_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/r02an_bench.json 2> $O/r02an_bench.err; echo "bench rc=$?" >> $O/r02an_bench.err
echo done
