set -u
O=gpurun_out
for i in 1 2; do
DSE_LIB=build/ab_old.so python scripts/exact_time.py pairs | sed "s/^/old /" >> $O/r02ad.log 2>&1
DSE_PAIRS_SYM=0 python scripts/exact_time.py pairs | sed "s/^/nosym /" >> $O/r02ad.log 2>&1
python scripts/exact_time.py pairs | sed "s/^/sym /" >> $O/r02ad.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_dropin.py tests/test_gpu_distributed.py tests/test_gpu_batch.py -q -m gpu > $O/r02ad_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02ad_pytest.log
echo done
