set -u
O=gpurun_out
DSE_CREATE_TIMING=1 python scripts/create_probe.py > $O/r02af.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_batch.py tests/test_gpu_dropin.py -q -m gpu > $O/r02af_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02af_pytest.log
echo done
