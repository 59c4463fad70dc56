set -u
O=gpurun_out
DSE_MOM_CLUSTER=0 python scripts/mom_tts.py > $O/r02at.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_solve.py tests/test_gpu_sweep.py tests/test_gpu_batch.py tests/test_gpu_dropin.py tests/test_gpu_distributed.py tests/test_gpu_paths.py -q -m gpu > $O/r02at_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02at_pytest.log
echo done
