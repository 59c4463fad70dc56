set -u
O=gpurun_out
python scripts/mom_tts.py > $O/r02ag.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_sweep.py tests/test_gpu_batch.py tests/test_gpu_dropin.py tests/test_gpu_distributed.py -q -m gpu > $O/r02ag_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02ag_pytest.log
echo done
