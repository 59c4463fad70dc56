set -u
O=gpurun_out
python scripts/batch_mom_probe.py > $O/r02ay.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_batch.py -q -m gpu > $O/r02ay_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02ay_pytest.log
echo done
