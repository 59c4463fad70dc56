set -u
O=gpurun_out
python scripts/mu_batch_probe.py >> $O/r02w.log 2>&1
python scripts/mu_sa_probe.py >> $O/r02w.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mu.py tests/test_gpu_mu_full.py -q -x > $O/r02w_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02w_pytest.log
echo done
