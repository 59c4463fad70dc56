set -u
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exp.py tests/test_gpu_interp.py tests/test_cubic.py tests/test_gpu_mu_full.py tests/test_gpu_mu.py -q -m gpu > $O/r02cb_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02cb_pytest.log
for i in 1 2; do python scripts/interp_sweep.py >> $O/r02cb_interp.log 2>&1; done
echo done
