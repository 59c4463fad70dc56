set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mu.py tests/test_gpu_mu_full.py -q -x > $O/r02o_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02o_pytest.log
timeout 600 python scripts/mu_sa_probe.py > $O/r02o_sa.log 2>&1; echo "rc=$?" >> $O/r02o_sa.log
echo done
