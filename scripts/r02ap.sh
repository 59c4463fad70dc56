set -u
O=gpurun_out
for r in 1 2; do
DSE_MU_MIRROR=0 python scripts/mu_step_probe.py bcb 10 | sed "s/^/plain /" >> $O/r02ap.log 2>&1
python scripts/mu_step_probe.py bcb 10 | sed "s/^/mirror /" >> $O/r02ap.log 2>&1
done
DSE_MU_MIRROR=0 python scripts/mu_moments_time.py 10 | sed "s/^/plain_moments /" >> $O/r02ap.log 2>&1
python scripts/mu_moments_time.py 10 | sed "s/^/mirror_moments /" >> $O/r02ap.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_mu.py tests/test_gpu_mu_full.py -q -m gpu > $O/r02ap_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02ap_pytest.log
echo done
