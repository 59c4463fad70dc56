set -u
O=gpurun_out
T=r02s3d
timeout 900 python -m pytest tests/test_gpu_mu.py -q -m gpu -k "newton or anderson" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
echo done
