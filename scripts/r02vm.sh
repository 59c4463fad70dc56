set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_interp.py tests/test_cubic.py tests/test_gpu_dropin.py -m gpu -q > $O/r02vm_pytest.log 2>&1; echo "rc=$?" >> $O/r02vm_pytest.log
python scripts/interp_sweep.py > $O/r02vm_interp.log 2>&1
echo done
