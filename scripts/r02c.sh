set -u
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r02c_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02c_pytest.log
echo done
