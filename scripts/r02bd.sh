set -u
O=gpurun_out
python scripts/api_tts.py > $O/r02bd.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/r02bd_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02bd_pytest.log
echo done
DSE_LIB=build/ab_prev.so python scripts/api_tts.py > gpurun_out/r02bd_prev.log 2>&1
