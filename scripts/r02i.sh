set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_interp.py tests/test_cubic.py -q -m gpu > $O/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02i_pytest.log
python scripts/interp_sweep.py > $O/r02i_interp.jsonl 2>&1
DSE_INTERP_NOSTREAM=1 python scripts/interp_sweep.py >> $O/r02i_interp.jsonl 2>&1
DSE_INTERP_REP=2 python scripts/interp_sweep.py >> $O/r02i_interp.jsonl 2>&1
echo done
