set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_interp.py tests/test_cubic.py tests/test_gpu_paths.py -q -m gpu > $O/r02g_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02g_pytest.log
for R in 0 2 3; do for T in 256 512 1024; do DSE_INTERP_REP=$R DSE_INTERP_THREADS=$T python scripts/interp_sweep.py >> $O/r02g_interp.jsonl 2>&1; done; done
python scripts/interp_sweep.py >> $O/r02g_interp.jsonl 2>&1
echo done
