set -u
O=gpurun_out
for v in prev new; do DSE_LIB=build/ab_$v.so python scripts/c0_tts.py >> $O/r02bt.log 2>&1; done
for a in pairs fast; do for v in prev new; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py $a | sed "s/^/$v /" >> $O/r02bt.log 2>&1; done; done
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_dropin.py tests/test_gpu_paths.py tests/test_gpu_batch.py tests/test_gpu_checked.py -q -m gpu > $O/r02bt_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02bt_pytest.log
echo done
