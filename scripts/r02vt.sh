set -u
O=gpurun_out
export DSE_LIB=build/ab_ws.so
DSE_PAIRS_WS=1 timeout 120 python scripts/exact_time.py pairs > $O/r02vt_time.log 2>&1; echo "rc=$?" >> $O/r02vt_time.log
DSE_PAIRS_WS=0 timeout 120 python scripts/exact_time.py pairs >> $O/r02vt_time.log 2>&1; echo "rc=$?" >> $O/r02vt_time.log
DSE_PAIRS_WS=1 timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_distributed.py tests/test_gpu_checked.py -m gpu -q -x > $O/r02vt_pytest.log 2>&1; echo "rc=$?" >> $O/r02vt_pytest.log
for i in 1 2; do
DSE_PAIRS_WS=1 timeout 300 bash scripts/ab_pairs.sh build/ab_ws.so >> $O/r02vt_ab.log 2>&1
DSE_PAIRS_WS=0 timeout 300 bash scripts/ab_pairs.sh build/ab_ws.so >> $O/r02vt_ab.log 2>&1
done
echo done
