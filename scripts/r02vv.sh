set -u
O=gpurun_out
DSE_LIB=build/ab_ws768u4.so DSE_PAIRS_WS=1 timeout 600 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py -m gpu -q -x > $O/r02vv_pytest.log 2>&1; echo "rc=$?" >> $O/r02vv_pytest.log
for i in 1 2; do
for v in ws768u4 ws768u3 ws768u2 ws768u8 ws640b; do
DSE_PAIRS_WS=1 timeout 300 bash scripts/ab_pairs.sh build/ab_$v.so >> $O/r02vv_ab.log 2>&1
done; done
echo done
