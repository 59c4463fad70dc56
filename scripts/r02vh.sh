set -u
O=gpurun_out
DSE_LIB=build/ab_ne640u4.so timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_distributed.py tests/test_gpu_batch.py tests/test_gpu_checked.py tests/test_gpu_dropin.py -m gpu -q > $O/r02vh_pytest.log 2>&1; echo "rc=$?" >> $O/r02vh_pytest.log
for i in 1 2; do
bash scripts/ab_pairs.sh build/ab_t640m1u4.so build/ab_wf640u4.so build/ab_ne640u4.so build/ab_ne640u8.so build/ab_ne512u8.so build/ab_ne256u8.so build/ab_ne768u4.so >> $O/r02vh_ab.log 2>&1
done
echo done
