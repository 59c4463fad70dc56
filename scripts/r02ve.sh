set -u
O=gpurun_out
DSE_LIB=build/ab_s640u4.so timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_distributed.py tests/test_gpu_batch.py tests/test_gpu_checked.py -m gpu -q -x > $O/r02ve_pytest.log 2>&1; echo "rc=$?" >> $O/r02ve_pytest.log
for lib in paper_2012_03667_b200/libdse_b200.so build/ab_s256.so build/ab_s640u4.so build/ab_s640u8.so; do
for sp in 0,4 1,4 2,4 3,4 4,4 2,2 4,2 1,8 2,8; do
echo -n "split=$sp " >> $O/r02ve_ab.log
DSE_PAIRS_SPLIT=$sp bash scripts/ab_pairs.sh $lib >> $O/r02ve_ab.log 2>&1
done; done
echo done
