set -u
O=gpurun_out
DSE_LIB=build/ab_st640u4.so timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_distributed.py tests/test_gpu_batch.py tests/test_gpu_checked.py tests/test_gpu_dropin.py -m gpu -q > $O/r02vf_pytest.log 2>&1; echo "rc=$?" >> $O/r02vf_pytest.log
for lib in build/ab_st640u4.so build/ab_st640u8.so build/ab_st256u8.so build/ab_st512u8.so build/ab_st768u4.so build/ab_st704u4.so build/ab_st576u4.so build/ab_st320m2u4.so; do
bash scripts/ab_pairs.sh $lib >> $O/r02vf_ab.log 2>&1
done
for c in 1 2 4 8 16; do
echo -n "chunks=$c " >> $O/r02vf_ab.log
DSE_PAIRS_CHUNKS=$c bash scripts/ab_pairs.sh build/ab_st640u4.so >> $O/r02vf_ab.log 2>&1
done
echo done
