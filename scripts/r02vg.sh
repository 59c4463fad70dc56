set -u
O=gpurun_out
DSE_LIB=build/ab_g640u4.so timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_distributed.py tests/test_gpu_batch.py tests/test_gpu_checked.py tests/test_gpu_dropin.py -m gpu -q > $O/r02vg_pytest.log 2>&1; echo "rc=$?" >> $O/r02vg_pytest.log
for lib in build/ab_g640u4.so build/ab_g640u8.so build/ab_g512u8.so build/ab_g256u8.so build/ab_g320m2u4.so; do
for c in 1 2 4; do for gd in 1 2 4; do
echo -n "chunks=$c guide=$gd " >> $O/r02vg_ab.log
DSE_PAIRS_GUIDE=$gd DSE_PAIRS_CHUNKS=$c bash scripts/ab_pairs.sh $lib >> $O/r02vg_ab.log 2>&1
done; done; done
echo done
