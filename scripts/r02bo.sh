set -u
O=gpurun_out
for r in 1 2; do for v in prev new; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py exact | sed "s/^/$v /" >> $O/r02bo.log 2>&1; done; done
DSE_AB_EXTRA=40 DSE_LIB=build/ab_prev.so timeout 900 python scripts/exact_ab.py $O/r02bo_a.npz >> $O/r02bo.log 2>&1
DSE_AB_EXTRA=40 DSE_LIB=build/ab_new.so timeout 900 python scripts/exact_ab.py $O/r02bo_b.npz >> $O/r02bo.log 2>&1
python -c "
import numpy as np
a=np.load('$O/r02bo_a.npz'); b=np.load('$O/r02bo_b.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('keys', len(a.files), 'differ', bad)" >> $O/r02bo.log 2>&1
DSE_LIB=build/ab_new.so timeout 600 python -m pytest tests/test_gpu_exp.py -q -m gpu >> $O/r02bo.log 2>&1
echo done
