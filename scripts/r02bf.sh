set -u
O=gpurun_out
for r in 1 2 3; do for v in base sz; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py pairs | sed "s/^/$v /" >> $O/r02bf.log 2>&1; done; done
DSE_AB_VARIANT=indexed-gpu-pairs DSE_LIB=build/ab_base.so timeout 600 python scripts/exact_ab.py $O/r02bf_a.npz > /dev/null 2>&1
DSE_AB_VARIANT=indexed-gpu-pairs DSE_LIB=build/ab_sz.so timeout 600 python scripts/exact_ab.py $O/r02bf_b.npz > /dev/null 2>&1
python -c "
import numpy as np
a=np.load('$O/r02bf_a.npz'); b=np.load('$O/r02bf_b.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('keys', len(a.files), 'differ', bad)" >> $O/r02bf.log 2>&1
echo done
