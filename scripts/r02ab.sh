set -u
O=gpurun_out
for v in old tpf0 tpf1 tpf2 tpf4 old tpf0 tpf1 tpf2 tpf4; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py pairs | sed "s/^/$v /" >> $O/r02ab.log 2>&1; done
DSE_AB_VARIANT=indexed-gpu-pairs DSE_LIB=build/ab_old.so timeout 600 python scripts/exact_ab.py $O/r02ab_old.npz > /dev/null 2>&1
DSE_AB_VARIANT=indexed-gpu-pairs DSE_LIB=build/ab_tpf1.so timeout 600 python scripts/exact_ab.py $O/r02ab_new.npz > /dev/null 2>&1
python -c "
import numpy as np
a=np.load('$O/r02ab_old.npz'); b=np.load('$O/r02ab_new.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('keys', len(a.files), 'differ', bad)" >> $O/r02ab.log 2>&1
echo done
