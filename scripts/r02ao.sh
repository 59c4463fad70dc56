set -u
O=gpurun_out
for r in 1 2; do for v in base t3 hd t3hd; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py exact | sed "s/^/$v /" >> $O/r02ao.log 2>&1; done; done
DSE_LIB=build/ab_base.so timeout 600 python scripts/exact_ab.py $O/r02ao_base.npz > /dev/null 2>&1
for v in t3 hd t3hd; do
DSE_LIB=build/ab_$v.so timeout 600 python scripts/exact_ab.py $O/r02ao_$v.npz > /dev/null 2>&1
python -c "
import numpy as np
a=np.load('$O/r02ao_base.npz'); b=np.load('$O/r02ao_$v.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('$v keys', len(a.files), 'differ', bad)" >> $O/r02ao.log 2>&1
done
echo done
