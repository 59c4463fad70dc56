set -u
O=gpurun_out
for v in prev base prev base; do DSE_LIB=build/ab_$v.so python scripts/c0_tts.py >> $O/r02bk.log 2>&1; done
for a in pairs exact fast; do for v in prev base; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py $a | sed "s/^/$v /" >> $O/r02bk.log 2>&1; done; done
for var in indexed-gpu-exact indexed-gpu; do
DSE_AB_VARIANT=$var DSE_LIB=build/ab_prev.so timeout 600 python scripts/exact_ab.py $O/r02bk_a.npz > /dev/null 2>&1
DSE_AB_VARIANT=$var DSE_LIB=build/ab_base.so timeout 600 python scripts/exact_ab.py $O/r02bk_b.npz > /dev/null 2>&1
python -c "
import numpy as np
a=np.load('$O/r02bk_a.npz'); b=np.load('$O/r02bk_b.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('$var keys', len(a.files), 'differ', bad)" >> $O/r02bk.log 2>&1
done
echo done
