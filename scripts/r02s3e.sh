set -u
O=gpurun_out
T=r02s3e
for r in 1 2 3; do for v in base late; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py pairs | sed "s/^/$v /" >> $O/${T}.log 2>&1; done; done
DSE_AB_VARIANT=indexed-gpu-pairs DSE_LIB=build/ab_base.so timeout 600 python scripts/exact_ab.py $O/${T}_base.npz > /dev/null 2>&1
DSE_AB_VARIANT=indexed-gpu-pairs DSE_LIB=build/ab_late.so timeout 600 python scripts/exact_ab.py $O/${T}_late.npz > /dev/null 2>&1
python -c "
import numpy as np
a=np.load('$O/${T}_base.npz'); b=np.load('$O/${T}_late.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('keys', len(a.files), 'differ', bad)" >> $O/${T}.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mu.py -q -m gpu -k "newton" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
echo done
