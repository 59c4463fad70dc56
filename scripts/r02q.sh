set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_exp.py -q > $O/r02q_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02q_pytest.log
DSE_LIB=build/ab_base.so timeout 600 python scripts/exact_ab.py $O/r02q_base.npz > $O/r02q_ab.log 2>&1
DSE_LIB=build/ab_exprep.so timeout 600 python scripts/exact_ab.py $O/r02q_new.npz >> $O/r02q_ab.log 2>&1
python -c "
import numpy as np
a=np.load('$O/r02q_base.npz'); b=np.load('$O/r02q_new.npz')
bad=[k for k in a.files if not np.array_equal(a[k].view(np.int64) if a[k].dtype==np.float64 else a[k], b[k].view(np.int64) if b[k].dtype==np.float64 else b[k])]
print('keys', len(a.files), 'differ', bad)" >> $O/r02q_ab.log 2>&1
for v in base exprep base exprep; do DSE_LIB=build/ab_$v.so python scripts/exact_time.py exact >> $O/r02q_time.log 2>&1; done
echo done
