set -u
O=gpurun_out
for i in 1 2; do
python scripts/interp_sweep.py | sed "s/^/default /" >> $O/r02by.log 2>&1
DSE_INTERP_FAST=1 python scripts/interp_sweep.py | sed "s/^/fast1 /" >> $O/r02by.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_mu.py -q -m gpu -k "sharded_world1 or batched_successive" > $O/r02by_pytest.log 2>&1; echo "rc=$?" >> $O/r02by_pytest.log
echo done
