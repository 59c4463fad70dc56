set -u
O=gpurun_out
for i in 1 2; do
DSE_INTERP_FAST=0 python scripts/interp_sweep.py >> $O/r02m_interp.jsonl 2>&1
DSE_INTERP_FAST=1 python scripts/interp_sweep.py >> $O/r02m_interp.jsonl 2>&1
done
echo done
