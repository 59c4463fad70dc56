set -u
O=gpurun_out
T=r02va
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_smi.txt 2>&1
nproc > $O/${T}_nproc.txt
timeout 2700 python -m pytest tests -m gpu -q --durations=15 > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?" >> $O/${T}_bench.err
timeout 600 python bench.py --impl reference > $O/${T}_ref.json 2> $O/${T}_ref.err; echo "ref rc=$?" >> $O/${T}_ref.err
echo done
