set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r02a_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02a_pytest.log
python scripts/interp_probe.py search 3 > $O/r02a_interp_search_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_batch -s 1 -c 1 -o $O/r02a_interp_search python scripts/interp_probe.py search 3 > $O/r02a_ncu_interp_search.log 2>&1
echo done
