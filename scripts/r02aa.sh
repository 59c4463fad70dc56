set -u
O=gpurun_out
T=r02aa
timeout 2400 python -m pytest tests -m gpu -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
python scripts/interp_sweep.py > $O/${T}_interp_sweep.log 2>&1
python scripts/interp_sweep.py >> $O/${T}_interp_sweep.log 2>&1
python scripts/interp_probe.py direct 3 > $O/${T}_interp_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/${T}_interp_direct python scripts/interp_probe.py direct 3 > $O/${T}_ncu_interp1.log 2>&1
echo done
