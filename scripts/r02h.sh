set -u
O=gpurun_out
python scripts/interp_probe.py direct 3 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_batch -s 1 -c 1 -o $O/r02h_interp_direct python scripts/interp_probe.py direct 3 > $O/r02h_ncu1.log 2>&1
python scripts/interp_probe.py cubic_direct 3 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_batch -s 1 -c 1 -o $O/r02h_interp_cubic python scripts/interp_probe.py cubic_direct 3 > $O/r02h_ncu2.log 2>&1
echo done
