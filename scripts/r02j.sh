set -u
O=gpurun_out
python scripts/interp_probe.py direct 3 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/r02j_stream_direct python scripts/interp_probe.py direct 3 > $O/r02j_ncu1.log 2>&1
python scripts/interp_probe.py cubic_direct 3 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_stream -s 1 -c 1 -o $O/r02j_stream_cubic python scripts/interp_probe.py cubic_direct 3 > $O/r02j_ncu2.log 2>&1
echo done
