set -u
O=gpurun_out
python scripts/pairs_shape_probe.py pairs > $O/r02vb_pairs.log 2>&1
python scripts/pairs_shape_probe.py exact > $O/r02vb_exact.log 2>&1
echo done
