set -u
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dse_solve_kernel -s 5 -c 1 -o $O/r02r_exact python scripts/exact_time.py exact > $O/r02r_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mu_batch_kernel -s 7 -c 1 -o $O/r02r_mubatch python scripts/mu_batch_probe.py > $O/r02r_ncu2.log 2>&1
echo done
