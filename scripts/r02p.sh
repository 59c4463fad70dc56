set -u
O=gpurun_out
for v in base smacc minb1 base smacc; do DSE_LIB=build/ab_$v.so python scripts/mu_sa_group.py >> $O/r02p_ab.log 2>&1; done
echo done
