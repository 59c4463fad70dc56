set -u
O=gpurun_out
T=r02s3c
timeout 1500 python scripts/mu_newton_c3.py > $O/${T}_newton.log 2>&1; echo "rc=$?" >> $O/${T}_newton.log
echo done
