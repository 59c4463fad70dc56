set -u
O=gpurun_out
T=r02s3b
timeout 1200 python scripts/mu_newton_probe.py all > $O/${T}_newton.log 2>&1; echo "rc=$?" >> $O/${T}_newton.log
echo done
