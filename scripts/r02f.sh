set -u
O=gpurun_out
python scripts/cluster_probe.py > $O/r02f_cluster.log 2>&1
DSE_NO_CLUSTER=1 python scripts/cluster_probe.py >> $O/r02f_cluster.log 2>&1
DSE_NO_CLUSTER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/r02f_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/r02f_ncu_smoke.log 2>&1; echo "ncu rc=$?" >> $O/r02f_ncu_smoke.log
echo done
