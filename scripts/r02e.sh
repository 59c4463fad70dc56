set -u
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/r02e_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/r02e_ncu_smoke.log 2>&1; echo "ncu rc=$?" >> $O/r02e_ncu_smoke.log
DSE_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 > $O/r02e_dist.json 2> $O/r02e_dist.err; echo "dist rc=$?" >> $O/r02e_dist.err
echo done
