set -u
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r02d_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02d_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 > $O/r02d_torchrun.json 2> $O/r02d_torchrun.err; echo "torchrun rc=$?" >> $O/r02d_torchrun.err
echo done
