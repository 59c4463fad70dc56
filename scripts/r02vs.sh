set -u
O=gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 5 > $O/r02vs_torchrun.json 2> $O/r02vs_torchrun.err; echo "rc=$?" >> $O/r02vs_torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $O/r02vs_torchrun_ref.json 2> $O/r02vs_torchrun_ref.err; echo "rc=$?" >> $O/r02vs_torchrun_ref.err
echo done
