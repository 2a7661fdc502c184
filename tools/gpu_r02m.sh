#!/bin/bash
# the N > 1 bench path on one GPU: two ranks over gloo sharing cuda:0 (the driver's scaling run uses NCCL)
O=gpurun_out/m; mkdir -p $O
UKAN_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
tail -c 1500 $O/bench2.json; grep -v "^\s*$" $O/bench2.err | tail -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/ref2.json 2> $O/ref2.err; echo "ref2 rc=$?"
tail -c 800 $O/ref2.json
