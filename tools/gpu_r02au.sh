#!/bin/bash
# N = 2 bench path (two ranks sharing one GPU over gloo) with the final code
O=gpurun_out/au; mkdir -p $O
UKAN_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
python -c "
import json; d=json.loads(open('$O/bench2.json').read().strip().splitlines()[-1])
print(d['n_gpus'], d['value'], d['e2e']['value'], d['config']['parallelism'], d['cfg5_ukan_dp']['ms_per_step'], d['cfg5_ukan_dp']['n_gpus'])"
tail -3 $O/bench2.err
