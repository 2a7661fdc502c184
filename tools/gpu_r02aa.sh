#!/bin/bash
# full GPU suite + smoke + the N=2 reference arm under torchrun (rank 0 runs, rank 1 exits 0)
O=gpurun_out/aa; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/ref2.json 2> $O/ref2.err; echo "ref2 rc=$?"
tail -c 800 $O/ref2.json
