#!/bin/bash
# quick GPU iteration: parity tests + kernel timings on the bench shapes
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -15 gpurun_out/pytest_$TAG.log
O=gpurun_out/kb_$TAG.jsonl; : > $O
shift
for env in "$@"; do
  for shp in "8192 784 256 32 3" "8192 256 10 32 3 dx" "8192 256 256 32 3 dx" "16384 4096 4096 64 3 dx"; do
    env $env timeout 120 python tools/kbench.py $shp >> $O 2>&1
  done
done
cat $O
