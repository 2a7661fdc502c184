#!/bin/bash
# variants of the KAN kernels on the bench shapes
mkdir -p gpurun_out
O=gpurun_out/kbench_${1:-a}.jsonl
: > $O
for env in "" "UKAN_NO_TC=1" "UKAN_NO_TC=1 UKAN_NO_DMMA=1" "UKAN_FWD_V2=1"; do
  for shp in "8192 784 256 32 3" "8192 256 10 32 3 dx" "8192 256 256 32 3 dx" "16384 4096 4096 64 3 dx"; do
    env $env timeout 120 python tools/kbench.py $shp >> $O 2>&1
  done
done
cat $O
