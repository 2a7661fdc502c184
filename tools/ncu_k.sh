#!/bin/bash
# ncu --set full of the KAN kernels on one shape: tools/ncu_k.sh TAG "B d_in d_out G k [dx]" [env...]
TAG=$1; SHAPE=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:'kan|spline' -s 2 -c 4 \
  -o gpurun_out/prof_$TAG -f python tools/kbench.py $SHAPE > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
