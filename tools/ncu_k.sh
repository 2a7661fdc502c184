#!/bin/bash
# ncu --set full of one kernel family on one KAN shape:
#   tools/ncu_k.sh TAG "B d_in d_out G k [dx]" KERNEL_REGEX [env...]
TAG=$1; SHAPE=$2; KRE=$3; shift 3
mkdir -p gpurun_out
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 3 -c 1 \
  -o gpurun_out/prof_$TAG -f python tools/kbench.py $SHAPE > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
