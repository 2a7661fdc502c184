#!/bin/bash
# A/B kernel variants on one KAN shape: tools/ab.sh TAG "B d_in d_out G k [dx]" "ENV1" "ENV2" ...
TAG=$1; SHAPE=$2; shift 2
mkdir -p gpurun_out; O=gpurun_out/ab_$TAG.jsonl; : > $O
for env in "$@"; do env $env timeout 300 python tools/kbench.py $SHAPE >> $O 2>&1; done
cat $O
