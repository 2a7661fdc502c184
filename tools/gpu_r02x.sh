#!/bin/bash
O=gpurun_out/x; mkdir -p $O
for e in "X=0" "UKAN_BWD=sw" "UKAN_BWD=reg" "UKAN_BWD=wide" "UKAN_BWD=dmma" "UKAN_FWD=smem" "UKAN_FWD_V2=1"; do
  env $e timeout 120 python tools/kbench.py 1024 64 64 10 3 | sed "s/^/$e /" >> $O/kb.txt 2>&1
done
cat $O/kb.txt | cut -c1-250
