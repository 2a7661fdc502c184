#!/bin/bash
# where the DMMA kernels lose time: staging / barriers vs the DMMA inner loop (diag modes give wrong results)
O=gpurun_out/n; mkdir -p $O
for e in "X=0" "UKAN_DX_DIAG=1" "UKAN_DX_DIAG=2" "UKAN_TC2_DIAG=1" "UKAN_TC2_DIAG=2"; do
  env $e timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx | sed "s/^/$e /" >> $O/kb.txt 2>&1
done
cat $O/kb.txt | cut -c1-260
