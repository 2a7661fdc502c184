#!/bin/bash
# dx band sweep at the full cfg3 batch
O=gpurun_out/bc; mkdir -p $O
for bnd in 8 4 16 32 8; do
  UKAN_DX_BAND=$bnd timeout 600 python tools/kbench.py 65536 4096 4096 64 3 dx | sed "s/^/band=$bnd /" | cut -c1-230 >> $O/kb.txt
done
cat $O/kb.txt
