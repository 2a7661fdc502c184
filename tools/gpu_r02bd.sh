#!/bin/bash
O=gpurun_out/bd; mkdir -p $O
for bnd in 32 64 128 32; do
  UKAN_DX_BAND=$bnd timeout 600 python tools/kbench.py 65536 4096 4096 64 3 dx | sed "s/^/band=$bnd /" | cut -c1-230 >> $O/kb.txt
done
cat $O/kb.txt
