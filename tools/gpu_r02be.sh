#!/bin/bash
O=gpurun_out/be; mkdir -p $O
for pn in 16 8 32 64 4 16; do
  UKAN_TC3_PANEL=$pn timeout 300 python tools/bucket_ab.py 8 | sed "s/^/panel=$pn /" >> $O/kb.txt
done
cat $O/kb.txt
