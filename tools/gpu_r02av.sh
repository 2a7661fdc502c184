#!/bin/bash
# forward slab multicast across a 2-CTA cluster (UKAN_FWD_MC=1): bitwise A/B + timing
O=gpurun_out/av; mkdir -p $O
for sh in "2048 512 1024 64" "1000 300 384 20" "4096 784 256 32" "333 70 256 64"; do
  n=$(echo $sh | tr ' ' '_')
  timeout 120 python tools/fwd_ab.py $O/a_$n.npy $sh > /dev/null 2>&1
  UKAN_FWD_MC=1 timeout 120 python tools/fwd_ab.py $O/b_$n.npy $sh > $O/err_$n.txt 2>&1
  python -c "
import numpy as np
a=np.load('$O/a_$n.npy'); b=np.load('$O/b_$n.npy'); print('$n bitwise', np.array_equal(a,b), float(np.abs(a-b).max()))" >> $O/ab.txt 2>&1
done
cat $O/ab.txt; rm -f $O/*.npy
for e in "X=0" "UKAN_FWD_MC=1" "X=0" "UKAN_FWD_MC=1"; do
  for sh in "16384 4096 4096 64 3" "8192 784 256 32 3"; do
    env $e timeout 300 python tools/kbench.py $sh | sed "s|^|$e |" | cut -c1-200
  done
done
