#!/bin/bash
# FFMA2 TMEM forward: bitwise A/B against the previous build (abtmp/lib_old.so) + timing
O=gpurun_out/af; mkdir -p $O
for sh in "2048 512 1024 64" "1000 300 384 20" "4096 784 256 32"; do
  n=$(echo $sh | tr ' ' '_')
  UKAN_B200_LIB=abtmp/lib_old.so timeout 300 python tools/fwd_ab.py $O/old_$n.npy $sh > /dev/null 2>&1
  timeout 300 python tools/fwd_ab.py $O/new_$n.npy $sh > /dev/null 2>&1
  python -c "
import numpy as np
a=np.load('$O/old_$n.npy'); b=np.load('$O/new_$n.npy'); print('$n bitwise', np.array_equal(a,b), float(np.abs(a-b).max()))" >> $O/ab.txt
done
cat $O/ab.txt; rm -f $O/*.npy
for L in abtmp/lib_old.so paper_2408_11200_b200/libukan_b200.so abtmp/lib_old.so paper_2408_11200_b200/libukan_b200.so; do
  for sh in "16384 4096 4096 64 3" "8192 784 256 32 3"; do
    UKAN_B200_LIB=$L timeout 300 python tools/kbench.py $sh | sed "s|^|$L |" >> $O/kb.txt 2>&1
  done
done
cut -c1-260 $O/kb.txt
