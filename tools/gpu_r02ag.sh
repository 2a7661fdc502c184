#!/bin/bash
# FFMA2 in spline_fwd_kernel (UKAN / general KAN forward): bitwise A/B against abtmp/lib_old.so + UKAN layer timing
O=gpurun_out/ag; mkdir -p $O
for sh in "ukan 1024 256 512" "ukan 333 64 128" "3000 100 100 20" "2000 50 512 100"; do
  n=$(echo $sh | tr ' ' '_')
  UKAN_B200_LIB=abtmp/lib_old.so timeout 300 python tools/fwd_ab.py $O/old_$n.npy $sh > /dev/null 2>&1
  timeout 300 python tools/fwd_ab.py $O/new_$n.npy $sh > /dev/null 2>&1
  python -c "
import numpy as np
a=np.load('$O/old_$n.npy'); b=np.load('$O/new_$n.npy'); print('$n bitwise', np.array_equal(a,b), float(np.abs(a-b).max()))" >> $O/ab.txt 2>&1
done
cat $O/ab.txt; rm -f $O/*.npy
for L in abtmp/lib_old.so paper_2408_11200_b200/libukan_b200.so abtmp/lib_old.so paper_2408_11200_b200/libukan_b200.so; do
  UKAN_B200_LIB=$L timeout 300 python tools/ukbench.py 4096 1024 1024 0.5 32 32 | sed "s|^|$L |" >> $O/kb.txt 2>&1
done
cut -c1-300 $O/kb.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spline_fwd -c 4 --csv --log-file $O/fwd_new.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
UKAN_B200_LIB=abtmp/lib_old.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spline_fwd -c 4 --csv --log-file $O/fwd_old.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
grep -h "gpu__time" $O/fwd_old.csv $O/fwd_new.csv | awk -F'","' '{print $NF}'
