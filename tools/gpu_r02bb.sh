#!/bin/bash
# tc3 for the 8-row-block / NT=8 shapes (cfg2 layer 0) now actually dispatched: bitwise A/B + timing
O=gpurun_out/bb; mkdir -p $O
for sh in "8192 784 256 32" "3001 37 100 30"; do
  n=$(echo $sh | tr ' ' '_')
  UKAN_TC3=0 timeout 300 python tools/tc3_ab.py $O/tc2_$n.npz $sh > /dev/null 2>&1
  timeout 300 python tools/tc3_ab.py $O/tc3_$n.npz $sh > /dev/null 2>&1
  python -c "
import numpy as np
A=np.load('$O/tc2_$n.npz'); B=np.load('$O/tc3_$n.npz')
print('$n', 'bitwise dC', np.array_equal(A['dC'],B['dC']), 'ds', np.array_equal(A['ds'],B['ds']))" >> $O/ab.txt
done
rm -f $O/*.npz
for e in "UKAN_TC3=0" "X=1" "UKAN_TC3=0" "X=1"; do env $e timeout 300 python tools/kbench.py 8192 784 256 32 3 | sed "s/^/$e /" | cut -c1-220 >> $O/kb.txt; done
cat $O/ab.txt $O/kb.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg2.csv python tools/cfg2_probe.py 3 > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg2.csv > $O/launch_cfg2.txt 2>&1; head -3 $O/launch_cfg2.txt
timeout 900 python -m pytest tests/test_parity_kan.py tests/test_parity_bench_shapes.py tests/test_train_gpu.py -x -q -m gpu 2>&1 | tail -1
