#!/bin/bash
# tc3 with NT = 8 (cfg2 layer-0 sweep): bitwise A/B vs tc2, timing A/B, parity tests
O=gpurun_out/ad; mkdir -p $O
for sh in "8192 784 256 32" "3001 37 100 30" "5000 70 256 64"; do
  n=$(echo $sh | tr ' ' '_')
  UKAN_TC3=0 timeout 300 python tools/tc3_ab.py $O/tc2_$n.npz $sh > /dev/null 2>&1
  timeout 300 python tools/tc3_ab.py $O/tc3_$n.npz $sh > /dev/null 2>&1
  python -c "
import numpy as np
A=np.load('$O/tc2_$n.npz'); B=np.load('$O/tc3_$n.npz')
print('$n', 'bitwise dC', np.array_equal(A['dC'],B['dC']), 'ds', np.array_equal(A['ds'],B['ds']), 'maxdiff', float(np.abs(A['dC']-B['dC']).max()))" >> $O/ab.txt 2>&1
done
cat $O/ab.txt
rm -f $O/*.npz
timeout 1200 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_train_gpu.py tests/test_dp_trainer_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
for e in "UKAN_TC3=0" "X=1" "UKAN_TC3=0" "X=1"; do
  env $e timeout 300 python tools/kbench.py 8192 784 256 32 3 | sed "s/^/$e /" >> $O/kb.txt 2>&1
done
cut -c1-300 $O/kb.txt
