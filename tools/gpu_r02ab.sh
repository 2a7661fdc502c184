#!/bin/bash
# tc3 sweep (TMA + mbarriers): bitwise A/B against tc2, parity tests, timing A/B, ncu
O=gpurun_out/ab; mkdir -p $O
UKAN_TC3=0 timeout 300 python tools/tc3_ab.py $O/tc2.npz > $O/ab.txt 2>&1
timeout 300 python tools/tc3_ab.py $O/tc3.npz >> $O/ab.txt 2>&1
UKAN_TC3=0 timeout 300 python tools/tc3_ab.py $O/tc2b.npz 3001 37 100 40 >> $O/ab.txt 2>&1
timeout 300 python tools/tc3_ab.py $O/tc3b.npz 3001 37 100 40 >> $O/ab.txt 2>&1
python -c "
import numpy as np
for a,b in (('tc2','tc3'),('tc2b','tc3b')):
    A=np.load('$O/'+a+'.npz'); B=np.load('$O/'+b+'.npz')
    print(a,b,'bitwise dC', np.array_equal(A['dC'],B['dC']), 'ds', np.array_equal(A['ds'],B['ds']), 'maxdiff', float(np.abs(A['dC']-B['dC']).max()))
" >> $O/ab.txt 2>&1
cat $O/ab.txt
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_dp_trainer_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for e in "UKAN_TC3=0" "X=1" "UKAN_TC3=0" "X=1"; do
  env $e timeout 300 python tools/kbench.py 16384 4096 4096 64 3 | sed "s/^/$e /" >> $O/kb.txt 2>&1
done
cut -c1-300 $O/kb.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc3 -c 1 -o $O/tc3 -f python tools/kbench.py 16384 4096 4096 64 3 > /dev/null 2>&1
python tools/ncu_digest.py $O/tc3.ncu-rep > $O/ncu_digest_tc3.jsonl 2>&1; rm -f $O/*.ncu-rep
head -c 3000 $O/ncu_digest_tc3.jsonl
