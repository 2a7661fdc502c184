#!/bin/bash
O=gpurun_out/ac; mkdir -p $O
UKAN_TC3=0 timeout 300 python tools/tc3_ab.py $O/tc2.npz 3001 37 100 40 > $O/ab.txt 2>&1
for d in 0 1 2 3; do UKAN_TC3_DBG=$d timeout 300 python tools/tc3_ab.py $O/tc3_$d.npz 3001 37 100 40 >> $O/ab.txt 2>&1; done
UKAN_TC3_DBG=0 timeout 300 python tools/tc3_ab.py $O/tc3_0b.npz 3001 37 100 40 >> $O/ab.txt 2>&1
python -c "
import numpy as np
A=np.load('$O/tc2.npz')
for d in ['0','1','2','3','0b']:
    B=np.load('$O/tc3_'+d+'.npz'); dd=np.abs(A['dC']-B['dC'])
    bad=np.argwhere(dd>1e-3)
    print(d,'bitwise', np.array_equal(A['dC'],B['dC']), np.array_equal(A['ds'],B['ds']), 'maxdiff', float(dd.max()), 'nbad', len(bad), 'feat', np.unique(bad[:,0])[:20] if len(bad) else None, 'rows', np.unique(bad[:,1])[:20] if len(bad) else None, 'outs', np.unique(bad[:,2])[:40] if len(bad) else None)
" >> $O/ab.txt 2>&1
cat $O/ab.txt
