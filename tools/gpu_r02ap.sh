#!/bin/bash
# racecheck after per-thread stage releases in the tc3 sweep; tc3 timing A/B vs tc2 at the cfg3 shape
O=gpurun_out/ap; mkdir -p $O
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -2 $O/sanitize_racecheck.log
UKAN_TC3=0 timeout 300 python tools/tc3_ab.py $O/tc2.npz > /dev/null 2>&1; timeout 300 python tools/tc3_ab.py $O/tc3.npz > /dev/null 2>&1
python -c "
import numpy as np
A=np.load('$O/tc2.npz'); B=np.load('$O/tc3.npz'); print('bitwise', np.array_equal(A['dC'],B['dC']), np.array_equal(A['ds'],B['ds']))"
rm -f $O/*.npz
for e in "UKAN_TC3=0" "X=1"; do env $e timeout 300 python tools/kbench.py 16384 4096 4096 64 3 | sed "s/^/$e /" | cut -c1-200; done
