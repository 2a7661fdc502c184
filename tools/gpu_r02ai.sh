#!/bin/bash
# pre-split table GEMM: bitwise A/B (UKAN_CG_PRESPLIT=0), parity tests, timing
O=gpurun_out/ai; mkdir -p $O
for sh in "ukan 1024 256 512" "ukan 333 64 128" "ukan 4096 1024 1024"; do
  n=$(echo $sh | tr ' ' '_')
  UKAN_CG_PRESPLIT=0 timeout 300 python tools/fwd_ab.py $O/old_$n.npy $sh > $O/err_old_$n.txt 2>&1
  timeout 300 python tools/fwd_ab.py $O/new_$n.npy $sh > $O/err_new_$n.txt 2>&1
  python -c "
import numpy as np
a=np.load('$O/old_$n.npy'); b=np.load('$O/new_$n.npy'); print('$n bitwise', np.array_equal(a,b), float(np.abs(a-b).max()))" >> $O/ab.txt 2>&1
done
cat $O/ab.txt; tail -3 $O/err_new_*.txt; rm -f $O/*.npy
timeout 1200 python -m pytest tests/test_parity_ukan.py tests/test_cg_tc.py tests/test_parity_bench_shapes.py tests/test_dp_trainer_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
for e in "UKAN_CG_PRESPLIT=0" "X=1" "UKAN_CG_PRESPLIT=0" "X=1"; do
  env $e timeout 300 python tools/ukbench.py 4096 1024 1024 0.5 32 32 | sed "s|^|$e |" >> $O/kb.txt 2>&1
done
cut -c1-250 $O/kb.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cg_table|cg_presplit" -c 6 --csv --log-file $O/tc.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
grep -h "gpu__time" $O/tc.csv | awk -F'","' '{print $5, $NF}' | cut -c1-120
timeout 600 ncu --set full --clock-control none -k regex:cg_table -c 1 -o $O/tbl -f python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
python tools/ncu_digest.py $O/tbl.ncu-rep > $O/ncu_digest_table.jsonl 2>&1; rm -f $O/*.ncu-rep; head -c 1500 $O/ncu_digest_table.jsonl
