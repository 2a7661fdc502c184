#!/bin/bash
O=gpurun_out/u; mkdir -p $O
for v in v5 v52; do
  UKAN_DX=$v timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py -q -m gpu -x -k "cfg3 or part or multichunk or degrees or base or deterministic" > $O/pytest_$v.log 2>&1; echo "$v rc=$?"; tail -1 $O/pytest_$v.log
done
for e in "X=0" "UKAN_DX=v5" "UKAN_DX=v52"; do env $e timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx | sed "s/^/$e /" >> $O/kb.txt 2>&1; done
cat $O/kb.txt | cut -c1-240
UKAN_DX=v5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_dx_v5 -c 1 -o $O/v5 -f python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null; rm -f $O/*.ncu-rep
