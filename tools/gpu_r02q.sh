#!/bin/bash
O=gpurun_out/q; mkdir -p $O
UKAN_DX_G64=1 timeout 900 python -m pytest tests/test_parity_bench_shapes.py -q -m gpu -x -k "cfg3 or part or multichunk" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for e in "X=0" "UKAN_DX_G64=1"; do env $e timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx | sed "s/^/$e /" >> $O/kb.txt 2>&1; done
cat $O/kb.txt | cut -c1-250
UKAN_DX_G64=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_dx_tc -c 1 -o $O/dx64 -f python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null; rm -f $O/*.ncu-rep
