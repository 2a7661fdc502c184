#!/bin/bash
O=gpurun_out/j; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py -q -m gpu -x -k "cfg3 or cfg2 or multichunk or part or side_stream" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
UKAN_TC2_RB16_WPF=8 timeout 900 python -m pytest tests/test_parity_bench_shapes.py -q -m gpu -x -k "cfg3 or part" >> $O/pytest.log 2>&1; echo "rc8=$?" >> $O/pytest.log
tail -6 $O/pytest.log
for e in "UKAN_TC2_RB16_WPF=4" "UKAN_TC2_RB16_WPF=8"; do env $e UKAN_DX_WARPS=16 timeout 300 python tools/kbench.py 16384 4096 4096 64 3 >> $O/kb.jsonl 2>&1; done
timeout 300 python tools/kbench.py 8192 784 256 32 3 >> $O/kb.jsonl 2>&1
cat $O/kb.jsonl
for e in 4 8; do UKAN_TC2_RB16_WPF=$e timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg3_tc2_$e -f python tools/kbench.py 16384 4096 4096 64 3 > /dev/null 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg2_tc2 -f python tools/kbench.py 8192 784 256 32 3 > /dev/null 2>&1
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null
rm -f $O/*.ncu-rep
