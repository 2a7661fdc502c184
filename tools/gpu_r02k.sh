#!/bin/bash
O=gpurun_out/k; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_bench_shapes.py -q -m gpu -x -k "cfg3 or part or multichunk" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
UKAN_TC2_RB16_WPF=84 timeout 900 python -m pytest tests/test_parity_bench_shapes.py -q -m gpu -x -k "cfg3 or part" >> $O/pytest.log 2>&1; echo "rc84=$?" >> $O/pytest.log
tail -4 $O/pytest.log
for e in "UKAN_TC2_RB16_WPF=4" "UKAN_TC2_RB16_WPF=84"; do env $e timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx >> $O/kb.jsonl 2>&1; done
cat $O/kb.jsonl
for b in 4 8 32; do UKAN_DX_BAND=$b timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:kan_dx_tc -c 1 --csv python tools/kbench.py 16384 4096 4096 64 3 dx 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/band=$b /" >> $O/dx_band.txt; done
cat $O/dx_band.txt | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_dx_tc -c 1 -o $O/cfg3_dx -f python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
UKAN_TC2_RB16_WPF=84 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg3_tc2_84 -f python tools/kbench.py 16384 4096 4096 64 3 > /dev/null 2>&1
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null
rm -f $O/*.ncu-rep
