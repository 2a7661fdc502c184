#!/bin/bash
O=gpurun_out/l; mkdir -p $O
timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx >> $O/kb.jsonl 2>&1
cat $O/kb.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"kan_dx_tc|kan_bwd_tc2" --csv python tools/kbench.py 16384 4096 4096 64 3 dx 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-160 | tail -6
