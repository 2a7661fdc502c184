#!/bin/bash
O=gpurun_out/ba; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg2.csv python tools/cfg2_probe.py 3 > $O/probe.txt 2>&1
python tools/launch_summary.py $O/launch_cfg2.csv > $O/launch_cfg2.txt 2>&1; head -20 $O/launch_cfg2.txt; tail -1 $O/probe.txt
