#!/bin/bash
O=gpurun_out/ak; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg5.csv python tools/cfg5_probe.py 2 > $O/probe.txt 2>&1
python tools/launch_summary.py $O/launch_cfg5.csv > $O/launch_cfg5.txt 2>&1; head -25 $O/launch_cfg5.txt; tail -2 $O/probe.txt
