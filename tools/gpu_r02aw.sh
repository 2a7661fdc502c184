#!/bin/bash
O=gpurun_out/aw; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg4.csv python -c "
import sys; sys.argv=['x']; import bench, torch, json
r = bench.cfg4_rate(torch.device('cuda', 0), steps=1, warmup=1) if 'steps' in bench.cfg4_rate.__code__.co_varnames else bench.cfg4_rate(torch.device('cuda', 0))
print(json.dumps(r))" > $O/run.txt 2>&1
python tools/launch_summary.py $O/launch_cfg4.csv > $O/launch_cfg4.txt 2>&1; head -16 $O/launch_cfg4.txt; tail -2 $O/run.txt | cut -c1-300
