#!/bin/bash
# DRAM bytes of the dx launch at the bench shape after the band change
O=gpurun_out/bf; mkdir -p $O
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:kan_dx_tc -c 1 --csv --log-file $O/dx_traffic.csv python bench.py --steps 1 --warmup 0 --no-configs --no-cpu-baseline > /dev/null 2>&1
grep -h "dram__\|gpu__time" $O/dx_traffic.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
