#!/bin/bash
# bench after the tc3 sweep + cfg3 launch list + traffic of the tc3 sweep at the bench shape
O=gpurun_out/ae; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], json.dumps(d['phase_ms'])); print(json.dumps(d['roofline']))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launch_cfg3.csv python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg3.csv 2>&1 | head -20
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:kan_bwd_tc3 -c 8 --csv --log-file $O/tc3_traffic.csv python bench.py --steps 1 --warmup 0 --no-configs --no-cpu-baseline > /dev/null 2>&1
tail -30 $O/tc3_traffic.csv | cut -c1-400
