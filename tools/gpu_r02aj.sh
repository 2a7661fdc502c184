#!/bin/bash
# full GPU suite + smoke + bench after the FFMA2 / pre-split table GEMM changes
O=gpurun_out/aj; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], json.dumps(d['phase_ms'])); print(json.dumps(d['roofline'])); print(d['clocks'])
print('cfg1', d['kan_layers']['cfg1_graph_step']['ms_per_step'], 'cfg2', d['cfg2_kan_stack_dp']['ms_per_step'], 'cfg5', d['cfg5_ukan_dp']['ms_per_step'], 'ukan', d['ukan_layer']['ms_per_step'], 'cfg4', d['cfg4_ukan_layer']['ms_per_step'], d['cfg4_ukan_layer']['samples_per_s'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_ukan.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
python tools/launch_summary.py $O/launch_ukan.csv > $O/launch_ukan.txt 2>&1; head -16 $O/launch_ukan.txt
