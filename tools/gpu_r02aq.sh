#!/bin/bash
# full validation: GPU suite, smoke, bench (default args), reference arm
O=gpurun_out/aq; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], json.dumps(d['phase_ms'])); print(d['roofline']['frac'], d['clocks'], d['gpu_launches'])
print('cfg1', d['kan_layers']['cfg1_graph_step']['ms_per_step'], 'cfg2', d['cfg2_kan_stack_dp']['ms_per_step'], 'cfg5', d['cfg5_ukan_dp']['ms_per_step'], 'ukan', d['ukan_layer']['ms_per_step'], 'cfg4', d['cfg4_ukan_layer']['ms_per_step'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; tail -c 400 $O/bench_ref.json
