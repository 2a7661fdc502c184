#!/bin/bash
O=gpurun_out/w; mkdir -p $O
T0=$(date +%s); timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall=$(( $(date +%s) - T0 ))s"
tail -3 $O/bench.err
python - <<'PY'
import json
l=[x for x in open("gpurun_out/w/bench.json") if x.startswith("{")][-1]
d=json.loads(l)
print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["traffic"])
for k in ("cfg4_ukan_layer","ukan_layer","cfg5_ukan_dp","cfg2_kan_stack_dp"): print(k, d[k]["samples_per_s"], d[k]["ms_per_step"], d[k].get("n_u"))
print(d["kan_layers"])
PY
