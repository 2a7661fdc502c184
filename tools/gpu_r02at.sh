#!/bin/bash
# final ncu --set full digests of the cfg3 step kernels at the bench shape
O=gpurun_out/at; mkdir -p $O
for k in kan_fwd_tm_kernel kan_dx_tc_kernel kan_bwd_tc3_sweep_kernel; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/cfg3_$k -f python bench.py --steps 1 --warmup 0 --no-configs --no-cpu-baseline > /dev/null 2>&1
  echo "$k rc=$?"
done
python tools/ncu_digest.py $O/cfg3_kan_fwd_tm_kernel.ncu-rep $O/cfg3_kan_dx_tc_kernel.ncu-rep $O/cfg3_kan_bwd_tc3_sweep_kernel.ncu-rep > $O/ncu_digest_cfg3_final.jsonl 2>&1
rm -f $O/*.ncu-rep
python -c "
import json
for l in open('$O/ncu_digest_cfg3_final.jsonl'):
    d=json.loads(l); print(d['kernel'][:50], d.get('duration'), d.get('duration_unit'), 'dmma', d.get('dmma_pipe_pct'), 'fma', d.get('fma_pipe_pct'), 'issue', d.get('issue_active_pct'), 'dram', d.get('dram_read'), d.get('dram_write'))"
