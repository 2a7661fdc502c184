#!/bin/bash
# small-layer path v2 (one table-gradient kernel; mse block partials)
O=gpurun_out/z; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_kan.py tests/test_dp_trainer_gpu.py tests/test_train_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1
tail -5 $O/pytest.txt
for e in "X=0" "UKAN_SMALL=0"; do
  for s in "1024 64 64 10 3" "2048 64 64 10 3" "256 128 128 10 3" "1024 32 128 20 3"; do
    env $e timeout 120 python tools/kbench.py $s | sed "s/^/$e $s /" >> $O/kb.txt 2>&1
  done
done
cut -c1-250 $O/kb.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg1.csv python tools/cfg1_probe.py 3 > /dev/null 2>&1
for k in kan_small_fwd kan_small_tablegrad kan_small_records sum_f64; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/$k python tools/cfg1_probe.py 1 > /dev/null 2>&1
done
python tools/ncu_digest.py $O/kan_small_fwd.ncu-rep $O/kan_small_tablegrad.ncu-rep $O/kan_small_records.ncu-rep $O/sum_f64.ncu-rep > $O/ncu_digest_small.jsonl 2>&1; rm -f $O/*.ncu-rep
head -c 4000 $O/ncu_digest_small.jsonl
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(json.dumps(d['supplementary']['kan_layers']))" 2>&1 | tail -3
