#!/bin/bash
# small-layer path (kan_small.cu): parity tests, A/B vs the tiled kernels, cfg1 launch list, bench
O=gpurun_out/y; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_kan.py tests/test_dp_trainer_gpu.py tests/test_parity_bench_shapes.py tests/test_train_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1
tail -5 $O/pytest.txt
for e in "X=0" "UKAN_SMALL=0"; do
  for s in "1024 64 64 10 3" "513 128 128 20 3" "8192 64 64 10 3" "65536 64 64 10 3"; do
    env $e timeout 120 python tools/kbench.py $s | sed "s/^/$e $s /" >> $O/kb.txt 2>&1
  done
done
cut -c1-250 $O/kb.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg1.csv python tools/cfg1_probe.py 3 > /dev/null 2>&1
python tools/ncu_summary.py $O/launch_cfg1.csv 2>&1 | head -20
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 3000 $O/bench.json
