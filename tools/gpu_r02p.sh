#!/bin/bash
O=gpurun_out/p; mkdir -p $O
timeout 1200 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_train_gpu.py tests/test_dp_trainer_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for s in "16384 4096 4096 64 3 dx" "8192 784 256 32 3" "8192 256 10 32 3 dx"; do timeout 300 python tools/kbench.py $s >> $O/kb.jsonl 2>&1; done
cat $O/kb.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch.csv python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
python tools/launch_summary.py $O/launch.csv 2>/dev/null | head -5
