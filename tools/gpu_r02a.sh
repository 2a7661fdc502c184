#!/bin/bash
# round-2 baseline: GPU tests + cfg3 timings with dx + launch list of the cfg3 layer
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
free -g >> gpurun_out/a_smi.txt; nproc >> gpurun_out/a_smi.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/a_pytest.log
tail -3 gpurun_out/a_pytest.log
for shp in "65536 4096 4096 64 3 dx" "16384 4096 4096 64 3 dx" "8192 784 256 32 3"; do
  timeout 300 python tools/kbench.py $shp >> gpurun_out/a_kb.jsonl 2>&1
done
cat gpurun_out/a_kb.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_launch_cfg3.csv python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/a_launch_cfg3.csv 2>&1 | head -30
