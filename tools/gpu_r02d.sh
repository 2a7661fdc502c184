#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_compat_gpu.py -q -m gpu -x > gpurun_out/d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d_pytest.log
tail -25 gpurun_out/d_pytest.log
for shp in "16384 4096 4096 64 3 dx" "16384 1024 1024 32 3 dx"; do
  timeout 300 python tools/kbench.py $shp >> gpurun_out/d_kb.jsonl 2>&1
done
cat gpurun_out/d_kb.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_dx_tc -s 1 -c 1 -o gpurun_out/prof_dx_d -f python tools/kbench.py 16384 4096 4096 64 3 dx > gpurun_out/d_ncu.log 2>&1
tail -2 gpurun_out/d_ncu.log
