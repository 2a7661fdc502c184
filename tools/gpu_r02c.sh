#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_cg_tc.py tests/test_parity_ukan.py tests/test_train_gpu.py tests/test_dp_trainer_gpu.py tests/test_tangent_gpu.py -q -m gpu -k "cfg3 or multichunk or degrees or base or precision or deterministic or ukan or trainer" > gpurun_out/c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c_pytest.log
tail -5 gpurun_out/c_pytest.log
for shp in "65536 4096 4096 64 3 dx" "16384 4096 4096 64 3 dx" "16384 1024 1024 32 3 dx"; do
  timeout 300 python tools/kbench.py $shp >> gpurun_out/c_kb.jsonl 2>&1
  UKAN_DX=simt timeout 300 python tools/kbench.py $shp >> gpurun_out/c_kb.jsonl 2>&1
done
cat gpurun_out/c_kb.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launch_cfg3.csv python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c_launch_cfg3.csv 2>&1 | head -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_dx_tc -s 1 -c 1 -o gpurun_out/prof_dx_c -f python tools/kbench.py 16384 4096 4096 64 3 dx > gpurun_out/c_ncu.log 2>&1
tail -2 gpurun_out/c_ncu.log
