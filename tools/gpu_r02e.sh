#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py -q -m gpu -x > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
tail -5 gpurun_out/e_pytest.log
timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx >> gpurun_out/e_kb.jsonl 2>&1
cat gpurun_out/e_kb.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kan_dx_tc|kan_bwd_tc2_sweep|kan_fwd_tm_kernel" -s 3 -c 3 -o gpurun_out/prof_e -f python tools/kbench.py 16384 4096 4096 64 3 dx > gpurun_out/e_ncu.log 2>&1
tail -2 gpurun_out/e_ncu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/e_bench.json; tail -5 gpurun_out/e_bench.err
