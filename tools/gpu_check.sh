#!/bin/bash
# One GPU round-trip: parity tests, smoke, bench, launch list + ncu captures of the bench command.
# Usage (from this container): gpurun --timeout 1800 -- bash tools/gpu_check.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
# every launch of a short bench run (cold-cache, serialised: compare shares, not absolutes)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ukan --no-configs > gpurun_out/ncu_bench_$TAG.log 2>&1
# full sections of the two layer-0 kernels inside the bench step
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kan_bwd_tc2_sweep|kan_bwd_tc_prep|kan_fwd_tm_kernel|kan_pack_coeffs|kan_fwd_records" -s 18 -c 6 \
  -o gpurun_out/prof_bench_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ukan --no-configs > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log gpurun_out/smoke_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
