#!/bin/bash
# round-2 evidence run: tensor peaks, full bench, launch lists, per-kernel ncu, sanitizers
mkdir -p gpurun_out/f
O=gpurun_out/f
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_peak tools/tf32_peak.cu && ./tools/tf32_peak > $O/tf32_peak.json 2>&1
cat $O/tf32_peak.json
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 600 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg3.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg3.csv | head -12
for k in kan_dx_tc kan_bwd_tc2_sweep kan_fwd_tm_kernel kan_bwd_tc_prep kan_pack_coeffs kan_fwd_records; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/cfg3_$k -f python tools/kbench.py 16384 4096 4096 64 3 dx > $O/ncu_$k.log 2>&1
done
for k in seg_fsweep spline_fwd_kernel spline_dx64 cg_gemm_tc cg_dmma_gemm seg_fsort seg_prep keys_ ukan; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/uk_$k -f python tools/ukbench.py 4096 1024 1024 0.5 32 32 > $O/ncu_uk_$k.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_ukan.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
python tools/launch_summary.py $O/launch_ukan.csv | head -20
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 $O/sanitize_$tool.log
done
ls $O
