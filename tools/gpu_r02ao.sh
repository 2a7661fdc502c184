#!/bin/bash
# compute-sanitizer over the round-2 kernels (tc3 TMA sweep, pre-split table GEMM, dense UKAN, small-layer cluster kernel)
O=gpurun_out/ao; mkdir -p $O
timeout 300 python tools/sanitize_probe.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -1 $O/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 $O/sanitize_$tool.log
done
