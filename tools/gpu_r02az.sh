#!/bin/bash
# UKAN dx on the per-feature sorted order: parity + UKAN layer A/B
O=gpurun_out/az; mkdir -p $O
timeout 1500 python -m pytest tests/test_parity_ukan.py tests/test_parity_bench_shapes.py tests/test_dp_trainer_gpu.py tests/test_train_gpu.py tests/test_compat_gpu.py tests/test_tangent_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-300
for e in "UKAN_DX_SORTED=0" "X=1" "UKAN_DX_SORTED=0" "X=1"; do
  env $e timeout 300 python tools/ukbench.py 4096 1024 1024 0.5 32 32 | sed "s|^|$e |" | cut -c1-220
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg_dx_sorted|spline_dx64" -c 4 --csv --log-file $O/dx.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
grep -h "gpu__time" $O/dx.csv | awk -F'","' '{print $5, $NF}' | cut -c1-100
