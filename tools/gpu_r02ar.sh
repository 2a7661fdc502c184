#!/bin/bash
# dx kernel after making the UKAN segment support compile-time: A/B against the pre-dense library
O=gpurun_out/ar; mkdir -p $O
for L in abtmp/lib_old.so paper_2408_11200_b200/libukan_b200.so abtmp/lib_old.so paper_2408_11200_b200/libukan_b200.so; do
  UKAN_B200_LIB=$L timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx | sed "s|^|$L |" | cut -c1-260
done
timeout 900 python -m pytest tests/test_parity_ukan.py tests/test_parity_bench_shapes.py -x -q -m gpu 2>&1 | tail -1
