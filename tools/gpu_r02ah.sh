#!/bin/bash
# table GEMM tile width A/B (UKAN_CG_BN): UKAN layer timing + kernel durations
O=gpurun_out/ah; mkdir -p $O
for bn in 0 64 128 0 64 128; do
  UKAN_CG_BN=$bn timeout 300 python tools/ukbench.py 4096 1024 1024 0.5 32 32 | sed "s|^|BN=$bn |" >> $O/kb.txt 2>&1
done
cut -c1-250 $O/kb.txt
for bn in 0 64 128; do
  UKAN_CG_BN=$bn timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cg_gemm_tc -c 3 --csv --log-file $O/tc_$bn.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
  echo "BN=$bn"; grep -h "gpu__time" $O/tc_$bn.csv | awk -F'","' '{print $NF}'
done
