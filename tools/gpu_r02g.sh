#!/bin/bash
# tc2 sweep v2 (LDS.128 B operand, two groups in flight) + dx 16 vs 32 warps: parity and timing
mkdir -p gpurun_out/g
O=gpurun_out/g
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_train_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
for w in 32 16; do
  UKAN_DX_WARPS=$w timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx >> $O/kb.jsonl 2>&1
done
timeout 300 python tools/kbench.py 8192 784 256 32 3 >> $O/kb.jsonl 2>&1
cat $O/kb.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch.csv python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
python tools/launch_summary.py $O/launch.csv | head -6
for k in kan_dx_tc kan_bwd_tc2_sweep; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/cfg3_$k -f python tools/kbench.py 16384 4096 4096 64 3 dx > $O/ncu_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg2_tc2 -f python tools/kbench.py 8192 784 256 32 3 > $O/ncu_cfg2.log 2>&1
ls $O
