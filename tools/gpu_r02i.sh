#!/bin/bash
O=gpurun_out/i; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_train_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
UKAN_DX_WARPS=16 timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx >> $O/kb.jsonl 2>&1
timeout 300 python tools/kbench.py 8192 784 256 32 3 >> $O/kb.jsonl 2>&1
timeout 300 python tools/kbench.py 16384 1024 1024 32 3 dx >> $O/kb.jsonl 2>&1
cat $O/kb.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg3_tc2 -f python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg2_tc2 -f python tools/kbench.py 8192 784 256 32 3 > /dev/null 2>&1
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null
rm -f $O/*.ncu-rep
