#!/bin/bash
O=gpurun_out/v; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_ukan.py tests/test_parity_bench_shapes.py tests/test_tangent_gpu.py -q -m gpu -x -k "ukan" > $O/pytest.log 2>&1; echo "rc=$?"; tail -1 $O/pytest.log
timeout 300 python tools/ukbench.py 4096 1024 1024 0.5 32 32 > $O/uk.json 2>&1; cat $O/uk.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_ukan.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
python tools/launch_summary.py $O/launch_ukan.csv 2>/dev/null | head -6
