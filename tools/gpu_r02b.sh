#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_bench_shapes.py tests/test_dp_trainer_gpu.py tests/test_cg_tc.py tests/test_train_gpu.py -q -s -m gpu -rA --durations=15 > gpurun_out/b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest.log
tail -40 gpurun_out/b_pytest.log
