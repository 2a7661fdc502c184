#!/bin/bash
# UKAN backward with the max_rows hint: parity + cfg4 full (B = 65536) timing
O=gpurun_out/ax; mkdir -p $O
timeout 1500 python -m pytest tests/test_parity_ukan.py tests/test_parity_bench_shapes.py tests/test_dp_trainer_gpu.py tests/test_train_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-300
timeout 900 python -c "
import bench, torch, json; r = bench.cfg4_rate(torch.device('cuda', 0)); print(json.dumps({'ms': r['ms_per_step'], 'sps': r['samples_per_s'], 'n_u': r.get('n_u')}))" 2>&1 | tail -1
timeout 600 python tools/ukbench.py 4096 1024 1024 0.5 32 32 | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg4.csv python -c "
import bench, torch, json; r = bench.cfg4_rate(torch.device('cuda', 0), steps=1, warmup=1); print(json.dumps(r['ms_per_step']))" > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg4.csv > $O/launch_cfg4.txt 2>&1; head -8 $O/launch_cfg4.txt
