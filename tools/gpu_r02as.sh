#!/bin/bash
# dense UKAN forward on the TMEM gather: parity + cfg5 A/B
O=gpurun_out/as; mkdir -p $O
timeout 1500 python -m pytest tests/test_parity_ukan.py tests/test_dp_trainer_gpu.py tests/test_train_gpu.py tests/test_compat_gpu.py -x -q -m gpu > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.txt | cut -c1-300
for e in "UKAN_FWD=smem" "X=1" "UKAN_FWD=smem" "X=1"; do
  env $e timeout 600 python -c "
import bench, torch, json; r = bench.cfg5_rate(torch.device('cuda', 0), 1, 0); print(json.dumps({'ms': r['ms_per_step'], 'sps': r['samples_per_s']}))" 2>&1 | tail -1 | sed "s|^|$e |" >> $O/cfg5.txt
done
cat $O/cfg5.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg5.csv python tools/cfg5_probe.py 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg5.csv > $O/launch_cfg5.txt 2>&1; head -12 $O/launch_cfg5.txt
