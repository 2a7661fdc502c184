#!/bin/bash
# final round-2 evidence: GPU tests, smoke, bench (ours + reference arm), launch lists, ncu of the
# dominant kernels inside the bench process at the bench shape, sanitizers
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 300 $O/bench.json
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; tail -c 600 $O/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg3.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg3.csv > $O/launch_cfg3.txt 2>&1; head -8 $O/launch_cfg3.txt
for k in kan_dx_tc kan_bwd_tc2_sweep kan_fwd_tm_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/bench_$k -f python bench.py --steps 1 --warmup 0 --no-configs --no-cpu-baseline > /dev/null 2>&1
done
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null; wc -l $O/ncu_digest.jsonl
rm -f $O/*.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_ukan.csv python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
python tools/launch_summary.py $O/launch_ukan.csv > $O/launch_ukan.txt 2>&1; head -12 $O/launch_ukan.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 $O/sanitize_$tool.log
done
du -sh $O
