#!/bin/bash
O=gpurun_out/s; mkdir -p $O
timeout 1200 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_train_gpu.py tests/test_dp_trainer_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; tail -c 700 $O/bench_ref.json
for sh in "16384 4096 4096 64 3 dx" "8192 784 256 32 3" "8192 256 10 32 3 dx" "16384 1024 1024 32 3 dx"; do timeout 300 python tools/kbench.py $sh >> $O/kb.jsonl 2>&1; done
cat $O/kb.jsonl | cut -c1-240
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_probe.py > $O/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 $O/racecheck.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg3_tc2 -f python tools/kbench.py 16384 4096 4096 64 3 > /dev/null 2>&1
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2>/dev/null; rm -f $O/*.ncu-rep
