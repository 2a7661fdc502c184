#!/bin/bash
# tc2 v2 + dx warp variants: parity + timing; then evidence (bench, launch lists, ncu digests)
O=gpurun_out/h; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_bench_shapes.py tests/test_parity_kan.py tests/test_train_gpu.py -q -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for w in 32 16; do UKAN_DX_WARPS=$w timeout 300 python tools/kbench.py 16384 4096 4096 64 3 dx >> $O/kb.jsonl 2>&1; done
timeout 300 python tools/kbench.py 8192 784 256 32 3 >> $O/kb.jsonl 2>&1
cat $O/kb.jsonl
# pick the faster dx variant for the rest of the run
W=$(python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/h/kb.jsonl") if l.startswith("{")]
a=[r for r in rows if r["shape"][1]==4096]
print(32 if len(a)<2 or a[0]["bwd_ms"]<=a[1]["bwd_ms"] else 16)
PY
)
echo "dx warps: $W"; export UKAN_DX_WARPS=$W
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 400 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_cfg3.csv python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/launch_cfg3.csv > $O/launch_cfg3.txt 2>&1; head -8 $O/launch_cfg3.txt
for k in kan_dx_tc kan_bwd_tc2_sweep kan_fwd_tm_kernel kan_bwd_tc_prep kan_pack_coeffs kan_fwd_records; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/cfg3_$k -f python tools/kbench.py 16384 4096 4096 64 3 dx > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_bwd_tc2 -c 1 -o $O/cfg2_tc2 -f python tools/kbench.py 8192 784 256 32 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kan_fwd_tm -c 1 -o $O/cfg2_fwd -f python tools/kbench.py 8192 784 256 32 3 > /dev/null 2>&1
for k in seg_fsweep spline_fwd_kernel spline_dx64 cg_gemm_tc cg_dmma_gemm seg_fsort seg_prep keys_insert; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/uk_$k -f python tools/ukbench.py 4096 1024 1024 0.5 32 32 > /dev/null 2>&1
done
python tools/ncu_digest.py $O/*.ncu-rep > $O/ncu_digest.jsonl 2> $O/ncu_digest.err
wc -l $O/ncu_digest.jsonl
# traffic per launch group for the bench's roofline field
python - <<'PY'
import json
d=[json.loads(l) for l in open("gpurun_out/h/ncu_digest.jsonl")]
out={}
for r in d:
    n=r["rep"].replace(".ncu-rep","")
    if n.startswith("cfg3_"):
        key={"cfg3_kan_dx_tc":"cfg3.backward_dx","cfg3_kan_bwd_tc2_sweep":"cfg3.backward_table_bucket_at_B16384","cfg3_kan_fwd_tm_kernel":"cfg3.forward_main"}.get(n)
        if key and isinstance(r.get("dram_read"),float):
            out[key]={"dram_bytes_B16384": r["dram_read"]+r["dram_write"], "unit_note":"ncu dram__bytes (see digest units)", "duration": r["duration"]}
json.dump(out, open("gpurun_out/h/traffic_probe.json","w"), indent=1)
PY
mkdir -p $O/keep; mv $O/cfg3_kan_dx_tc.ncu-rep $O/cfg3_kan_bwd_tc2_sweep.ncu-rep $O/keep/ 2>/dev/null
rm -f $O/*.ncu-rep
du -sh $O
