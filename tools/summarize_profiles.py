"""Summarise gpurun_out captures into profiles/ (tracked): launch-list shares and the key
ncu --set full metrics of each captured kernel.

python tools/summarize_profiles.py TAG   (reads gpurun_out/launches_TAG.csv, prof_bench_TAG.ncu-rep)
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)


def read_csv_log(path):
    lines = open(path).read().splitlines()
    start = [n for n, l in enumerate(lines) if l.startswith('"ID"')][0]
    return list(csv.reader(lines[start:]))


launches = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(launches):
    rows = read_csv_log(launches)
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi:
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
            agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    summ = sorted(({"kernel": k, "launches": len(v), "total_us": round(sum(v), 1),
                    "median_us": round(sorted(v)[len(v) // 2], 1), "share": round(sum(v) / tot, 4)}
                   for k, v in agg.items()), key=lambda d: -d["total_us"])
    with open(os.path.join(out, f"launches_{tag}.json"), "w") as f:
        json.dump({"source": f"ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py "
                             f"--steps 3 --warmup 3 (cold-cache, serialised; compare shares)", "kernels": summ}, f,
                  indent=1)
    print(json.dumps(summ[:12], indent=1))

rep = os.path.join(ROOT, "gpurun_out", f"prof_bench_{tag}.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
            "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size"]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:90]}
        for w in want:
            if w in h:
                d[w] = r[h.index(w)] + (" " + units[h.index(w)] if units[h.index(w)] else "")
        res.append(d)
    with open(os.path.join(out, f"ncu_full_{tag}.json"), "w") as f:
        json.dump({"source": "ncu --set full --clock-control none --import-source on, inside python bench.py "
                             "(KAN [784,256,10] B=8192 training step), layer-0 kernels", "kernels": res}, f, indent=1)
    print(json.dumps(res, indent=1))

    # per-launch DRAM traffic of the dominant kernel groups (bench.py's roofline.traffic)
    def _bytes(d, key):
        v, _, unit = d.get(key, "0 byte").partition(" ")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit.strip(), 1)
        return float(v.replace(",", "")) * mult

    def _us(d):
        v, _, unit = d.get("gpu__time_duration.sum", "0 us").partition(" ")
        return float(v.replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                            "msecond": 1e3}.get(unit.strip(), 1.0)

    def _group(names):
        picked = {}
        for d in res:
            for n in names:
                if n in d["kernel"] and (n not in picked or _us(d) > _us(picked[n])):
                    picked[n] = d
        if len(picked) < len(names):
            return None
        return {"kernels": [picked[n]["kernel"] for n in names],
                "dram_bytes": sum(_bytes(picked[n], "dram__bytes_read.sum") + _bytes(picked[n], "dram__bytes_write.sum")
                                  for n in names)}

    traffic = {"source": f"profiles/ncu_full_{tag}.json (ncu --set full, one launch per kernel, largest of each name)",
               "layer0.kan_backward": _group(["kan_bwd_tc_prep_kernel", "kan_bwd_tc2_sweep_kernel"]),
               "layer0.kan_backward_sweep": _group(["kan_bwd_tc2_sweep_kernel"]),
               "layer0.kan_forward": _group(["kan_pack_coeffs_kernel", "kan_fwd_records_kernel", "kan_fwd_tm_kernel"])}
    with open(os.path.join(out, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print(json.dumps(traffic, indent=1))
