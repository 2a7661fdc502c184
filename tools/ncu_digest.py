"""Small JSON digest of an .ncu-rep (so the GPU box can ship results without the 10 MB reports):
key metrics (tools/ncu_summary.py KEYS), warp-stall ratios, and the top SASS lines by stall
samples.  python tools/ncu_digest.py REP [REP ...] > digest.jsonl"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import KEYS  # noqa: E402


def digest(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return {"rep": rep, "error": "no data"}
    h, units, v = rows[0], rows[1], rows[2]
    d = {"rep": rep.rsplit("/", 1)[-1], "kernel": v[h.index("Kernel Name")][:120]}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for k, name in KEYS.items():
        if k in h:
            try:
                d[name] = float(v[h.index(k)].replace(",", ""))
            except ValueError:
                d[name] = v[h.index(k)]
            u = units[h.index(k)]
            if name == "duration":
                d["duration_unit"] = u
            elif name.startswith("dram_") and isinstance(d[name], float):
                d[name] = d[name] * scale.get(u, 1.0)  # bytes
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                val = float(v[i])
            except ValueError:
                continue
            if val >= 0.05:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(val, 3)
    d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hdr = next((i for i, r in enumerate(srows[:5]) if "Warp Stall Sampling (All Samples)" in r), None)
    if hdr is not None:
        sh = srows[hdr]
        si, sc = sh.index("Warp Stall Sampling (All Samples)"), sh.index("Source")
        data = [r for r in srows[hdr + 1:] if len(r) > si and r[si].isdigit()]
        tot = sum(int(r[si]) for r in data) or 1
        top = sorted(data, key=lambda r: -int(r[si]))[:20]
        d["top_sass_stalls"] = [[round(100.0 * int(r[si]) / tot, 2), r[sc].strip()[:80]] for r in top]
        ops = {}
        for r in data:
            parts = r[sc].split()
            if not parts:
                continue
            op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + int(r[si])
        d["stall_share_by_opcode"] = {k: round(100.0 * c / tot, 1) for k, c in sorted(ops.items(), key=lambda kv: -kv[1])[:12]}
    return d


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(json.dumps(digest(rep)))
