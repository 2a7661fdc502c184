"""Per-kernel SASS opcode counts of the shipped library (tensor-core / TMA / TMEM / DMMA evidence):
python tools/sass_summary.py > profiles/r02/sass_summary.json"""
import collections
import json
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2408_11200_b200/libukan_b200.so"
KEYS = ("UTCHMMA", "UTCQMMA", "UTMALDG", "UBLKCP", "LDTM", "STTM", "DMMA", "HMMA", "FFMA2", "FFMA", "DFMA", "F2F",
        "LDS", "LDG", "STG", "STS", "LDGSTS", "SYNCS", "UCGABAR_ARV", "UCGABAR_WAIT")
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
demangled = subprocess.run(["c++filt"], input=sass, capture_output=True, text=True).stdout
out, cur, cnt = {}, None, collections.Counter()
for line in demangled.splitlines():
    m = re.match(r"\s+Function : (.*)", line)
    if m:
        if cur:
            out[cur] = {k: cnt[k] for k in KEYS if cnt[k]}
        cur, cnt = m.group(1)[:110], collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P[0-9T]\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        cnt[op] += 1
        if op.startswith("SYNCS"):
            cnt["SYNCS"] += 1
if cur:
    out[cur] = {k: cnt[k] for k in KEYS if cnt[k]}
json.dump(out, sys.stdout, indent=1)
