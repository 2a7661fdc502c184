"""Summarise an ncu source page (SASS): instruction mix and top stall sites.
ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv; python tools/sass_hot.py X.csv"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, ei = h.index('Address'), h.index('Source'), h.index('Instructions Executed')
st = h.index('Warp Stall Sampling (All Samples)')
data = [(r[ai], r[si].strip(), int(r[ei] or 0), int(r[st] or 0)) for r in rows[2:] if len(r) > ei]
tot = sum(d[2] for d in data)
tots = sum(d[3] for d in data)
print('total inst', tot, 'stall samples', tots)
c, cs = Counter(), Counter()
for a, s, e, smp in data:
    op = s.split()[0] if not s.startswith('@') else s.split()[1]
    c[op.split('.')[0]] += e
    cs[op.split('.')[0]] += smp
for op, n in c.most_common(14):
    print(f'{op:10s} {n:12d} {n / tot * 100:5.1f}%  stall {cs[op] / tots * 100:5.1f}%')
print('--- top stall sites')
for a, s, e, smp in sorted(data, key=lambda d: -d[3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(a[-5:], f'{s[:58]:58s}', e, smp)
