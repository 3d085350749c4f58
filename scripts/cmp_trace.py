"""Compare two DPK_SPD_TRACE logs by GEMM shape (per-call totals)."""
import collections
import re
import sys


def load(path):
    rows = []
    for l in open(path):
        m = re.match(r'\s*(\d+)\s+(\d+)\(\s*(\d+)\)\s+([\d.]+)\s+(\d+)\s+([\d.]+)\s+([\d.]+)\s+([\d.]+)\s+(\S+)', l)
        if m:
            rows.append(m.groups())
    calls = max(1, sum(1 for g in rows if g[0] == '0'))
    by = collections.defaultdict(float)
    leaf = 0.0
    for g in rows:
        leaf += float(g[3])
        if int(g[4]) > 0:
            by[g[8]] += float(g[5])
    return {k: v / calls for k, v in by.items()}, leaf / calls


a, la = load(sys.argv[1])
b, lb = load(sys.argv[2])
print(f"leaves {la:.0f} vs {lb:.0f} us; gemms {sum(a.values()):.0f} vs {sum(b.values()):.0f} us")
for k in sorted(set(a) | set(b), key=lambda k: -max(a.get(k, 0), b.get(k, 0)))[:30]:
    print(f"{k:20s} {a.get(k, 0):8.1f} {b.get(k, 0):8.1f}")
