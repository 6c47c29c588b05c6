"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) of
scripts/wcycle_launches.py: the second of its two cycles, per kernel and
launch shape (dev tool).  python scripts/launch_summary.py <csv> [top]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
gi, bi = h.index("Grid Size"), h.index("Block Size")
L = [(r[ki], r[gi] + " x " + r[bi], float(r[vi].replace(",", ""))) for r in rows[1:]]
half = L[len(L) // 2:]
t = defaultdict(lambda: [0, 0.0])
for k, g, v in half:
    key = (k.split("(")[0][:48], g)
    t[key][0] += 1
    t[key][1] += v
print(f"| kernel | grid x block | launches | total ms | us/launch |\n|---|---|---|---|---|")
for (k, g), (n, s) in sorted(t.items(), key=lambda x: -x[1][1])[:top]:
    print(f"| `{k}` | {g} | {n} | {s / 1e6:.3f} | {s / n / 1e3:.1f} |")
print(f"\ncycle total: {sum(v[1] for v in t.values()) / 1e6:.2f} ms in {len(half)} launches")
