"""stdin: ncu --csv metrics output -> one line per kernel name: mean of each metric (GB / ms)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
hdr = rows[0]
agg = defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    d = dict(zip(hdr, r))
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    key = d["Kernel Name"][:48] + " grid=" + d.get("Grid Size", "")
    agg[key][d["Metric Name"]].append(v)
for k, m in agg.items():
    parts = []
    for name, vs in sorted(m.items()):
        mean = sum(vs) / len(vs)
        parts.append(f"{name.split('__')[1]}={mean / 1e9:.3f}G" if "bytes" in name else f"{name.split('__')[1]}={mean / 1e6:.3f}ms")
    print(k, len(next(iter(m.values()))), " ".join(parts))
