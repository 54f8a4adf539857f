"""Per-kernel shares of the timed C2 step from an ncu launch list (dev aid):
python scripts/launch_shares.py profiles/r02_launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
t = defaultdict(list)
for r in rows[1:]:
    if len(r) == len(h) and r[im] == "gpu__time_duration.sum" and "supra::" in r[ik]:
        t[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")))
n = max(len(v) for v in t.values())
tot = sum(sum(v) for v in t.values()) / n
print("Product kernels of the timed C2 step (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised),")
print(f"from {sys.argv[1]} ({n} steps):")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {k:45s} launches {len(v):3d}  {sum(v) / len(v) / 1000 if max(v) > 1e4 else sum(v) / len(v):9.1f} us/launch  share {sum(v) / n / tot * 100:5.1f} %")
print(f"  step total {tot / 1000 if tot > 1e5 else tot:.1f} us (ncu); live bench step: see r02_bench.json ms_per_step")
