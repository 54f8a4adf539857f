"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass` (dev aid)."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = Counter()
for r in data:
    for k in stall_cols:
        agg[k] += int(r[ix[k]] or 0)
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {v/tot*100:.1f}%" for k, v in agg.most_common(12)))
# by opcode
op = Counter(); opn = Counter()
for r in data:
    o = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if o.startswith("@"): o = r[ix["Source"]].split()[1]
    op[o] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    opn[o] += int(r[ix["Instructions Executed"]] or 0)
print("by opcode (samples%, executed%):")
te = sum(opn.values())
for o, v in op.most_common(25):
    print(f"  {o:28s} {v/tot*100:5.1f}%  exec {opn[o]/te*100:5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top instructions:")
for r in sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:3]
    print(f"  {s/tot*100:5.2f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} {top}")
