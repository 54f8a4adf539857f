"""Static SASS check: instruction mix between consecutive MUFU.RSQ (one per DAS tile body)."""
import re, subprocess, sys
from collections import Counter
so, fn = sys.argv[1], sys.argv[2]
out = subprocess.check_output(["cuobjdump", "-sass", "-fun", fn, so], stderr=subprocess.DEVNULL).decode()
ops = []
for line in out.splitlines():
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m: ops.append(m.group(2))
idx = [i for i, o in enumerate(ops) if o == "MUFU.RSQ"]
lens = [b - a for a, b in zip(idx, idx[1:])]
print("tile bodies:", len(idx), "median length", sorted(lens)[len(lens) // 2] if lens else None)
if len(idx) > 3:
    a, b = idx[2], idx[3]
    print(sorted(Counter(ops[a:b]).items(), key=lambda x: -x[1]))
