"""Quick look at an ncu --set full capture: key counters, SASS opcode mix and
the hottest instructions (stall samples).  python tools/ncu_brief.py rep [kernel-regex] [ntop]"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles"))
from summarize import full  # noqa: E402

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 25
print(full(rep)[0])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hi = his[0]
hdr = rows[hi]
data = rows[hi + 1:his[1] - 1] if len(his) > 1 else rows[hi + 1:]  # first kernel in the capture
ix = {h: i for i, h in enumerate(hdr)}
ie, isamp, ath = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"], ix["Avg. Threads Executed"]
f = lambda r, i: float(r[i] or 0) if len(r) > i else 0.0
tot = sum(f(r, ie) for r in data)
tsamp = sum(f(r, isamp) for r in data)
c, s = collections.Counter(), collections.Counter()
for r in data:
    if len(r) < 2 or not r[1]:
        continue
    parts = r[1].split()
    op = parts[1] if parts[0].startswith("@") else parts[0]
    op = op.split(".")[0]
    c[op] += f(r, ie)
    s[op] += f(r, isamp)
print(f"warp instructions {tot:.4g}  stall samples {tsamp:.0f}")
for op, v in c.most_common(22):
    print(f"  {op:10s} {100 * v / tot:6.2f}% inst   {100 * s[op] / max(tsamp, 1):6.2f}% samples")
print("hottest instructions:")
for r in sorted(data, key=lambda r: -f(r, isamp))[:ntop]:
    print(f"  {r[0][-5:]} {r[1][:58]:58s} samp {f(r, isamp):6.0f} exec {f(r, ie):9.0f} thr {f(r, ath):4.1f}")
