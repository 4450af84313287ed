"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    d[r[ii]]["name"] = r[ki].split("(")[0]
    d[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k in sorted(d, key=int):
    v = d[k]
    a = agg[v["name"]]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0)
    a[2] += v.get("dram__bytes_read.sum", 0)
    a[3] += v.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    bw = (a[2] + a[3]) / (a[1] * 1e-9) / 1e12 if a[1] else 0
    print(f"{n[:42]:42s} n={a[0]:5d} t={a[1] / 1e6:9.3f}ms {100 * a[1] / tot:5.1f}%  rd={a[2] / 1e9:8.3f}GB wr={a[3] / 1e9:7.3f}GB {bw:5.2f}TB/s")
