"""Summarise an ncu --metrics gpu__time_duration.sum,dram__bytes_* launch-list CSV per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per, name = collections.defaultdict(dict), {}
for r in data:
    per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    n = r[ki].split("(")[0]
    name[r[idi]] = n.split("::")[-1]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[name[i]]
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"]
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:36s} n={a[0]:5d} ms={a[1] / 1e6:8.2f} share={a[1] / tot:.3f} avg_us={a[1] / a[0] / 1e3:7.2f} "
          f"GB/s={a[2] / a[1]:8.1f}")
print("total ms", round(tot / 1e6, 3))
if len(sys.argv) > 3:
    ids = sorted(per, key=int)
    for i in ids[int(sys.argv[2]):int(sys.argv[3])]:
        m = per[i]
        print(i, name[i], round(m["gpu__time_duration.sum"] / 1e3, 2),
              round((m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6, 2))
