"""Aggregate an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel name."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d, name = defaultdict(dict), {}
for r in rows:
    d[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    name[r[idi]] = r[ki].split("(")[0]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in d.items():
    a = agg[name[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{a[1] / 1e6:8.2f} ms {a[0]:5d} launches {a[2] / 1e9:8.2f} GB {a[2] / max(a[1], 1):7.1f} GB/s  {k}")
print("total ms", tot / 1e6)
