"""Summarise an ncu --csv launch list: total time per kernel name (share of the listed launches)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    v = {"ns": v / 1000.0, "nsecond": v / 1000.0, "us": v, "usecond": v, "ms": v * 1000.0,
         "msecond": v * 1000.0}.get(unit, v)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print("total %.1f us over %d launches" % (T, sum(cnt.values())))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print("%8.1f us %5.1f%% %5d  %s" % (v, 100 * v / T, cnt[k], k))
