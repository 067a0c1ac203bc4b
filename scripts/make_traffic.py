"""profiles/traffic.json from `ncu --set full` raw CSV exports: DRAM bytes (read + write) per launch
of each captured kernel, averaged per kernel name (bench.py reports it as roofline.traffic).
usage: python scripts/make_traffic.py out.json capture1.raw.csv [capture2.raw.csv ...]"""
import csv
import json
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name):
    n = re.sub(r"\(CUtensorMap.*$|\(PoolArgs.*$|\(EltArgs.*$", "", name).replace("void ", "").strip()
    return n.replace("lrcnn::", "").replace("(int)", "")


per, launches = {}, []
for path in sys.argv[2:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        def val(k):
            i = ix.get(k)
            return float(r[i]) * UNIT.get(units[i], 1.0) if i is not None and r[i] else 0.0
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        k = short(r[ix["Kernel Name"]])
        launches.append({"kernel": k, "dram_bytes": b, "duration_us": val("gpu__time_duration.sum") / 1e3
                         if units[ix["gpu__time_duration.sum"]] == "nsecond" else val("gpu__time_duration.sum"),
                         "tensor_active_pct": val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")})
        per.setdefault(k, []).append(b)
out = {"per_kernel": {k: sum(v) / len(v) for k, v in per.items()}, "launches": launches,
       "source": [p.split("/")[-1] for p in sys.argv[2:]]}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out["per_kernel"], indent=1))
