"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
# several captured launches: keep the first kernel's block (up to the next "Kernel Name" line)
end = next((i for i in range(2, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
data = [dict(zip(hdr, r)) for r in rows[2:end] if len(r) == len(hdr)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(int(d[h] or 0) for d in data) for h in stall_cols}
print("total samples", tot)
print("by reason:", ", ".join("%s %.1f%%" % (k[6:], 100.0 * v / max(tot, 1)) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for d in top:
    n = int(d["Warp Stall Sampling (All Samples)"] or 0)
    why = sorted(((int(d[h] or 0), h[6:]) for h in stall_cols), reverse=True)[:2]
    print("%5.1f%% %s %-60s %s" % (100.0 * n / max(tot, 1), d["Address"][-5:], d["Source"].strip()[:60], why))
