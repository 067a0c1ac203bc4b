"""Summarise a per-op profile CSV (bench.py --per-op-csv): time share and TFLOP/s per op/kind."""
import csv
import sys

rows = list(csv.DictReader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot = sum(float(r["ms"]) for r in rows)
print("total %.2f ms per step over %d entries" % (tot / steps, len(rows)))
for r in sorted(rows, key=lambda r: -float(r["ms"]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    ms = float(r["ms"]) / steps
    fl = float(r["flops"]) / steps
    tf = fl / (ms / 1000) / 1e12 if ms > 0 and fl > 0 else 0.0
    print("%3s %-10s k%s s%s %4s->%-4s %4sx%-4s  %7.3f ms %5.1f%%  %7.1f TF/s  n=%s" % (
        r["op"], r["kind"], r["k"], r["s"], r["c_in"], r["c_out"], r["h_out"], r["w_out"], ms, 100 * float(r["ms"]) / tot,
        tf, r["launches"]))
