"""Per-role instruction counts of a warp-specialised kernel from the ncu SASS source page: the
regions between consecutive mbarrier waits / named barriers are printed with their executed
warp-instructions (per unit given by argv[2]) and top opcodes."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
unit = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot = sum(int(d["Instructions Executed"] or 0) for d in data)
print("total warp-instr %d, per unit %.0f" % (tot, tot / unit))
cur, n, ops, smp = None, 0, {}, 0
def flush():
    if cur is not None and n:
        top = ", ".join("%s %d" % (k, v / unit) for k, v in sorted(ops.items(), key=lambda x: -x[1])[:8])
        print("%s  %7.0f  samples %5d  %s" % (cur, n / unit, smp, top))
for d in data:
    src = d["Source"].strip()
    if "TRYWAIT" in src or "BAR.SYNC" in src:
        flush()
        cur, n, ops, smp = d["Address"][-5:] + " " + src[:48], 0, {}, 0
    e = int(d["Instructions Executed"] or 0)
    n += e
    smp += int(d["Warp Stall Sampling (All Samples)"] or 0)
    tok = src.split()
    op = (tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")).split(".")[0]
    ops[op] = ops.get(op, 0) + e
flush()
