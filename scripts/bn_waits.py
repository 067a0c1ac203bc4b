"""Which mbarrier waits spin in k_bneck_fwd (ncu source page, SASS): samples and retry-loop executions
per barrier, named from the kernel's barrier layout (offset of the barrier block given as argv[2])."""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = int(sys.argv[2], 16)
names = ["wbar", "tfull0", "tfull1", "tfull2", "tempty0", "tempty1", "tempty2", "a1full0", "a1full1", "a1empty0",
         "a1empty1", "t1full", "t1empty", "a2full", "t2full", "t2empty", "a3full", "a3empty", "rbar0", "rbar1", "rbar2", "rbar3"]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
for i, d in enumerate(data):
    if "TRYWAIT" not in d["Source"]:
        continue
    m = re.search(r"\+0x([0-9a-f]+)\]", d["Source"])
    off = int(m.group(1), 16) if m else -1
    k = (off - base) // 8
    nm = names[k] if 0 <= k < len(names) else hex(off)
    smp = sum(int(data[j]["Warp Stall Sampling (All Samples)"] or 0) for j in range(i, min(i + 3, len(data))))
    print("%s %-9s samples %5d (%4.1f%%) executed %s" % (d["Address"][-5:], nm, smp, 100.0 * smp / max(tot, 1),
                                                        d["Instructions Executed"]))
