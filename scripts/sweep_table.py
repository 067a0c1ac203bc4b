"""Markdown table of the C3 (2PS-H vs OverL-H, N bands) and C5 (band height) sweeps from the bench JSON lines
saved by scripts/gpu_sweep_c3c5.sh, with the paper's coordination counters recomputed from the same plans.
usage: python scripts/sweep_table.py <dir with *_c3_*.json / *_c5_*.json>"""
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads as WL  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main(d):
    print("| config | mode | bands | images/s | ms/step | SM MHz | peak GB | Omega / feature maps | CI | OD rows | SD MB |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for cfg in ("c3", "c5"):
        rows = []
        for p in glob.glob(os.path.join(d, "*_%s_*.json" % cfg)):
            mode, n = os.path.basename(p).rsplit(".", 1)[0].split("_")[-2:]
            try:
                j = line(p)
            except Exception:
                continue
            rows.append((mode, int(n), j))
        for mode, n, j in sorted(rows, key=lambda r: (r[0], r[1])):
            if cfg == "c3":
                net, B, kw = WL.resnet50(H=224, W=224), 256, {"n_bands": n}
            else:
                net, B, kw = WL.vgg16(H=2048, W=2048, segments="pool"), 16, {"band_rows": n}
            flags = LB.FLAG_ALLOW_OVERLAP_EXHAUSTION | LB.FLAG_FP_MERGE
            cc = bench.coordination_counters(LB.Plan(net, B, mode=mode, prec="bf16", flags=flags, **kw))
            m = j["memory"]
            print("| %s | %s | %s %d | %.1f | %.2f | %s | %.2f | %.2fx | %d | %d | %.0f |" % (
                cfg.upper(), "2PS-H" if mode == "2ps" else "OverL-H", "N =" if cfg == "c3" else "rows", n,
                j["value"], j["ms_per_step"], j["clocks"]["sm_mhz"], m["peak_allocated_bytes"] / 1e9,
                m["reduction_vs_omega_x"], cc["computation_interruptions"], cc["overlapped_rows"],
                cc["sharing_data_bytes"] / 1e6))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/sweep")
