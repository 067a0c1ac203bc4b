#!/usr/bin/env python
"""bench.py -- row-centric ResNet-50 training on climate-scale images on B200 (the north star).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]

One step = one lrcnn_step (Alg. 1 l.5-24: row-centric FP, head, row-centric BP with
recompute, SGD) over one batch of synthetic input.  Default workload C4 (BASELINE.json
configs[3], the north star): ResNet-50 v1.5 on 3600x2400x3 images, batch 8, bf16, 2PS-H
(2PS bands inside per-stage checkpoint segments), tcgen05 kernels only.  N>1: one process
per GPU (torchrun); the same batch's rows are split across the ranks (--parallel rows,
default: NCCL halo exchange at every segment input + GAP / wgrad all-reduce, strong
scaling); --parallel dp gives data-parallel replicas (weak scaling).  C2 / C3 / C5 are
selectable with --config.  Prints ONE JSON line (rank 0).  --impl reference times the fp64
CPU oracle (the reference arm of this tier) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as WL  # noqa: E402

METRIC = "train images/s (row-centric 2PS-H, bf16) + peak feature-map HBM vs layer-wise"
UNIT = "images/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4", "c5"],
                    help="BASELINE.json configs: c4 ResNet-50 3600x2400 B8 (default, the north star), c2 VGG-16 "
                         "224^2 B32, c3 ResNet-50 224^2 B256, c5 VGG-16 2048^2 B16")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--hw", type=int, default=0)
    ap.add_argument("--mode", default="2ps", choices=["2ps", "overl", "column"])
    ap.add_argument("--segments", default=None,
                    help="checkpoint segments (2PS-H): pool = after every pool (VGG) / stage (ResNet, the default); "
                         "none = whole-net 2PS; ResNet cut string, e.g. 3 = one checkpoint after conv3_x, p234 = "
                         "stage; block = after every bottleneck (the --bn-train default: 3 BN levels per segment)")
    ap.add_argument("--n-bands", type=int, default=None,
                    help="bands of the largest segment (default: 4; 8 for the climate-scale C4 / C5, where "
                         "it meets the north star's >= 5x feature-map reduction vs layer-wise)")
    ap.add_argument("--band-rows", type=int, default=0)
    ap.add_argument("--mem-budget-gb", type=float, default=0.0,
                    help="budget-driven planning: the smallest band count whose workspace fits (lrcnn_plan_budget)")
    ap.add_argument("--no-baselines", action="store_true", help="skip the layer-wise memory and cpu baselines")
    ap.add_argument("--no-eager", action="store_true", help="skip the PyTorch-eager layer-wise context run")
    ap.add_argument("--simt", action="store_true", help="disable the tcgen05 kernels (debug)")
    ap.add_argument("--allow-overlap", action="store_true",
                    help="OverL: accept N > H / o^0 at a segment input (LRCNN_FLAG_ALLOW_OVERLAP_EXHAUSTION)")
    ap.add_argument("--no-fuse-block", action="store_true",
                    help="run the conv2_x identity bottlenecks unfused (default: one fused kernel per band, "
                         "LRCNN_FLAG_NO_FUSE_BLOCK off)")
    ap.add_argument("--no-fp-merge", action="store_true",
                    help="forward pass on the BP bands (default: merged FP bands, LRCNN_FLAG_FP_MERGE)")
    ap.add_argument("--no-balanced", action="store_true",
                    help="same band count in every segment (default: balanced bands, LRCNN_FLAG_BALANCED_BANDS)")
    ap.add_argument("--bn-train", action="store_true",
                    help="ResNet with training-mode BatchNorm after every conv (SURVEY 8(f) f4: statistics / sums "
                         "sweeps per dependency level, DESIGN.md §5.2) instead of frozen-statistics affine")
    ap.add_argument("--per-op-csv", default="", help="write the per-op kernel profile (CSV) here")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group backend; gloo only to exercise the N>1 code path on one GPU")
    ap.add_argument("--zero-redundancy", action="store_true",
                    help="--parallel rows: zero-redundancy sharding (every row on one rank, halo from the rank "
                         "below after the first band; LRCNN_FLAG_ZERO_REDUNDANCY) instead of OverL at the cuts")
    ap.add_argument("--parallel", default="rows", choices=["dp", "rows"],
                    help="N>1: rows = the same batch row-sharded across ranks with NCCL halo exchange (default, "
                         "the north star's split, SURVEY 8(e)); dp = each rank its own batch, wgrad all-reduce")
    return ap.parse_args()


def demangle(name):
    """lrcnn::k_conv_tc2h<256> from the mangled kernel name cudaFuncGetName returns."""
    try:
        import subprocess
        out = subprocess.run(["c++filt", name], capture_output=True, text=True, timeout=5).stdout.strip()
        if out:
            name = out
    except Exception:
        pass
    name = name.split("(")[0].replace("lrcnn::", "").replace("(int)", "")
    return name[5:] if name.startswith("void ") else name


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, dev_index):
        super().__init__(daemon=True)
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def run(self):
        while self.nv is not None and not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def result(self):
        self.stop_ev.set()
        self.join(timeout=1)
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


CONFIGS = {   # (model, H, W, batch, description)
    "c2": ("vgg16", 224, 224, 32, "C2: VGG-16 conv stack 224x224x3"),
    "c3": ("resnet50", 224, 224, 256, "C3: ResNet-50 v1.5 224x224x3"),
    "c4": ("resnet50", 3600, 2400, 8, "C4: ResNet-50 v1.5 3600x2400x3 (climate-scale)"),
    "c5": ("vgg16", 2048, 2048, 16, "C5: VGG-16 conv stack 2048x2048x3"),
}


def make_net(a):
    if a.segments is None:
        a.segments = "block" if getattr(a, "bn_train", False) and CONFIGS[a.config][0] == "resnet50" else "pool"
    model, H, W, _, _ = CONFIGS[a.config]
    if a.hw:
        H = W = a.hw
    if model == "vgg16":
        return WL.vgg16(H=H, W=W, segments=a.segments if a.segments in ("pool", "none") else "pool")
    return WL.resnet50(H=H, W=W, segments="stage" if a.segments == "pool" else a.segments,
                       bn_train=getattr(a, "bn_train", False))


def cpu_baseline(a, steps=1):
    """The fp64 oracle (column dataflow, as it stands) on a bounded sample of the workload: one
    training step (FP, head, BP, SGD) on one image (C2 / C3) or on a full-width strip of one image
    (C4 / C5, images/s extrapolated by strip / H), on all host cores and on 1 thread (a smaller
    strip, so the default run stays within minutes)."""
    import oracle
    from oracle import column as C
    cores = os.cpu_count() or 1

    def run(threads, strip):
        oracle.set_threads(threads)
        net, scale, what = oracle_sample(a, strip)
        params = WL.make_params(net, seed=2)
        x = WL.make_input(net, 1, seed=0)
        lab = WL.make_labels(net, 1)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            params, loss, _, _, _ = C.step(net, params, x, lab, 0.01)
            times.append(time.perf_counter() - t0)
        return scale / statistics.mean(times), what
    v, what = run(cores, 224)
    v1, what1 = run(1, 32)
    oracle.set_threads(cores)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "%s, one fp64 column step (FP+head+BP+SGD), OpenMP over (b, c_out), mean of %d"
                      % (what, steps),
            "s_per_image": 1.0 / v,
            "one_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": what1}}


def oracle_sample(a, strip=224):
    """Bounded CPU sample of the workload: one full image for C2/C3; for the climate-scale
    configs one full-width strip of `strip` image rows (images/s extrapolated by strip/H)."""
    net = make_net(a)
    if net["H"] * net["W"] <= 512 * 512:
        return net, 1.0, "1 image of the %s batch" % a.config.upper()
    sub = dict(net, H=strip)
    return sub, strip / net["H"], ("1 image strip of %d rows x full width %d of %s (extrapolated x%d/%d)"
                                   % (strip, net["W"], a.config.upper(), strip, net["H"]))


def eager_layerwise(net, B, params, x_np, lab_np, dev, steps=3):
    """External layer-wise context: the same DAG trained layer by layer in PyTorch
    eager mode -- bf16 channels_last cuDNN convolutions, frozen-BN affine, residual adds, max-pool,
    GAP -> FC -> CE, autograd keeping whatever it keeps, plain SGD.  Returns its peak allocated HBM
    and images/s (CUDA events), or {"error": ...} (e.g. out of memory).  Not our product path."""
    import torch
    import torch.nn.functional as F
    try:
        torch.cuda.empty_cache()
        base = torch.cuda.memory_allocated(dev)
        dt = torch.bfloat16
        ws = []
        for i, op in enumerate(net["ops"]):
            if op["kind"] == "bn":   # fp32 gamma / beta (torch's batch_norm parameters under autocast)
                p = params["convs"][i]
                ws.append({k: torch.tensor(p[k], dtype=torch.float32, device=dev).requires_grad_(True)
                           for k in ("gamma", "beta")})
                continue
            if op["kind"] != "conv":
                ws.append(None)
                continue
            p = params["convs"][i]
            d = {"w": torch.tensor(p["w"], dtype=dt, device=dev).contiguous(memory_format=torch.channels_last)}
            for k in ("b", "gamma", "beta"):
                if k in p:
                    d[k] = torch.tensor(p[k], dtype=dt, device=dev)
            for v in d.values():
                v.requires_grad_(True)
            ws.append(d)
        fw = torch.tensor(params["head"]["fc_w"], dtype=dt, device=dev, requires_grad=True)
        fb = torch.tensor(params["head"]["fc_b"], dtype=dt, device=dev, requires_grad=True)
        leaves = [v for d in ws if d for v in d.values()] + [fw, fb]
        x = torch.tensor(x_np, dtype=dt, device=dev).contiguous(memory_format=torch.channels_last)
        lab = torch.tensor(lab_np, dtype=torch.long, device=dev)

        def step():
            ts = [x]
            for i, op in enumerate(net["ops"]):
                src = ts[op["src"]]
                if op["kind"] == "conv":
                    y = F.conv2d(src, ws[i]["w"], None, op["s"], op["p"])
                    if op["epi"] == "bias":
                        y = y + ws[i]["b"].view(1, -1, 1, 1)
                    elif op["epi"] == "affine":
                        y = y * ws[i]["gamma"].view(1, -1, 1, 1) + ws[i]["beta"].view(1, -1, 1, 1)
                    if op["res"] >= 0:
                        y = y + ts[op["res"]]
                    if op["relu"]:
                        y = F.relu(y)
                elif op["kind"] == "maxpool":
                    y = F.max_pool2d(src, op["k"], op["s"], op["p"])
                elif op["kind"] == "bn":   # training-mode batch statistics (cuDNN / native BN kernel)
                    y = F.batch_norm(src, None, None, ws[i]["gamma"].to(dt), ws[i]["beta"].to(dt), training=True,
                                     eps=1e-5)
                    if op["res"] >= 0:
                        y = y + ts[op["res"]]
                    if op["relu"]:
                        y = F.relu(y)
                else:
                    y = src + ts[op["res"]]
                    if op["relu"]:
                        y = F.relu(y)
                ts.append(y)
            logits = F.linear(ts[-1].float().mean(dim=(2, 3)), fw.float(), fb.float())
            loss = F.cross_entropy(logits, lab)
            loss.backward()
            with torch.no_grad():
                for v in leaves:
                    v -= 1e-3 * v.grad
                    v.grad = None
            return loss

        step()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        step()
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated(dev) - base
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        param_bytes = sum(v.numel() * v.element_size() for v in leaves)
        x_bytes = x.numel() * x.element_size()
        out = {"peak_allocated_bytes": peak, "feature_map_bytes": peak - param_bytes - x_bytes,
               "images_per_s": B / (ms / 1000.0), "ms_per_step": ms,
               "what": "PyTorch %s eager, bf16 channels_last cuDNN, autograd, same DAG (%s), "
                       "SGD; feature maps = peak - params - input"
                       % (torch.__version__, "training-mode BN" if any(o["kind"] == "bn" for o in net["ops"])
                          else "frozen-BN affine")}
    except torch.cuda.OutOfMemoryError as e:
        out = {"error": "out of memory: %s" % str(e).split("\n")[0][:200]}
    except Exception as e:   # context only: never fail the bench on it
        out = {"error": repr(e)[:300]}
    finally:
        torch.cuda.empty_cache()
    return out


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(a, steps=1)             # warm-up/first measurement
    import oracle
    from oracle import column as C
    net, scale, what = oracle_sample(a, 96)
    params = WL.make_params(net, seed=2)
    x = WL.make_input(net, 1, seed=0)
    lab = WL.make_labels(net, 1)
    for _ in range(max(0, a.warmup - 1)):
        params, _, _, _, _ = C.step(net, params, x, lab, 0.01)
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        params, _, _, _, _ = C.step(net, params, x, lab, 0.01)
        times.append(time.perf_counter() - t0)
    ms = 1000.0 * statistics.mean(times) / scale
    v = 1000.0 / ms
    cb = dict(cb, value=v, sample=cb["sample"].replace("mean of 1", "mean of %d" % a.steps))
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
                      "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": "%s (bounded sample per step: %s)" % (CONFIGS[a.config][4], what),
                                 "global_batch": 1, "parallelism": "cpu"},
                      "cpu_baseline": cb,
                      "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def coordination_counters(plan):
    """The paper's two coordination counters (Sec. V-D, Fig. 9): Computation Interruptions
    (2PS-H: one per band boundary and band tensor whose next band reads shared rows computed by the
    band before it) and Overlapped Dimensions (OverL-H: rows of a band tensor that consecutive bands both
    compute), counted from the plan's exact per-band row ranges (lrcnn_plan_rows); plus the sharing
    data the 2PS cache holds (bytes)."""
    ci = od = 0
    for s in range(plan.nsegs()):
        tin, tout, nb = plan.seg(s)
        for r in range(1, nb):
            for t in range(tin + 1, tout + 1):
                lo, a_, _ = plan.rows(s, r, t)
                _, _, b_prev = plan.rows(s, r - 1, t)
                if lo < a_:
                    ci += 1
                od += max(0, b_prev - a_)
    return {"computation_interruptions": ci, "overlapped_rows": od,
            "sharing_data_bytes": plan.memory()["halo_cache"]}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist
    from paper_2401_11471_b200 import lrcnn as LB

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.backend == "gloo":   # code-path check with several ranks sharing the visible GPUs (not a bench)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if a.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)     # non-default stream: lrcnn_step replays a CUDA graph
    torch.cuda.set_stream(stream)

    net = make_net(a)
    B = a.batch or CONFIGS[a.config][3]
    flags = (LB.FLAG_NO_TCGEN05 if a.simt else LB.FLAG_REQUIRE_TC) | (0 if a.no_balanced else LB.FLAG_BALANCED_BANDS)
    if a.no_fuse_block:
        flags |= LB.FLAG_NO_FUSE_BLOCK
    if not a.no_fp_merge:   # decoupled FP bands (N_FP < N_BP, same peak memory)
        flags |= LB.FLAG_FP_MERGE
    if a.allow_overlap:
        flags |= LB.FLAG_ALLOW_OVERLAP_EXHAUSTION
    if a.n_bands is None:
        a.n_bands = 8 if a.config in ("c4", "c5") else 4
    kw = {"band_rows": a.band_rows} if a.band_rows else {"n_bands": a.n_bands}
    if a.mode == "column":
        kw = {}
    rows = world > 1 and a.parallel == "rows"
    # data-parallel replicas over NCCL: the library all-reduces the gradient per segment on its own
    # stream, overlapped with the backward (LRCNN_FLAG_DP); with gloo (N ranks sharing one GPU, to
    # exercise the code path) the caller all-reduces after the step
    lib_dp = world > 1 and not rows and a.backend == "nccl"
    if lib_dp:
        try:
            plan = LB.Plan(net, B, mode=a.mode, prec="bf16", flags=flags | LB.FLAG_DP, world=world, rank=rank, **kw)
            uid = [LB.Comm.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = LB.Comm.nccl(uid[0], rank, world)
            plan.set_comm(comm)
        except Exception as e:   # the library's NCCL communicator could not be created: caller all-reduce
            print("bench: library data-parallel path unavailable (%s); all-reduce after the step" % e, file=sys.stderr)
            lib_dp = False
            plan = LB.Plan(net, B, mode=a.mode, prec="bf16", flags=flags, **kw)
    elif rows:
        if a.bn_train and not a.zero_redundancy:   # batch statistics need every row on exactly one rank
            a.zero_redundancy = True
            if rank == 0:
                print("bench: --bn-train with row sharding uses the zero-redundancy cuts", file=sys.stderr)
        rflags = flags | (LB.FLAG_ZERO_REDUNDANCY if a.zero_redundancy else 0)
        plan = LB.Plan(net, B, mode=a.mode, prec="bf16", flags=rflags, world=world, rank=rank, **kw)
        uid = [LB.Comm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = LB.Comm.nccl(uid[0], rank, world)
        plan.set_comm(comm)
    elif a.mem_budget_gb > 0 and a.mode != "column":
        plan = LB.Plan.for_budget(net, B, int(a.mem_budget_gb * 1e9), max_bands=64, mode=a.mode, prec="bf16",
                                  flags=flags)
        kw = {"n_bands": plan.n_bands, "mem_budget_gb": a.mem_budget_gb}
    else:
        plan = LB.Plan(net, B, mode=a.mode, prec="bf16", flags=flags, **kw)
    mem = plan.memory()

    torch.cuda.reset_peak_memory_stats(dev)
    ds = LB.DeviceState(plan, device=dev)
    params = WL.make_params(net, seed=2)
    x_np = WL.make_input(net, B, seed=1000 + (0 if rows else rank))   # rows: every rank sees the same batch
    lab_np = WL.make_labels(net, B, seed=1 + (0 if rows else rank))
    ds.load(params=params, x=x_np, labels=lab_np)
    xi_bytes = ds.x.numel() * ds.x.element_size()
    lab_bytes = ds.labels.numel() * 4
    lr = 1e-3

    def one_step():
        if lib_dp:   # sum over replicas inside the step; the mean folded into lr
            plan.step(ds.master, ds.params, ds.grads, ds.x, ds.labels, lr / world, ds.loss, ds.ws, stream)
        elif world > 1 and not rows:
            plan.step_grads(ds.params, ds.grads, ds.x, ds.labels, ds.loss, ds.ws, stream)
            dist.all_reduce(ds.grads)          # wgrad all-reduce (NCCL, fp32, sum)
            plan.sgd(ds.master, ds.params, ds.grads, lr / world, stream)   # mean over replicas folded into lr
        else:
            plan.step(ds.master, ds.params, ds.grads, ds.x, ds.labels, lr, ds.loss, ds.ws, stream)

    for i in range(a.warmup):
        if i == 0 and lib_dp:
            try:
                one_step()
                torch.cuda.synchronize()
            except Exception as e:   # same workspace layout (DP plans the whole image): switch paths
                print("bench: library data-parallel step failed (%s); all-reduce after the step" % e, file=sys.stderr)
                plan.set_comm(None)
                comm.free()
                lib_dp = False
                plan = LB.Plan(net, B, mode=a.mode, prec="bf16", flags=flags, **kw)
                ds.plan = plan
                one_step()
            continue
        one_step()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated(dev)
    xi = ds.params.numel() * ds.params.element_size() + (ds.master.numel() + ds.grads.numel()) * 4
    launches_per_step = plan.last_launches()

    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed region (device)
    sampler = ClockSampler(local)
    sampler.start()
    times = []
    host_s = 0.0
    barrier()
    for _ in range(a.steps):
        flush.zero_()                               # L2 flushed between timed steps (untimed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        one_step()
        host_s += time.perf_counter() - h0
        e1.record(stream)
        times.append((e0, e1))
    barrier()
    clocks = sampler.result()
    ms = [s.elapsed_time(e) for s, e in times]
    ms_step = sum(ms) / len(ms)
    if world > 1:
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t)
    gb = B if rows else B * world        # images per step of the whole job
    value = gb / (ms_step / 1000.0)

    # ---------------------------------------------------------------- end-to-end through the public API
    # Every step copies its batch from pinned host memory and reads the loss back.  The H2D copy of
    # batch i+1 runs on a copy stream into a device staging buffer while step i computes (double
    # buffering, as a training loop feeding the library would); the step then takes its batch with a
    # device-to-device copy.  Steps run back to back (no L2 flush: the per-step working set, ~0.6 GB
    # for C2, exceeds the 126 MB L2).  Timed as a whole on the device: first copy to last loss.
    x_host = ds.x.cpu().pin_memory()
    lab_host = ds.labels.cpu().pin_memory()
    loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
    x_stage, lab_stage = torch.empty_like(ds.x), torch.empty_like(ds.labels)
    cstream = torch.cuda.Stream(device=dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    cstream.wait_event(e0)
    staged = torch.cuda.Event()
    with torch.cuda.stream(cstream):
        x_stage.copy_(x_host, non_blocking=True)
        lab_stage.copy_(lab_host, non_blocking=True)
        staged.record(cstream)
    for i in range(a.steps):
        stream.wait_event(staged)
        ds.x.copy_(x_stage, non_blocking=True)
        ds.labels.copy_(lab_stage, non_blocking=True)
        taken = torch.cuda.Event()
        taken.record(stream)
        if i + 1 < a.steps:
            cstream.wait_event(taken)
            staged = torch.cuda.Event()
            with torch.cuda.stream(cstream):
                x_stage.copy_(x_host, non_blocking=True)
                lab_stage.copy_(lab_host, non_blocking=True)
                staged.record(cstream)
        one_step()
        loss_host.copy_(ds.loss, non_blocking=True)
    e1.record(stream)
    barrier()
    ms_e2e = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    plan.profile(True)
    plan.profile_reset()
    for _ in range(max(2, min(a.steps, 5))):
        flush.zero_()
        one_step()
    tc_ms, tc_n, tc_fl = plan.profile_read(0, stream)
    wg_ms, wg_n, wg_fl = plan.profile_read(1, stream)
    ot_ms, ot_n, _ = plan.profile_read(2, stream)
    kern = plan.profile_kernels(0, stream) + plan.profile_kernels(1, stream)
    if a.per_op_csv:
        plan.profile_dump(a.per_op_csv, stream)
    plan.profile(False)
    peaks, peak_src = measured_peaks()
    achieved = tc_fl / (tc_ms / 1000.0) / 1e12 if tc_ms > 0 else 0.0
    # the burst bf16 peak when the SM clock sat at its maximum during the timed steps, else the
    # sustained (power-capped) one (B200_PROFILING: burst for a kernel at full clock)
    at_max = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and
                  clocks["sm_mhz"] >= 0.97 * clocks["sm_max_mhz"])
    peak_kind = "bf16_tflops" if at_max else "bf16_tflops_sustained"
    peak_tf = peaks.get(peak_kind, peaks.get("bf16_tflops_sustained", 1385.7))
    prof_steps = max(2, min(a.steps, 5))
    hbm_gbs = peaks.get("hbm_gbs", 6550.0)
    ridge = peak_tf * 1e12 / (hbm_gbs * 1e9)          # FLOP/B where the two rooflines meet
    # each kernel against the roofline its algorithmic intensity puts it under:
    # tensor-bound: algorithmic conv FLOPs / time vs the bf16 tensor peak; HBM-bound: algorithmic
    # bytes (every operand read once, every result written once) / time vs the measured copy bandwidth
    # HBM writes alone sustain less than a copy on this GPU (measured here: a 1 GiB fill), so an
    # HBM-bound kernel that writes more than it reads has a lower ceiling than the copy peak: its
    # mixed roofline is bytes / max(bytes / copy_bw, written / write_bw) (reported beside `frac`)
    wbuf = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    wbuf.fill_(1)
    wts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        wbuf.fill_(0)
        e1.record(stream)
        e1.synchronize()
        wts.append(e0.elapsed_time(e1))
    write_gbs = wbuf.numel() / (min(wts) / 1000.0) / 1e9
    del wbuf

    def _rl(k):
        sec = k["ms"] / 1000.0
        if sec <= 0:
            return {"bound": "tensor", "achieved": 0.0, "peak": peak_tf, "unit": "TFLOP/s", "frac": 0.0}
        if k.get("bytes", 0) > 0 and k["flops"] / k["bytes"] < ridge:
            gbs = k["bytes"] / sec / 1e9
            t_min = max(k["bytes"] / (hbm_gbs * 1e9), k.get("wbytes", 0.0) / (write_gbs * 1e9))
            mix = k["bytes"] / t_min / 1e9
            return {"bound": "hbm", "achieved": gbs, "peak": hbm_gbs, "unit": "GB/s", "frac": gbs / hbm_gbs,
                    "write_share": k.get("wbytes", 0.0) / k["bytes"],
                    "mixed_rw_roofline": {"peak": mix, "frac": gbs / mix, "write_gbs_measured": write_gbs}}
        tf = k["flops"] / sec / 1e12
        return {"bound": "tensor", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": tf / peak_tf}
    # the dominant kernel: the tcgen05 kernel with the largest share of the step (CUDA events around
    # each of its launches on the launching stream)
    kern = [dict(k, name=demangle(k["name"])) for k in kern]
    dom = max(kern, key=lambda k: k["ms"]) if kern else None
    traffic = None
    try:   # DRAM bytes per launch of this kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get("per_kernel", {}).get(dom["name"]) if dom else None
    except Exception:
        pass
    drl = _rl(dom) if dom else _rl({"ms": 0, "flops": 0})
    roofline = dict(drl, kernel=dom["name"] if dom else None, traffic=traffic,
                    algorithmic_bytes_per_launch=dom["bytes"] / dom["launches"] if dom and dom["launches"] else None,
                    peak_source="%s %s" % (peak_src, peak_kind if drl["bound"] == "tensor" else "hbm_gbs"),
                    frac_vs_sustained=(drl["achieved"] / peaks.get("bf16_tflops_sustained", 1385.7)
                                       if drl["bound"] == "tensor" else None),
                    frac_vs_burst=(drl["achieved"] / peaks.get("bf16_tflops", 1642.8)
                                   if drl["bound"] == "tensor" else None),
                    # NVIDIA's nominal dense bf16 2.25 PFLOP/s (B200_PROFILING) scaled to the median SM clock of
                    # the timed steps: the hardware ceiling at the clock the power cap left (the measured cuBLAS
                    # peaks were taken at other clocks -- the sustained one at ~1357 MHz -- so a kernel at a
                    # higher clock can exceed them)
                    nominal_tflops_at_clock=(2250.0 * clocks["sm_mhz"] / 1965.0 if clocks.get("sm_mhz") else None),
                    frac_vs_nominal_at_clock=(drl["achieved"] / (2250.0 * clocks["sm_mhz"] / 1965.0)
                                              if drl["bound"] == "tensor" and clocks.get("sm_mhz") else None),
                    exceeds_measured_peak=bool(drl["frac"] > 1.0),
                    ridge_flop_per_byte=ridge,
                    launches_per_step=dom["launches"] / prof_steps if dom else 0,
                    ms_per_step=dom["ms"] / prof_steps if dom else 0,
                    share_of_step=(dom["ms"] / prof_steps) / ms_step if dom else 0,
                    all_conv_fp_dgrad={"achieved": achieved, "unit": "TFLOP/s",
                                       "frac": achieved / peak_tf if peak_tf else None,
                                       "launches_per_step": tc_n / prof_steps, "ms_per_step": tc_ms / prof_steps},
                    wgrad={"achieved": wg_fl / (wg_ms / 1000.0) / 1e12 if wg_ms else 0.0, "unit": "TFLOP/s",
                           "ms_per_step": wg_ms / prof_steps},
                    other_ms_per_step=ot_ms / prof_steps,
                    kernels=sorted([dict(_rl(k), name=k["name"], ms_per_step=k["ms"] / prof_steps,
                                         tflops=k["flops"] / (k["ms"] / 1000.0) / 1e12 if k["ms"] > 0 else 0.0)
                                    for k in kern], key=lambda k: -k["ms_per_step"])[:10])

    # ---------------------------------------------------------------- memory vs layer-wise (COLUMN)
    # feature-map HBM = allocator peak - xi (params, fp32 master, fp32 grads; the paper's xi),
    # compared with three layer-wise references: Eq. (3) Omega (every op output stored once, bf16 --
    # the analytical floor of layer-wise training), the same library in COLUMN mode (every map kept,
    # same kernels) and PyTorch eager autograd on the same DAG (measured, external context)
    fm = peak - xi
    mem_rep = {"peak_allocated_bytes": peak, "xi_bytes": xi, "feature_map_bytes": fm,
               "omega_eq3_bytes": mem["omega"], "reduction_vs_omega_x": mem["omega"] / max(1, fm),
               # Eq. (3) sums the op outputs l = 1..L; the input batch (bf16, channels padded 3 -> 8
               # for 16-byte TMA pixels) is data, like xi: the same ratio without it
               "input_batch_bytes": xi_bytes, "feature_map_excl_input_bytes": fm - xi_bytes,
               "reduction_vs_omega_excl_input_x": mem["omega"] / max(1, fm - xi_bytes),
               "plan": {k: mem[k] for k in ("omega", "band_act", "band_delta", "halo_cache", "carry",
                                            "checkpoints", "delta_full", "workspace")}}
    mem_rep["coordination"] = coordination_counters(plan)
    cpu = None
    if not a.no_baselines and world == 1 and a.mode != "column":   # layer-wise memory + cpu_baseline: N=1 only
        del ds, flush
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(dev)
        cplan = LB.Plan(net, B, mode="column", prec="bf16", flags=flags)
        cds = LB.DeviceState(cplan, device=dev)
        cds.load(params=params, x=x_np, labels=lab_np)
        cplan.step(cds.master, cds.params, cds.grads, cds.x, cds.labels, lr, cds.loss, cds.ws, stream)
        torch.cuda.synchronize()
        cpeak = torch.cuda.max_memory_allocated(dev)
        mem_rep["layerwise_column_peak_allocated_bytes"] = cpeak
        mem_rep["layerwise_column_feature_map_bytes"] = cpeak - xi
        mem_rep["reduction_vs_column_x"] = (cpeak - xi) / max(1, fm)
        del cds, cplan
        torch.cuda.empty_cache()
        if not a.no_eager:
            with torch.cuda.stream(torch.cuda.Stream(device=dev)):
                eg = eager_layerwise(net, B, params, x_np, lab_np, dev)
            mem_rep["layerwise_pytorch_eager"] = eg
            if "feature_map_bytes" in eg:
                mem_rep["reduction_vs_pytorch_eager_x"] = eg["feature_map_bytes"] / max(1, fm)
        cpu = cpu_baseline(a)

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               "scaling": "strong" if rows else "weak",
               "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded U[0,1) images, U{0..9} labels)",
               "config": {"workload": "%s, batch %d per GPU, bf16%s" % (CONFIGS[a.config][4], B,
                                                                       ", training-mode BatchNorm" if a.bn_train else ""),
                          "global_batch": gb, "seq_len": None,
                          "parallelism": ("rows%d (row sharding%s, NCCL halo exchange + per-segment wgrad all-reduce)"
                                          % (world, ", zero redundancy" if a.zero_redundancy else ", OverL at the cuts")
                                          if rows
                                          else "dp%d (per-segment NCCL wgrad all-reduce overlapped with the backward)" % world
                                          if lib_dp else "dp%d (wgrad all-reduce after the step, %s)" % (world, a.backend)
                                          if world > 1 else "single GPU"),
                          "mode": a.mode, "segments": a.segments, "bands": kw,
                          "bands_per_segment": [plan.seg(si)[2] for si in range(plan.nsegs())],
                          "fp_bands_per_segment": [plan.fp_bands(si)[0] for si in range(plan.nsegs())],
                          "l2": "flushed (512 MB write) between timed steps"},
               "clocks": clocks,
               "e2e": {"value": gb / (ms_e2e / 1000.0), "unit": UNIT, "h2d_bytes_per_step": xi_bytes + lab_bytes,
                       "d2h_bytes_per_step": 4, "ms_per_step": ms_e2e},
               "gpu_launches": launches_per_step * a.steps,
               "simt_fallbacks_per_step": plan.last_simt_fallbacks(),
               "host_enqueue_ms_per_step": 1000.0 * host_s / a.steps,
               "roofline": roofline, "memory": mem_rep, "cpu_baseline": cpu,
               "tensor_core_kernels": (not a.simt)}
        print(json.dumps(out), flush=True)
    if rows or lib_dp:
        plan.set_comm(None)
        comm.free()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
