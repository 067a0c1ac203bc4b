"""Thin Python binding of liblrcnn.so (include/lrcnn.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
packs arguments (ctypes structs, device pointers from torch tensors, the
caller's CUDA stream) and converts the parameter layout.  PyTorch is used for
device memory and streams.  If the shared library is missing the import fails
loudly: there is no CPU or PyTorch fallback for any compute.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblrcnn.so")

OP_CONV, OP_MAXPOOL, OP_ADD, OP_BN = 0, 1, 2, 3
EPI = {"none": 0, "bias": 1, "affine": 2}
MODES = {"column": 0, "2ps": 1, "overl": 2}
PRECS = {"fp32": 0, "bf16": 1}
FLAG_ALLOW_OVERLAP_EXHAUSTION = 1
FLAG_NO_TCGEN05 = 2
FLAG_BALANCED_BANDS = 4
FLAG_NO_FUSE_RES = 8
FLAG_FP_MERGE = 16
FLAG_DP = 32
FLAG_REQUIRE_TC = 64
FLAG_AUTO_SEGMENTS = 128
FLAG_ZERO_REDUNDANCY = 256
FLAG_NO_FUSE_BLOCK = 512
STATUS = {0: "OK", 1: "E_ARG", 2: "E_SHAPE", 3: "E_INFEASIBLE", 4: "E_DEGENERATE", 5: "E_STATE",
          6: "E_WORKSPACE", 7: "E_CUDA", 8: "E_NCCL", 9: "E_UNSUPPORTED"}


class LrcnnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("lrcnn %s: %s" % (STATUS.get(status, status), msg))
        self.status = status
        self.name = STATUS.get(status, str(status))


class Op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("src", ctypes.c_int), ("res", ctypes.c_int), ("c_out", ctypes.c_int),
                ("k", ctypes.c_int), ("s", ctypes.c_int), ("p", ctypes.c_int), ("epi", ctypes.c_int),
                ("relu", ctypes.c_int), ("seg_end", ctypes.c_int)]


class NetDesc(ctypes.Structure):
    _fields_ = [("n_ops", ctypes.c_int), ("ops", ctypes.POINTER(Op)), ("B", ctypes.c_int), ("C", ctypes.c_int),
                ("H", ctypes.c_int), ("W", ctypes.c_int), ("n_classes", ctypes.c_int)]


class PlanOpts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("prec", ctypes.c_int), ("band_rows", ctypes.c_int),
                ("n_bands", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("flags", ctypes.c_int), ("first_rows_pm", ctypes.c_int)]


class MemoryReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_size_t) for n in ("omega", "band_act", "band_delta", "halo_cache", "carry",
                                                "checkpoints", "delta_full", "other", "workspace")] + \
               [(n, ctypes.c_double) for n in ("tau_flops", "fwd_flops", "step_flops")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


# host-staged communicator callbacks (lrcnn_comm_init_host)
HOST_EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(ctypes.c_size_t))
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_size_t)

EXPORTS = ["lrcnn_plan", "lrcnn_plan_budget", "lrcnn_plan_greedy", "lrcnn_plan_turning_point", "lrcnn_plan_free", "lrcnn_plan_sizes", "lrcnn_plan_tensor", "lrcnn_plan_param",
           "lrcnn_plan_nsegs", "lrcnn_plan_seg", "lrcnn_plan_rows", "lrcnn_plan_read_end", "lrcnn_plan_zr_halo", "lrcnn_plan_fp_bands", "lrcnn_plan_memory", "lrcnn_forward_rows",
           "lrcnn_backward_rows", "lrcnn_step", "lrcnn_step_grads", "lrcnn_sgd", "lrcnn_profile_enable", "lrcnn_profile_read",
           "lrcnn_profile_reset", "lrcnn_profile_dump", "lrcnn_profile_kernels", "lrcnn_plan_shard", "lrcnn_plan_xfers",
           "lrcnn_comm_nccl_unique_id", "lrcnn_comm_init_nccl", "lrcnn_comm_loopback_group",
           "lrcnn_comm_loopback_group_free", "lrcnn_comm_init_loopback", "lrcnn_comm_init_host", "lrcnn_comm_free", "lrcnn_plan_set_comm",
           "lrcnn_last_launch_count", "lrcnn_last_tc_launch_count", "lrcnn_last_simt_fallbacks", "lrcnn_debug_capture",
           "lrcnn_last_error", "lrcnn_version"]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("liblrcnn.so not built (%s); run `python -m paper_2401_11471_b200.build` "
                          "-- there is no fallback path" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i, ip = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_int)
    szp = ctypes.POINTER(ctypes.c_size_t)
    L.lrcnn_plan.argtypes = [ctypes.POINTER(NetDesc), ctypes.POINTER(PlanOpts), ctypes.POINTER(vp)]
    L.lrcnn_plan_free.argtypes = [vp]
    L.lrcnn_plan_budget.argtypes = [ctypes.POINTER(NetDesc), ctypes.POINTER(PlanOpts), sz, i, ctypes.POINTER(vp), ip]
    L.lrcnn_plan_greedy.argtypes = [ctypes.POINTER(NetDesc), ctypes.POINTER(PlanOpts), sz, i, ctypes.POINTER(vp), ip,
                                    ip]
    L.lrcnn_plan_turning_point.argtypes = [ctypes.POINTER(NetDesc), ctypes.POINTER(PlanOpts), i, ip, szp]
    L.lrcnn_plan_sizes.argtypes = [vp, szp, szp, szp]
    L.lrcnn_plan_tensor.argtypes = [vp, i, ip, ip, ip, ip]
    L.lrcnn_plan_param.argtypes = [vp, i, i, szp, szp]
    L.lrcnn_plan_nsegs.argtypes = [vp, ip]
    L.lrcnn_plan_seg.argtypes = [vp, i, ip, ip, ip]
    L.lrcnn_plan_fp_bands.argtypes = [vp, i, ip, ip]
    L.lrcnn_plan_rows.argtypes = [vp, i, i, i, ip, ip, ip]
    L.lrcnn_plan_read_end.argtypes = [vp, i, i, i, ip]
    L.lrcnn_plan_zr_halo.argtypes = [vp, i, i, ip, ip, ip, ip, ip]
    L.lrcnn_plan_memory.argtypes = [vp, ctypes.POINTER(MemoryReport)]
    L.lrcnn_forward_rows.argtypes = [vp, vp, vp, vp, vp, sz, vp]
    L.lrcnn_backward_rows.argtypes = [vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.lrcnn_step.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_float, vp, vp, sz, vp]
    L.lrcnn_step_grads.argtypes = [vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.lrcnn_sgd.argtypes = [vp, vp, vp, vp, ctypes.c_float, vp]
    L.lrcnn_profile_enable.argtypes = [vp, i]
    L.lrcnn_profile_read.argtypes = [vp, i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong),
                                     ctypes.POINTER(ctypes.c_double), vp]
    L.lrcnn_profile_reset.argtypes = [vp]
    L.lrcnn_profile_dump.argtypes = [vp, ctypes.c_char_p, vp]
    L.lrcnn_profile_kernels.argtypes = [vp, i, ctypes.c_char_p, sz, vp]
    L.lrcnn_last_launch_count.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
    L.lrcnn_plan_shard.argtypes = [vp, i, i, ip, ip, ip, ip]
    L.lrcnn_plan_xfers.argtypes = [vp, i, i, ip, ip, ip, ip, ip]
    L.lrcnn_comm_nccl_unique_id.argtypes = [vp]
    L.lrcnn_comm_init_nccl.argtypes = [vp, i, i, ctypes.POINTER(vp)]
    L.lrcnn_comm_loopback_group.argtypes = [i, ctypes.POINTER(vp)]
    L.lrcnn_comm_loopback_group_free.argtypes = [vp]
    L.lrcnn_comm_init_loopback.argtypes = [vp, i, ctypes.POINTER(vp)]
    L.lrcnn_comm_init_host.argtypes = [i, i, HOST_EXCHANGE_FN, HOST_ALLREDUCE_FN, vp, ctypes.POINTER(vp)]
    L.lrcnn_comm_free.argtypes = [vp]
    L.lrcnn_plan_set_comm.argtypes = [vp, vp]
    L.lrcnn_last_tc_launch_count.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
    L.lrcnn_last_simt_fallbacks.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
    L.lrcnn_debug_capture.argtypes = [vp, i, vp]
    L.lrcnn_last_error.restype = ctypes.c_char_p
    L.lrcnn_version.restype = ctypes.c_char_p
    for n in EXPORTS:
        if n not in ("lrcnn_last_error", "lrcnn_version"):
            getattr(L, n).restype = ctypes.c_int
    _lib = L
    return L


def _check(st):
    if st != 0:
        raise LrcnnError(st, lib().lrcnn_last_error().decode())


def _ptr(t):
    """Device pointer of a torch tensor (or an int address)."""
    if t is None:
        return None
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def net_ops(net):
    """Marshal a workloads-style net dict into the C op array."""
    ops = (Op * len(net["ops"]))()
    for i, o in enumerate(net["ops"]):
        kind = {"conv": OP_CONV, "maxpool": OP_MAXPOOL, "add": OP_ADD, "bn": OP_BN}[o["kind"]]
        ops[i] = Op(kind, o["src"], o.get("res", -1) if o.get("res", -1) is not None else -1, o.get("cout", 0),
                    o.get("k", 1), o.get("s", 1), o.get("p", 0), EPI[o.get("epi", "none")] if kind == OP_CONV else 0,
                    1 if o.get("relu", False) else 0, 1 if o.get("seg_end", False) else 0)
    return ops


class Plan:
    """lrcnn_plan wrapper.  mode: column | 2ps | overl; prec: fp32 | bf16."""

    def __init__(self, net, B, mode="2ps", prec="bf16", band_rows=None, n_bands=None, flags=0, rank=0, world=1,
                 first_rows_pm=0):
        L = lib()
        self.net, self.B, self.mode, self.prec = net, B, mode, prec
        self._ops = net_ops(net)
        self._desc = NetDesc(len(net["ops"]), self._ops, B, net["C"], net["H"], net["W"], net["classes"])
        self._opts = PlanOpts(MODES[mode], PRECS[prec], band_rows or 0, n_bands or 0, rank, world, flags,
                              first_rows_pm)
        h = ctypes.c_void_p()
        _check(L.lrcnn_plan(ctypes.byref(self._desc), ctypes.byref(self._opts), ctypes.byref(h)))
        self.h = h
        ws, npar, zl = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(L.lrcnn_plan_sizes(self.h, ctypes.byref(ws), ctypes.byref(npar), ctypes.byref(zl)))
        self.ws_bytes, self.n_params, self.zl_elems = ws.value, npar.value, zl.value
        self.elem = 2 if prec == "bf16" else 4

    @classmethod
    def for_budget(cls, net, B, budget_bytes, max_bands=64, mode="2ps", prec="bf16", flags=0):
        """lrcnn_plan_budget: the smallest band count whose workspace fits budget_bytes."""
        L = lib()
        self = cls.__new__(cls)
        self.net, self.B, self.mode, self.prec = net, B, mode, prec
        self._ops = net_ops(net)
        self._desc = NetDesc(len(net["ops"]), self._ops, B, net["C"], net["H"], net["W"], net["classes"])
        self._opts = PlanOpts(MODES[mode], PRECS[prec], 0, 0, 0, 1, flags, 0)
        h, nb = ctypes.c_void_p(), ctypes.c_int()
        _check(L.lrcnn_plan_budget(ctypes.byref(self._desc), ctypes.byref(self._opts), budget_bytes, max_bands,
                                   ctypes.byref(h), ctypes.byref(nb)))
        self.h = h
        self.n_bands = nb.value
        ws, npar, zl = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(L.lrcnn_plan_sizes(self.h, ctypes.byref(ws), ctypes.byref(npar), ctypes.byref(zl)))
        self.ws_bytes, self.n_params, self.zl_elems = ws.value, npar.value, zl.value
        self.elem = 2 if prec == "bf16" else 4
        return self

    @classmethod
    def greedy(cls, net, B, budget_bytes, max_bands=64, prec="bf16", flags=0):
        """lrcnn_plan_greedy (Eq. (12)): min N, then the largest first band, whose workspace fits."""
        L = lib()
        self = cls.__new__(cls)
        self.net, self.B, self.mode, self.prec = net, B, "2ps", prec
        self._ops = net_ops(net)
        self._desc = NetDesc(len(net["ops"]), self._ops, B, net["C"], net["H"], net["W"], net["classes"])
        self._opts = PlanOpts(MODES["2ps"], PRECS[prec], 0, 0, 0, 1, flags, 0)
        h, nb, pm = ctypes.c_void_p(), ctypes.c_int(), ctypes.c_int()
        _check(L.lrcnn_plan_greedy(ctypes.byref(self._desc), ctypes.byref(self._opts), budget_bytes, max_bands,
                                   ctypes.byref(h), ctypes.byref(nb), ctypes.byref(pm)))
        self.h = h
        self.n_bands, self.first_rows_pm = nb.value, pm.value
        ws, npar, zl = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(L.lrcnn_plan_sizes(self.h, ctypes.byref(ws), ctypes.byref(npar), ctypes.byref(zl)))
        self.ws_bytes, self.n_params, self.zl_elems = ws.value, npar.value, zl.value
        self.elem = 2 if prec == "bf16" else 4
        return self

    @staticmethod
    def turning_point(net, B, max_bands=64, mode="2ps", prec="bf16", flags=0):
        """lrcnn_plan_turning_point: (n*, workspace bytes at n*)."""
        L = lib()
        ops = net_ops(net)
        desc = NetDesc(len(net["ops"]), ops, B, net["C"], net["H"], net["W"], net["classes"])
        opts = PlanOpts(MODES[mode], PRECS[prec], 0, 0, 0, 1, flags, 0)
        n, ws = ctypes.c_int(), ctypes.c_size_t()
        _check(L.lrcnn_plan_turning_point(ctypes.byref(desc), ctypes.byref(opts), max_bands, ctypes.byref(n),
                                          ctypes.byref(ws)))
        return n.value, ws.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().lrcnn_plan_free(self.h)
                self.h = None
        except Exception:
            pass

    # ------------------------------------------------------------ plan queries
    def tensor(self, tid):
        c, cp, h, w = (ctypes.c_int() for _ in range(4))
        _check(lib().lrcnn_plan_tensor(self.h, tid, ctypes.byref(c), ctypes.byref(cp), ctypes.byref(h), ctypes.byref(w)))
        return c.value, cp.value, h.value, w.value

    def param(self, op, which):
        o, n = ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().lrcnn_plan_param(self.h, op, which, ctypes.byref(o), ctypes.byref(n)))
        return o.value, n.value

    def nsegs(self):
        n = ctypes.c_int()
        _check(lib().lrcnn_plan_nsegs(self.h, ctypes.byref(n)))
        return n.value

    def seg(self, s):
        a, b, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().lrcnn_plan_seg(self.h, s, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, n.value

    def fp_bands(self, s):
        """(N_FP, N_BP) of segment s (lrcnn_plan_fp_bands; N_FP < N_BP with FLAG_FP_MERGE)."""
        nf, nb = ctypes.c_int(), ctypes.c_int()
        _check(lib().lrcnn_plan_fp_bands(self.h, s, ctypes.byref(nf), ctypes.byref(nb)))
        return nf.value, nb.value

    def rows(self, seg, band, tid):
        lo, a, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().lrcnn_plan_rows(self.h, seg, band, tid, ctypes.byref(lo), ctypes.byref(a), ctypes.byref(b)))
        return lo.value, a.value, b.value

    def read_end(self, seg, band, tid):
        """One past the last row of tid band `band` reads (lrcnn_plan_read_end)."""
        hb = ctypes.c_int()
        _check(lib().lrcnn_plan_read_end(self.h, seg, band, tid, ctypes.byref(hb)))
        return hb.value

    def zr_halo(self, seg):
        """Zero-redundancy halo schedule of segment seg: [(tensor, dir, r0, r1)] (lrcnn_plan_zr_halo)."""
        n = ctypes.c_int()
        arrs = [(ctypes.c_int * 256)() for _ in range(4)]
        _check(lib().lrcnn_plan_zr_halo(self.h, seg, 256, ctypes.byref(n), *arrs))
        return [tuple(a[i] for a in arrs) for i in range(n.value)]

    def shard(self, seg, tid):
        """(own_lo, own_hi, lo, hi): owned segment-output rows and tensor tid's extended range."""
        v = [ctypes.c_int() for _ in range(4)]
        _check(lib().lrcnn_plan_shard(self.h, seg, tid, *[ctypes.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def xfers(self, seg):
        """Halo transfers of segment seg's input: list of (peer, send, r0, r1)."""
        n = ctypes.c_int()
        arrs = [(ctypes.c_int * 16)() for _ in range(4)]
        _check(lib().lrcnn_plan_xfers(self.h, seg, 16, ctypes.byref(n), *arrs))
        return [tuple(a[i] for a in arrs) for i in range(n.value)]

    def set_comm(self, comm):
        _check(lib().lrcnn_plan_set_comm(self.h, comm.h if comm is not None else None))
        self._comm = comm

    def memory(self):
        m = MemoryReport()
        _check(lib().lrcnn_plan_memory(self.h, ctypes.byref(m)))
        return m.as_dict()

    # ------------------------------------------------------------ layouts (marshalling)
    def pack_params(self, params):
        """Canonical params (OIHW float arrays, workloads.make_params) -> flat plan layout (float32 numpy)."""
        flat = np.zeros(self.n_params, dtype=np.float32)
        for i, op in enumerate(self.net["ops"]):
            p = params["convs"][i]
            if p is None:
                continue
            if op["kind"] == "bn":   # gamma, beta (lrcnn.h: per BN op gamma[C], beta[C])
                off, n = self.param(i, 1)
                flat[off:off + n] = p["gamma"]
                off, n = self.param(i, 2)
                flat[off:off + n] = p["beta"]
                continue
            off, n = self.param(i, 0)
            w = np.asarray(p["w"], dtype=np.float64)
            co, ci, k, _ = w.shape
            cinp = self.tensor(op["src"])[1]
            ohwi = np.zeros((co, k, k, cinp))
            ohwi[..., :ci] = w.transpose(0, 2, 3, 1)
            assert ohwi.size == n
            flat[off:off + n] = ohwi.ravel()
            if op["epi"] == "bias":
                off, n = self.param(i, 1)
                flat[off:off + n] = p["b"]
            elif op["epi"] == "affine":
                off, n = self.param(i, 1)
                flat[off:off + n] = p["gamma"]
                off, n = self.param(i, 2)
                flat[off:off + n] = p["beta"]
        L = len(self.net["ops"])
        cl, clp = self.tensor(L)[0], self.tensor(L)[1]
        off, n = self.param(L, 0)
        fw = np.zeros((self.net["classes"], clp))
        fw[:, :cl] = params["head"]["fc_w"]
        flat[off:off + n] = fw.ravel()
        off, n = self.param(L, 1)
        flat[off:off + n] = params["head"]["fc_b"]
        return flat

    def unpack_grads(self, flat):
        """Flat fp32 gradients -> per-op dicts in the canonical (OIHW) layout."""
        flat = np.asarray(flat, dtype=np.float64)
        out = []
        for i, op in enumerate(self.net["ops"]):
            if op["kind"] == "bn":
                g = {}
                off, n = self.param(i, 1)
                g["gamma"] = flat[off:off + n]
                off, n = self.param(i, 2)
                g["beta"] = flat[off:off + n]
                out.append(g)
                continue
            if op["kind"] != "conv":
                out.append(None)
                continue
            off, n = self.param(i, 0)
            cin = self.tensor(op["src"])[0]
            cinp = self.tensor(op["src"])[1]
            k = op["k"]
            w = flat[off:off + n].reshape(op["cout"], k, k, cinp)[..., :cin].transpose(0, 3, 1, 2)
            g = {"w": w}
            if op["epi"] == "bias":
                off, n = self.param(i, 1)
                g["b"] = flat[off:off + n]
            elif op["epi"] == "affine":
                off, n = self.param(i, 1)
                g["gamma"] = flat[off:off + n]
                off, n = self.param(i, 2)
                g["beta"] = flat[off:off + n]
            out.append(g)
        L = len(self.net["ops"])
        cl = self.tensor(L)[0]
        clp = self.tensor(L)[1]
        off, n = self.param(L, 0)
        head = {"fc_w": flat[off:off + n].reshape(self.net["classes"], clp)[:, :cl]}
        off, n = self.param(L, 1)
        head["fc_b"] = flat[off:off + n]
        return out, head

    def to_nhwc(self, x_nchw, tid=0):
        """NCHW float array -> NHWC with channels padded to Cp (float32 numpy)."""
        c, cp, h, w = self.tensor(tid)
        x = np.asarray(x_nchw, dtype=np.float64)
        out = np.zeros((x.shape[0], h, w, cp), dtype=np.float32)
        out[..., :c] = x.transpose(0, 2, 3, 1)
        return out

    def from_nhwc(self, y, tid):
        c, cp, h, w = self.tensor(tid)
        y = np.asarray(y, dtype=np.float64).reshape(self.B, h, w, cp)
        return y[..., :c].transpose(0, 3, 1, 2)

    # ------------------------------------------------------------ device calls
    def forward_rows(self, params, x, zl, ws, stream=None):
        _check(lib().lrcnn_forward_rows(self.h, _ptr(params), _ptr(x), _ptr(zl), _ptr(ws), self.ws_bytes,
                                        _stream(stream)))

    def backward_rows(self, params, x, zl, dzl, grads, ws, stream=None):
        _check(lib().lrcnn_backward_rows(self.h, _ptr(params), _ptr(x), _ptr(zl), _ptr(dzl), _ptr(grads), _ptr(ws),
                                         self.ws_bytes, _stream(stream)))

    def step(self, master, params, grads, x, labels, lr, loss, ws, stream=None):
        _check(lib().lrcnn_step(self.h, _ptr(master), _ptr(params), _ptr(grads), _ptr(x), _ptr(labels),
                                ctypes.c_float(lr), _ptr(loss), _ptr(ws), self.ws_bytes, _stream(stream)))

    def step_grads(self, params, grads, x, labels, loss, ws, stream=None):
        _check(lib().lrcnn_step_grads(self.h, _ptr(params), _ptr(grads), _ptr(x), _ptr(labels), _ptr(loss),
                                      _ptr(ws), self.ws_bytes, _stream(stream)))

    def sgd(self, master, params, grads, lr, stream=None):
        _check(lib().lrcnn_sgd(self.h, _ptr(master), _ptr(params), _ptr(grads), ctypes.c_float(lr),
                               _stream(stream)))

    def profile(self, enable=True):
        _check(lib().lrcnn_profile_enable(self.h, 1 if enable else 0))

    def profile_reset(self):
        _check(lib().lrcnn_profile_reset(self.h))

    def profile_read(self, cls, stream=None):
        ms, n, fl = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
        _check(lib().lrcnn_profile_read(self.h, cls, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl),
                                        _stream(stream)))
        return ms.value, n.value, fl.value

    def profile_kernels(self, cls, stream=None):
        """Per-kernel totals of profile class cls: [{name, launches, ms, flops, bytes, wbytes}]
        (lrcnn_profile_kernels; bytes = algorithmic HBM bytes of the launches, wbytes = of which written)."""
        buf = ctypes.create_string_buffer(1 << 16)
        _check(lib().lrcnn_profile_kernels(self.h, cls, buf, len(buf), _stream(stream)))
        out = []
        for line in buf.value.decode().splitlines():
            name, n, ms, fl, by, wb = line.rsplit(",", 5)
            out.append({"name": name, "launches": int(n), "ms": float(ms), "flops": float(fl), "bytes": float(by),
                        "wbytes": float(wb)})
        return out

    def profile_dump(self, path, stream=None):
        _check(lib().lrcnn_profile_dump(self.h, path.encode(), _stream(stream)))

    def last_launches(self):
        n = ctypes.c_longlong()
        _check(lib().lrcnn_last_launch_count(self.h, ctypes.byref(n)))
        return n.value

    def last_tc_launches(self):
        n = ctypes.c_longlong()
        _check(lib().lrcnn_last_tc_launch_count(self.h, ctypes.byref(n)))
        return n.value

    def last_simt_fallbacks(self):
        """Convolution launches of a bf16 tensor-core plan that ran on SIMT (lrcnn_last_simt_fallbacks)."""
        n = ctypes.c_longlong()
        _check(lib().lrcnn_last_simt_fallbacks(self.h, ctypes.byref(n)))
        return n.value

    def debug_capture(self, tid, buf):
        """lrcnn_debug_capture: the forward copies every band's rows of tensor tid into buf
        ([B][H][W][Cp] tensor of the plan's dtype); buf=None unregisters (parity tests only)."""
        _check(lib().lrcnn_debug_capture(self.h, tid, _ptr(buf)))


class Comm:
    """Communicator for row sharding: NCCL (one process per GPU) or in-process loopback."""

    def __init__(self, h, group=None):
        self.h, self.group = h, group

    @staticmethod
    def nccl_unique_id():
        buf = (ctypes.c_char * 128)()
        _check(lib().lrcnn_comm_nccl_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(unique_id, rank, world):
        h = ctypes.c_void_p()
        buf = (ctypes.c_char * 128).from_buffer_copy(unique_id)
        _check(lib().lrcnn_comm_init_nccl(buf, rank, world, ctypes.byref(h)))
        return Comm(h)

    @staticmethod
    def loopback(world):
        """One communicator per rank of an in-process group (ranks = host threads, one GPU)."""
        g = ctypes.c_void_p()
        _check(lib().lrcnn_comm_loopback_group(world, ctypes.byref(g)))
        out = []
        for r in range(world):
            h = ctypes.c_void_p()
            _check(lib().lrcnn_comm_init_loopback(g, r, ctypes.byref(h)))
            out.append(Comm(h, g))
        return out

    @staticmethod
    def host(group=None):
        """Host-staged communicator over a torch.distributed process group (e.g. gloo): the library
        stages halo rows / gradients through pinned host buffers and these callbacks move them with
        the group's send / recv / all_reduce (marshalling only; the library does every computation)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def _arr(ptr, nbytes):
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)), shape=(nbytes,))

        def exchange(_user, n, peer, send, host_ptr, nbytes):
            try:
                reqs = []
                for i in range(n):
                    t = torch.from_numpy(_arr(host_ptr[i], nbytes[i]))
                    p = dist.get_global_rank(group, peer[i]) if group is not None else peer[i]
                    reqs.append(dist.isend(t, p, group=group) if send[i] else dist.irecv(t, p, group=group))
                for r in reqs:
                    r.wait()
                return 0
            except Exception:   # reported by the library as LRCNN_E_NCCL
                return 1

        def allreduce(_user, buf, n):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(n,))
                dist.all_reduce(torch.from_numpy(arr), group=group)
                return 0
            except Exception:
                return 1

        cb = (HOST_EXCHANGE_FN(exchange), HOST_ALLREDUCE_FN(allreduce))
        h = ctypes.c_void_p()
        _check(lib().lrcnn_comm_init_host(rank, world, cb[0], cb[1], None, ctypes.byref(h)))
        c = Comm(h)
        c._callbacks = cb   # keep the ctypes thunks alive as long as the communicator
        return c

    def free(self):
        if self.h:
            lib().lrcnn_comm_free(self.h)
            self.h = None


class DeviceState:
    """Device buffers for one plan, allocated with torch (the caller owns all device memory)."""

    def __init__(self, plan, device="cuda"):
        import torch
        self.plan = plan
        dt = torch.bfloat16 if plan.prec == "bf16" else torch.float32
        self.dtype = dt
        self.ws = torch.empty(plan.ws_bytes, dtype=torch.uint8, device=device)
        self.params = torch.zeros(plan.n_params, dtype=dt, device=device)
        self.master = torch.zeros(plan.n_params, dtype=torch.float32, device=device)
        self.grads = torch.zeros(plan.n_params, dtype=torch.float32, device=device)
        c, cp, h, w = plan.tensor(0)
        self.x = torch.zeros((plan.B, h, w, cp), dtype=dt, device=device)
        cL, cpL, hL, wL = plan.tensor(len(plan.net["ops"]))
        self.zl = torch.zeros((plan.B, hL, wL, cpL), dtype=dt, device=device)
        self.dzl = torch.zeros_like(self.zl)
        self.labels = torch.zeros(plan.B, dtype=torch.int32, device=device)
        self.loss = torch.zeros(1, dtype=torch.float32, device=device)

    def load(self, params=None, x=None, labels=None, dzl=None):
        import torch
        if params is not None:
            flat = torch.from_numpy(self.plan.pack_params(params))
            self.master.copy_(flat)
            self.params.copy_(flat.to(self.dtype))
        if x is not None:
            self.x.copy_(torch.from_numpy(self.plan.to_nhwc(x)).to(self.dtype))
        if labels is not None:
            self.labels.copy_(torch.from_numpy(np.asarray(labels, dtype=np.int32)))
        if dzl is not None:
            self.dzl.copy_(torch.from_numpy(self.plan.to_nhwc(dzl, len(self.plan.net["ops"]))).to(self.dtype))

    def forward(self, stream=None):
        self.plan.forward_rows(self.params, self.x, self.zl, self.ws, stream)

    def backward(self, stream=None):
        self.plan.backward_rows(self.params, self.x, self.zl, self.dzl, self.grads, self.ws, stream)

    def step_grads(self, stream=None):
        self.plan.step_grads(self.params, self.grads, self.x, self.labels, self.loss, self.ws, stream)

    def step(self, lr, stream=None):
        self.plan.step(self.master, self.params, self.grads, self.x, self.labels, lr, self.loss, self.ws, stream)
