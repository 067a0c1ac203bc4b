"""Decision-conditioned oracle checks (test infrastructure; reading R17d).

ReLU masks and max-pool argmax are integer decisions.  When two candidates differ by less than
the accumulation-order rounding of the kernel (fp32 sums in a different order than the fp64 oracle,
bf16 storage), both decisions are correct, and one flipped decision early in a deep bf16 net
cascades into gradients the oracle cannot reproduce element by element (R17c).  So the deep /
full-size tests split the comparison:

  1. VALIDITY of every stored map the GPU produced (captured with lrcnn_debug_capture): each op is
     recomputed by the fp64 oracle from the GPU's own stored inputs and must match the GPU's stored
     output within the tolerance -- a flipped ReLU decision is only accepted where the oracle's
     pre-activation is within rounding of zero, and a max-pool output must equal the oracle's
     window maximum exactly (a max of the same stored values);
  2. EXACTNESS of the backward given those (validated) decisions: the oracle's fp64 column backward
     runs on the GPU's stored maps (ReLU gates from them, argmax recomputed from them by the
     oracle's own lowest-index rule) and every GPU gradient must match it within the tolerance.

z^L is always ALSO compared with the plain, unconditioned oracle forward.  Nothing here imports the
CUDA path: the captured maps arrive as plain numpy arrays."""
import numpy as np

import oracle as O
from oracle import column as C
from oracle import enumerate as EN


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _pads(op):
    p = op.get("p", 0)
    return (p, p, p, p)


def validate_forward(net, params, ts, store, tol, rows=None):
    """Step 1.  ts[t] = the GPU's stored map of tensor t (NCHW fp64; ts[0] = the input).  For every
    op, the oracle output from the GPU's inputs, rounded with the kernel's storage model `store`,
    must match ts[t] within tol (max-abs over the tensor's max-abs); max-pool outputs exactly.
    rows: optional {t: (r0, r1)} -- compare only those rows (strips whose lower rows are cut off).
    Returns ({t: rel error}, aux) with aux the oracle's conv raw outputs / argmax (for backward)."""
    errs, aux = {}, []
    for i, op in enumerate(net["ops"]):
        t = i + 1
        src = ts[op["src"]]
        if op["kind"] == "conv":
            res = ts[op["res"]] if op["res"] >= 0 else None
            ref, c = C.conv_op_fwd(op, params["convs"][i], src, res, _pads(op))
            aux.append(c)
        elif op["kind"] == "maxpool":
            ref, am = O.maxpool_fwd(src, op["k"], op["s"], _pads(op))
            aux.append(am)
        elif op["kind"] == "bn":   # batch statistics of the GPU's stored full input map
            mean, var = C.bn_stats(src)
            res = ts[op["res"]] if op["res"] >= 0 else None
            ref = C.bn_apply(params["convs"][i], src, mean, var, res, op["relu"])
            aux.append((mean, var))
        else:
            a = src + ts[op["res"]]
            ref = np.maximum(a, 0.0) if op["relu"] else a
            aux.append(None)
        ref = store(ref)
        got = ts[t]
        if rows is not None and t in rows:
            r0, r1 = rows[t]
            ref, got = ref[:, :, r0:r1], got[:, :, r0:r1]
        if op["kind"] == "maxpool":
            assert np.array_equal(got, ref), ("max-pool output is not the window max of its stored input", i)
            errs[t] = 0.0
        else:
            errs[t] = rel(got, ref)
            assert errs[t] <= tol, ("stored map of op", i, errs[t])
    return errs, aux


def conditioned_grads(net, params, ts, aux, dzl):
    """Step 2: the oracle's fp64 column backward on the GPU's stored maps."""
    grads, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
    return grads


def compare_grads(g, g_ref, tol, tag=""):
    """rel(T) <= tol for every gradient tensor; on failure the message lists the five worst."""
    errs = []
    for i, (a, b) in enumerate(zip(g, g_ref)):
        if b is None:
            continue
        for k in b:
            errs.append((rel(a[k], b[k]), i, k))
    errs.sort(reverse=True)
    assert not errs or errs[0][0] <= tol, (tag, "worst (rel, op, param):", errs[:5])
    return errs[0][0] if errs else 0.0


def strip_rows(net, zl_rows):
    """{t: (0, max needed row + 1)}: rows of every tensor in the dependency cone of z^L rows
    [0, zl_rows) (oracle.enumerate.need_sets on the whole net, no segments)."""
    flat = dict(net, ops=[dict(o, seg_end=False) for o in net["ops"]])
    shp = C.out_hw(flat)
    seg = EN.segments(flat)[0]
    need = EN.need_sets(flat, shp, seg, range(0, zl_rows))
    return {t: (0, max(r) + 1) for t, r in need.items() if r}
