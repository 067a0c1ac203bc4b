"""GPU-side test helpers: run the CUDA path through the C-ABI with every map captured
(lrcnn_debug_capture) and return plain numpy arrays for the oracle checks."""
import numpy as np
import torch

from paper_2401_11471_b200 import lrcnn as LB


def _nchw(buf, c, images, r0=0, r1=None):
    v = buf[images][:, r0:r1, :, :c] if r1 is not None else buf[images][:, r0:, :, :c]
    return v.permute(0, 3, 1, 2).double().cpu().numpy()


def run_capture(net, B, prec, mode, params, x, dzl, flags=0, images=None, rows=None, **kw):
    """forward_rows + backward_rows with every map captured.  Returns (plan, z^L [selected images],
    grads, ts) with ts[t] = the stored map of tensor t for the selected images (rows [0, rows[t]))."""
    plan = LB.Plan(net, B, mode=mode, prec=prec, flags=flags, **kw)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, dzl=dzl)
    L = len(net["ops"])
    bufs = {}
    for t in range(1, L + 1):
        c, cp, h, w = plan.tensor(t)
        bufs[t] = torch.zeros((B, h, w, cp), dtype=ds.dtype, device=ds.x.device)
        plan.debug_capture(t, bufs[t])
    ds.forward()
    ds.backward()
    torch.cuda.synchronize()
    if prec == "bf16" and not flags & LB.FLAG_NO_TCGEN05:
        assert plan.last_simt_fallbacks() == 0
    images = list(range(B)) if images is None else images
    ts = [np.asarray(x, dtype=np.float64)[images] if rows is None else
          np.asarray(x, dtype=np.float64)[images][:, :, :rows[0]]]
    for t in range(1, L + 1):
        c = plan.tensor(t)[0]
        ts.append(_nchw(bufs[t], c, images, 0, None if rows is None else rows[t]))
    for t in range(1, L + 1):
        plan.debug_capture(t, None)
    del bufs
    g, _ = plan.unpack_grads(ds.grads.cpu().numpy())
    zl = ts[-1]
    del ds
    torch.cuda.empty_cache()
    return plan, zl, g, ts


