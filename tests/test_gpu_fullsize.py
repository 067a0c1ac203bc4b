"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot run a whole C2 batch or a 3600x2400 ResNet-50 image in test time, so
(R17c):
  * sampled outputs the oracle computes exactly: z^L of two images of the C2 batch (full
    224x224 forward in fp64 with bf16 storage, R17b), and the top z^L rows of a C4 image
    whose whole dependency cone (oracle/enumerate.need_sets) lies inside a 640-row strip;
  * a property that holds at any size: the row-centric 2PS-H step and the layer-wise
    (COLUMN) dataflow of the same library agree on z^L and every gradient (the method's
    invariant, "without any loss of accuracy"), here at the full batch and resolution.
Tolerance: bf16 mode 2e-2 (north_star, R18)."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from oracle import enumerate as EN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

TOL = 2e-2


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def gpu_fb(net, B, params, x, dzl, mode, **kw):
    flags = LB.FLAG_BALANCED_BANDS if mode == "2ps" else 0
    plan = LB.Plan(net, B, mode=mode, prec="bf16", flags=flags, **kw)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, dzl=dzl)
    ds.forward()
    zl = ds.zl.float().cpu()
    ds.backward()
    torch.cuda.synchronize()
    grads = ds.grads.cpu().numpy()
    zl = plan.from_nhwc(zl.numpy(), len(net["ops"]))
    g, _ = plan.unpack_grads(grads)
    del ds
    torch.cuda.empty_cache()
    return zl, g


def compare_grads(g, g_ref, tag):
    for i, (a, b) in enumerate(zip(g, g_ref)):
        if b is None:
            continue
        for k in b:
            e = rel(a[k], b[k])
            assert e <= TOL, (tag, i, k, e)


def test_c2_full_size():
    """C2 (VGG-16 224x224, batch 32, 2PS-H per pool, 4 balanced bands = bench.py's default):
    z^L of images 0 and 31 vs the oracle; z^L and all gradients vs the COLUMN dataflow."""
    net = WL.vgg16(H=224, W=224, segments="pool")
    B = 32
    params = WL.make_params(net, seed=2, bias_scale=0.05, bf16=True)
    x = WL.make_input(net, B, seed=1000, bf16=True)
    c, h, w = C.out_hw(net)[-1]
    dzl = WL.make_dzl((B, c, h, w), bf16=True)
    zl, g = gpu_fb(net, B, params, x, dzl, "2ps", n_bands=4)
    for b in (0, B - 1):
        ts, _ = C.forward(net, params, x[b:b + 1], store=C.bf16_store)
        assert rel(zl[b:b + 1], ts[-1]) <= TOL, ("zL vs oracle", b, rel(zl[b:b + 1], ts[-1]))
    zl_c, g_c = gpu_fb(net, B, params, x, dzl, "column")
    assert rel(zl, zl_c) <= TOL
    compare_grads(g, g_c, "c2 2ps-h vs column")


def test_c4_full_size():
    """C4 (ResNet-50 v1.5 3600x2400, batch 8, 2PS-H per stage, 4 balanced bands): the top z^L
    rows of image 0 vs the oracle on a 640-row strip that contains their whole dependency
    cone; z^L and all gradients vs the COLUMN dataflow at full size."""
    H, W, B = 3600, 2400, 8
    net = WL.resnet50(H=H, W=W, segments="stage")
    params = WL.make_params(net, seed=2, bias_scale=0.05, gamma_spread=0.1, bf16=True)
    x = WL.make_input(net, B, seed=1000, bf16=True)
    c, h, w = C.out_hw(net)[-1]
    dzl = WL.make_dzl((B, c, h, w), bf16=True)
    zl, g = gpu_fb(net, B, params, x, dzl, "2ps", n_bands=4)

    # oracle on a strip: rows of z^L whose dependency cone stays inside the strip are exact
    Hs = 640
    flat = WL.resnet50(H=H, W=W, segments="none")
    shp = C.out_hw(flat)
    seg = EN.segments(flat)[0]
    strip = WL.resnet50(H=Hs, W=W, segments="none")
    shp_s = C.out_hw(strip)
    j = 0
    while True:
        need = EN.need_sets(flat, shp, seg, range(0, j + 1))
        if any(rows and max(rows) >= shp_s[t][1] for t, rows in need.items()):
            break
        j += 1
    assert j >= 4, j
    ts, _ = C.forward(strip, params, x[0:1, :, :Hs, :], store=C.bf16_store)
    ref = ts[-1][:, :, :j, :]
    assert rel(zl[0:1, :, :j, :], ref) <= TOL, ("zL rows vs oracle strip", j, rel(zl[0:1, :, :j, :], ref))

    zl_c, g_c = gpu_fb(net, B, params, x, dzl, "column")
    assert rel(zl, zl_c) <= TOL
    compare_grads(g, g_c, "c4 2ps-h vs column")
