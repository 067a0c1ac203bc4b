"""Fused identity bottleneck forward (k_bneck_fwd): ResNet-50's conv2_x identity blocks
(t[256] -> 1x1 -> 3x3 -> 1x1 + t, 64-channel middle) run as one kernel per band that keeps t1 / t2 on
chip.  Its arithmetic equals the unfused kernels' (same K order, same epilogue), so z^L and the loss
with and without the fusion must agree BIT FOR BIT -- in every mode and band layout, including the FP
pass that stores only the 2PS cache rows of t1 (no debug capture here, so the windows path is the one
that runs) -- and the weight gradient up to the order of its fp32 atomic reductions (1e-5; a wrong
cache row read by the BP recompute would be an O(1) error).  The oracle comparison of the fused path is in test_gpu_conditioned.py
(test_resnet_stage2_full_width_fused_pointwise_backward, C4 full size)."""
import numpy as np
import pytest

import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

BENCH_FLAGS = LB.FLAG_BALANCED_BANDS | LB.FLAG_FP_MERGE | LB.FLAG_REQUIRE_TC


def _run(net, B, mode, flags, params, x, labels, **kw):
    """lrcnn_step_grads (FP, head, BP): loss, z^L, weight gradient"""
    plan = LB.Plan(net, B, mode=mode, prec="bf16", flags=flags, **kw)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, labels=labels)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ds.step_grads(stream=st)
    torch.cuda.synchronize()
    out = dict(loss=float(ds.loss), zl=ds.zl.clone(), grads=ds.grads.clone(), launches=plan.last_launches())
    del ds
    return out


def _same(f, u):
    assert f["launches"] < u["launches"], (f["launches"], u["launches"])   # the fused kernel ran
    assert torch.equal(f["zl"], u["zl"])
    assert f["loss"] == u["loss"], (f["loss"], u["loss"])
    err = float((f["grads"] - u["grads"]).abs().max() / u["grads"].abs().max())
    assert err <= 1e-5, err


@pytest.mark.parametrize("mode,kw,flags", [
    ("2ps", {"n_bands": 4}, BENCH_FLAGS),                  # bench's plan: merged FP bands, cache windows
    ("2ps", {"n_bands": 3}, LB.FLAG_REQUIRE_TC),           # one FP band per BP band
    ("2ps", {"band_rows": 1}, LB.FLAG_REQUIRE_TC),         # 1-row bands: every tile is a band edge
    ("column", {}, LB.FLAG_REQUIRE_TC),                    # no recompute: the FP stores t1 / t2 in full
    ("overl", {"n_bands": 2}, LB.FLAG_REQUIRE_TC | LB.FLAG_ALLOW_OVERLAP_EXHAUSTION),
])
def test_fused_block_bit_identical_to_unfused(mode, kw, flags):
    net = WL.resnet50(H=88, W=44, width_div=1, blocks=(3, 1, 1, 1))   # conv2_x 22 x 11: ragged tiles
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, seed=0, bf16=True)
    labels = WL.make_labels(net, B)
    _same(_run(net, B, mode, flags, params, x, labels, **kw),
          _run(net, B, mode, flags | LB.FLAG_NO_FUSE_BLOCK, params, x, labels, **kw))


def test_fused_block_full_c4_stage_bit_identical():
    """C4's band geometry (conv2_x 900 rows, 8 balanced bands, merged FP bands) on a 600-column strip
    of one image with bench's plan: fused vs unfused."""
    net = WL.resnet50(H=3600, W=600, width_div=1)
    B = 1
    params = WL.make_params(net, seed=2, bias_scale=0.05, gamma_spread=0.1, bf16=True)
    x = WL.make_input(net, B, seed=1000, bf16=True)
    labels = WL.make_labels(net, B)
    _same(_run(net, B, "2ps", BENCH_FLAGS, params, x, labels, n_bands=8),
          _run(net, B, "2ps", BENCH_FLAGS | LB.FLAG_NO_FUSE_BLOCK, params, x, labels, n_bands=8))
