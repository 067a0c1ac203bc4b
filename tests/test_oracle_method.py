"""Pins for the oracle's method layer: the brute-force enumerator against the
paper's worked examples and recursions, the CPU row-centric executor against
the column oracle (the method's invariant), negative controls, and the memory
/ FLOP formulas against the SPEC examples.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import column as C
from oracle import enumerate as EN
from oracle import rowcentric as RC
from oracle import memmodel as MM
import workloads as WL

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def chain_net(chain, H, W=5, C=1, ch=2):
    ops = []
    for i, (k, s, p) in enumerate(chain):
        ops.append(WL.conv(i, ch, k, s, p))
    return {"C": C, "H": H, "W": W, "classes": 3, "ops": ops}


# ----------------------------------------------------------------- enumerator pins
def test_fig4_forward_split():
    g = gold("paper_examples.json")
    for key in ("fig4a", "fig4b"):
        e = g[key]
        sizes = EN.forward_split([tuple(c) for c in e["chain"]], e["H"], e["in_split"])
        assert sizes == e["sizes"], key


def test_c1_band_table():
    g = gold("c1_bands.json")
    for key in ("p1", "p0"):
        e = g[key]
        net = WL.tiny3(p=e["p"])
        seg = EN.segments(net)[0]
        shp = C.out_hw(net)
        E = EN.band_ends(shp[3][1], band_rows=e["band_rows"])
        two = EN.enumerate_2ps(net, seg, E)
        ov = EN.enumerate_overl(net, seg, E)
        # x is the segment input: its 2PS "computed rows" are the rows read by band r beyond band r-1
        xr = []
        prev = 0
        for r in range(len(E)):
            need = EN.need_sets(net, shp, seg, range(0, E[r]))[0]
            end = max(need) + 1 if r < len(E) - 1 else shp[0][1]
            xr.append([prev, end])
            prev = end
        assert xr == e["x_2ps"]
        assert [list(b[0]) for b in ov] == e["x_overl"]
        if "z1_2ps" in e:
            assert [[b[1][1], b[1][2]] for b in two] == e["z1_2ps"]
            assert [[b[2][1], b[2][2]] for b in two] == e["z2_2ps"]
            assert [[b[3][1], b[3][2]] for b in two] == e["z3"]
            for b in two[1:]:
                assert b[1][1] - b[1][0] == e["cache"] and b[2][1] - b[2][0] == e["cache"]


def test_2ps_recursions_eq11_13_14():
    """Divisible chains: band heights equal Eq. (11) (first row), Eq. (13) (middle), Eq. (14) (last)."""
    rng = np.random.default_rng(5)
    for _ in range(30):
        L = int(rng.integers(1, 5))
        chain = [(int(rng.choice([2, 3, 5])), 1, int(rng.integers(0, 2))) for _ in range(L)]
        chain = [(k, s, min(p, (k - 1) // 2)) for k, s, p in chain]
        hL, N = int(rng.integers(2, 5)), int(rng.integers(2, 5))
        H_out = hL * N
        # input height giving exactly H_out at the output
        h = H_out
        for k, s, p in reversed(chain):
            h = (h - 1) * s + k - 2 * p
        net = chain_net(chain, h, W=24)
        seg = EN.segments(net)[0]
        E = EN.band_ends(H_out, band_rows=hL)
        two = EN.enumerate_2ps(net, seg, E)
        shp = C.out_hw(net)
        # the recursions assume no band end is clamped at H (padding reaching the
        # bottom edge before the last band); skip such draws
        if any(two[r][l][2] >= shp[l][1] for r in range(N - 1) for l in range(1, L)):
            continue
        # first row, Eq. (11): H_1^l = (H_1^{l+1}-1)s+k-p  (height of tensor l in band 1)
        H1 = hL
        for l in range(L - 1, 0, -1):
            k, s, p = chain[l]
            H1 = (H1 - 1) * s + k - p
            assert two[0][l][2] - two[0][l][1] == H1
        # middle rows, Eq. (13): H_r^l = (H_r^{l+1}-1)s+s  (= newly computed rows)
        for r in range(1, N - 1):
            Hr = hL
            for l in range(L - 1, 0, -1):
                k, s, p = chain[l]
                Hr = (Hr - 1) * s + s
                assert two[r][l][2] - two[r][l][1] == Hr
        # last row, Eq. (14): H_N^l = (H_N^{l+1}-1)s+s-p
        HN = hL
        for l in range(L - 1, 0, -1):
            k, s, p = chain[l]
            HN = (HN - 1) * s + s - p
            assert two[N - 1][l][2] - two[N - 1][l][1] == HN
        # cache rows c = k - s
        for r in range(1, N):
            for l in range(1, L):
                k, s, p = chain[l]
                assert two[r][l][1] - two[r][l][0] == k - s


def test_overl_examples_and_eq15():
    g = gold("paper_examples.json")
    e = g["overl_one_conv"]
    net = chain_net([tuple(c) for c in e["chain"]], e["H"])
    ov = EN.enumerate_overl(net, EN.segments(net)[0], e["E"])
    assert [list(b[0]) for b in ov] == e["ext_in"]
    assert ov[0][0][1] - ov[1][0][0] == e["o0"]
    e = g["overl_two_conv"]
    net = chain_net([tuple(c) for c in e["chain"]], e["H"])
    shp = C.out_hw(net)
    E = EN.band_ends(shp[-1][1], n_bands=e["N"])
    ov = EN.enumerate_overl(net, EN.segments(net)[0], E)
    assert ov[0][0][1] - ov[1][0][0] == e["o0"] == MM.overlap_chain([tuple(c) for c in e["chain"]])[0]
    assert all(b[0][1] - b[0][0] == e["ext_rows"] for b in ov)
    # Eq. (15) on random k>=s chains: overlap of consecutive extended ranges at every tensor
    rng = np.random.default_rng(9)
    for _ in range(40):
        L = int(rng.integers(1, 5))
        chain = []
        for _ in range(L):
            s = int(rng.integers(1, 3))
            k = int(rng.integers(s, 5))
            chain.append((k, s, 0))
        h = 60
        net = chain_net(chain, h, W=60)
        try:
            shp = C.out_hw(net)
        except ValueError:
            continue
        if shp[-1][1] < 4:
            continue
        E = EN.band_ends(shp[-1][1], n_bands=2)
        ov = EN.enumerate_overl(net, EN.segments(net)[0], E)
        o = MM.overlap_chain(chain)
        for t in range(L):
            assert ov[0][t][1] - ov[1][t][0] == o[t], (chain, t)


# ----------------------------------------------------------------- method invariant
def _nets():
    yield WL.tiny3(p=1, H=16, W=9)
    yield WL.tiny3(p=0, H=17, W=9)
    yield WL.vgg16(H=64, W=32, width_div=16)
    yield WL.vgg16(H=64, W=32, width_div=16, segments="pool")
    yield {"C": 3, "H": 23, "W": 10, "classes": 4,
           "ops": [WL.conv(0, 4, 7, 2, 3, epi="affine"), WL.maxpool(1, 3, 2, 1),
                   WL.conv(2, 3, 1, 1, 0, epi="affine"), WL.conv(3, 3, 3, 1, 1, epi="affine"),
                   WL.conv(4, 4, 1, 1, 0, epi="affine", res=2, seg_end=True),
                   WL.conv(5, 3, 1, 1, 0, epi="affine"), WL.conv(6, 3, 3, 2, 1, epi="affine"),
                   WL.conv(5, 4, 1, 2, 0, epi="affine", relu=False),
                   WL.conv(7, 4, 1, 1, 0, epi="affine", res=8)]}


def _rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("mode", ["2ps", "overl"])
def test_rowcentric_equals_column(mode):
    """Row-centric (any N, segments) == column at <= 1e-12 in fp64 (SURVEY 8(c) pin 5)."""
    for net in _nets():
        B = 2
        prm = WL.make_params(net, seed=2, bias_scale=0.2, gamma_spread=0.2)
        x = WL.make_input(net, B)
        lab = WL.make_labels(net, B)
        _, loss_c, g_c, hg_c, ts = C.step(net, prm, x, lab, 0.1)
        for kw in ({"n_bands": 1}, {"n_bands": 2}, {"band_rows": 1}, {"band_rows": 3}):
            plan = RC.Plan(net, mode, **kw)
            _, loss_r, g_r, hg_r, zl = RC.step(plan, prm, x, lab, 0.1)
            assert zl.shape == ts[-1].shape
            assert _rel(zl, ts[-1]) <= 1e-12
            assert abs(loss_r - loss_c) <= 1e-12 * abs(loss_c)
            for a, b in zip(g_r, g_c):
                if b is None:
                    continue
                for k in b:
                    assert _rel(a[k], b[k]) <= 1e-12, (net.get("name"), mode, kw, k)
            if kw == {"n_bands": 1} and len(plan.segs) == 1:
                assert np.array_equal(zl, ts[-1])          # N=1 is bitwise the column dataflow


def test_negative_controls():
    """Each must differ from the column oracle by >> tolerance (SURVEY 8(c) pin 6)."""
    net = WL.tiny3(p=1, H=16, W=9)
    B = 1
    prm = WL.make_params(net, seed=2, bias_scale=0.2)
    x = WL.make_input(net, B)
    ts, aux = C.forward(net, prm, x)
    dzl = WL.make_dzl(ts[-1].shape)
    g_c, _ = C.backward(net, prm, ts, aux, dzl)
    plan = RC.Plan(net, "2ps", band_rows=4)
    # sharing disabled -> padding redundancy at interior cuts
    zl, ck, ac = RC.forward(plan, prm, x, share=False)
    assert _rel(zl, ts[-1]) > 1e-2
    # 2PS without the delta carry
    zl, ck, ac = RC.forward(plan, prm, x)
    g, _ = RC.backward(plan, prm, ck, ac, dzl, carry_on=False)
    assert _rel(g[0]["w"], g_c[0]["w"]) > 1e-2
    # OverL with the paper's "average the redundant times" on top of disjoint ownership
    plan = RC.Plan(net, "overl", band_rows=4)
    zl, ck, ac = RC.forward(plan, prm, x)
    g, _ = RC.backward(plan, prm, ck, ac, dzl, overl_average=True)
    assert _rel(g[0]["w"], g_c[0]["w"]) > 1e-2


def test_trajectory_20_steps():
    """20 SGD iterations: row-centric losses track the column trajectory <= 1e-7."""
    net = WL.tiny3(p=1, H=12, W=8)
    B = 2
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    pc = pr = WL.make_params(net, seed=2, bias_scale=0.1)
    plan = RC.Plan(net, "2ps", band_rows=3)
    for _ in range(20):
        pc, lc, _, _, _ = C.step(net, pc, x, lab, 0.5)
        pr, lr_, _, _, _ = RC.step(plan, pr, x, lab, 0.5)
        assert abs(lc - lr_) <= 1e-7 * abs(lc)


# ----------------------------------------------------------------- memory / FLOP formulas
def test_memmodel_examples():
    g = gold("paper_examples.json")
    e = g["omega_example"]
    assert MM.omega_bp(e["rho"], e["N"]) == e["bp"] and MM.omega_fp(e["rho"], e["N"]) == e["fp"]
    e = g["solve_example"]
    assert MM.solve_n(e["rho"], 0, e["M"], "bp") == e["n_bp"] and MM.solve_n(e["rho"], 0, e["M"], "fp") == e["n_fp"]
    e = g["tau_example"]
    net = {"C": e["cin"], "H": e["Hout"] + 2, "W": e["Wout"] + 2, "classes": 2,
           "ops": [WL.conv(0, e["cout"], e["k"], 1, 0)]}
    assert MM.tau(net, e["B"]) == e["tau"]
    # Eq. (3) equals the bytes the column oracle stores (every op output)
    net = WL.vgg16(H=32, W=32, width_div=8)
    ts, _ = C.forward(net, WL.make_params(net), WL.make_input(net, 2))
    assert MM.omega(net, 2) == sum(t.size for t in ts[1:])


def test_executed_flops_2ps_and_overl():
    """2PS executes exactly tau per sweep; OverL executes tau + iota with iota from Eq. (15)."""
    chain = [(3, 1, 0), (3, 1, 0), (3, 1, 0)]
    net = chain_net(chain, 50, W=10, ch=3)
    for N in (2, 3, 4):
        p2 = RC.Plan(net, "2ps", n_bands=N)
        assert MM.executed_fwd_flops(p2, 2) == MM.tau(net, 2)
        po = RC.Plan(net, "overl", n_bands=N)
        o = MM.overlap_chain(chain)
        assert MM.executed_fwd_flops(po, 2) == MM.tau(net, 2) + MM.iota(net, 2, N, o)
