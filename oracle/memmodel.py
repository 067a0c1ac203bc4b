"""Memory and FLOP formulas of the paper -- TEST INFRASTRUCTURE ONLY.

  omega       Eq. (3)  Omega = sum_l B H^l W^l C^l
  omega_fp    Eq. (7)  Omega_FP(N) = max_{l<L} rho^l/N + rho^L
  omega_bp    Eq. (8)  Omega_BP(N) = sum_{l<L} rho^l/N + rho^L
  solve_n     Eqs. (9)-(10): min N s.t. Omega(N) + xi < M
  tau         tau = sum_l 2 k^2 B C^{l-1} C^l H^l W^l
  overlap     Eq. (15): o^l = (o^{l+1}-1) s^{l+1} + k^{l+1}, o^L=0
  iota        iota = sum_l 2 k^2 B (N-1) C^{l-1} C^l o^l W^l
  executed_flops  FLOPs a row-centric plan actually executes, counted band by band from
                  the enumerator (independent of the closed forms above).
"""
from oracle.column import out_hw


def omega(net, B):
    """Eq. (3) over every op output tensor (conv, pool, add), in elements."""
    shp = out_hw(net)
    return sum(B * c * h * w for (c, h, w) in shp[1:])


def rho_list(net, B):
    shp = out_hw(net)
    return [B * c * h * w for (c, h, w) in shp[1:]]


def omega_fp(rho, N):
    return max(r / N for r in rho[:-1]) + rho[-1]


def omega_bp(rho, N):
    return sum(r / N for r in rho[:-1]) + rho[-1]


def solve_n(rho, xi, M, phase, n_max=4096):
    f = omega_fp if phase == "fp" else omega_bp
    for n in range(1, n_max + 1):
        if f(rho, n) + xi < M:
            return n
    raise ValueError("infeasible-budget")


def tau(net, B):
    """Forward conv FLOPs (2 per MAC) of the whole net."""
    shp = out_hw(net)
    t = 0
    for i, op in enumerate(net["ops"]):
        if op["kind"] == "conv":
            cin = shp[op["src"]][0]
            c, h, w = shp[i + 1]
            t += 2 * op["k"] ** 2 * B * cin * c * h * w
    return t


def overlap_chain(chain):
    """Eq. (15) for a chain [(k,s,p), ...]: total overlap o^l at every tensor l=0..L (o^L = 0)."""
    L = len(chain)
    o = [0] * (L + 1)
    for l in range(L - 1, -1, -1):
        k, s, _ = chain[l]
        o[l] = (o[l + 1] - 1) * s + k
    return o


def iota(net, B, N, o):
    """Paper's redundant-overlap FLOPs for OverL with N rows; o[t] = overlap at tensor t."""
    shp = out_hw(net)
    t = 0
    for i, op in enumerate(net["ops"]):
        if op["kind"] == "conv":
            cin = shp[op["src"]][0]
            c, h, w = shp[i + 1]
            t += 2 * op["k"] ** 2 * B * (N - 1) * cin * c * o[i + 1] * w
    return t


def executed_fwd_flops(plan, B):
    """Conv FLOPs of one row-centric forward sweep, counted from the enumerated band rows."""
    net, shp = plan.net, plan.shp
    tot = 0
    for s, (seg_in, ids, out) in enumerate(plan.segs):
        E, bands = plan.bands[s]
        for r, band in enumerate(bands):
            for i in ids:
                op = net["ops"][i]
                if op["kind"] != "conv":
                    continue
                if plan.mode == "overl":
                    lo, hi = band[i + 1]
                    if i + 1 == out:
                        lo, hi = (E[r - 1] if r else 0), E[r]
                    rows = hi - lo
                else:
                    _, a, b = band[i + 1]
                    rows = b - a
                cin = shp[op["src"]][0]
                c, h, w = shp[i + 1]
                tot += 2 * op["k"] ** 2 * B * cin * c * rows * w
    return tot
