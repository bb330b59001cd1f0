"""Parity helpers: tolerances of north_star / DESIGN.md "Parity bar"."""
import numpy as np

WT_RTOL = 1e-5      # waiting times: relative (exact 0 when the oracle gives 0)
V_ATOL = 1e-5       # violation probabilities and S1: absolute
S2_RTOL = 1e-5      # S2: absolute 1e-5 * (sum wt + sum slo) of the candidate


def check_scores(s1, s2, ref, prob, wt_sum=None):
    s1 = np.asarray(s1, np.float64)
    s2 = np.asarray(s2, np.float64)
    assert np.all(np.isfinite(s1)) and np.all(np.isfinite(s2))
    d1 = np.abs(s1 - ref["s1"])
    assert d1.max(initial=0) <= V_ATOL, f"S1 max abs err {d1.max()}"
    # S2 = sum wt - sum slo; scale = sum wt + sum slo = S2 + 2 sum slo
    scale = np.abs(ref["s2"] + 2 * prob.slo.sum())
    d2 = np.abs(s2 - ref["s2"])
    assert np.all(d2 <= S2_RTOL * scale + 1e-6), f"S2 worst rel {np.max(d2 / scale)}"


def check_estimates(out, ref):
    """out: device tensors [G, count] (group-major); ref: oracle arrays [count, G]."""
    wt = out["wt"].cpu().numpy().astype(np.float64).T
    sd = out["sd"].cpu().numpy().astype(np.float64).T
    v = out["v"].cpu().numpy().astype(np.float64).T
    zero = ref["wt"] == 0
    assert np.all(wt[zero] == 0), "wt must be exactly 0 where the oracle gives 0"
    rel = np.abs(wt - ref["wt"])[~zero] / ref["wt"][~zero]
    assert rel.max(initial=0) <= WT_RTOL, f"wt max rel err {rel.max()}"
    zs = ref["sd"] == 0
    assert np.all(sd[zs] == 0), "sd must be exactly 0 where V = 0"
    rel = np.abs(sd - ref["sd"])[~zs] / ref["sd"][~zs]
    assert rel.max(initial=0) <= WT_RTOL, f"sd max rel err {rel.max()}"
    dv = np.abs(v - ref["v"])
    assert dv.max(initial=0) <= V_ATOL, f"v max abs err {dv.max()}"


def argmin_ok(gpu_index, s1_o, s2_o, prob, first=0):
    """SURVEY.md 8(c) parity rule for the argmin index (bit-exact whenever the
    oracle's objective gap exceeds the float tolerance)."""
    f1 = s1_o.astype(np.float32)
    f2 = s2_o.astype(np.float32)
    n = len(f1)
    order = np.lexsort((np.arange(n), f2, f1))
    cstar = int(order[0])
    E = np.where(f1.astype(np.float64) <= float(f1[cstar]) + V_ATOL)[0]
    g = gpu_index - first
    if len(E) == 1:
        return g == cstar, cstar
    if np.all(f1[E] == f1[cstar]):
        scale = abs(s2_o[cstar] + 2 * prob.slo.sum())
        gaps = np.abs(s2_o[E] - s2_o[cstar])
        gaps[E == cstar] = np.inf
        if gaps.min() > S2_RTOL * scale:
            return g == cstar, cstar
    return g in set(E.tolist()), cstar
