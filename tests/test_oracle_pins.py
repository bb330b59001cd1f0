"""Pins of the CPU oracle against what the paper / SPEC / mathematics fix.

None of these re-types the oracle's formulas: each expected value comes from
a SPEC worked example, a hand derivation stored under tests/golden/ (with its
citation), a closed form, a textbook algorithm (SPT, Moore-Hodgson), a
library-defined order (itertools), published known-answer vectors (Random123)
or a statistical law (CLT).  See DESIGN.md "Oracle pins".
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle as O
from tests.handmade import hand_problem, rank_of
from workloads.synth import make_config, make_problem, make_random_problem, balanced_row

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Philox (P13)
def test_philox_random123_kat():
    # Random123 kat_vectors, philox4x32_10 (Salmon et al. SC'11).
    kat = [
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for ctr, key, want in kat:
        assert tuple(int(x) for x in O.philox4x32_10(ctr, key)) == want


# ---------------------------------------------------------------- rows (Eq. 6)
@pytest.mark.parametrize("T", [1, 2, 3, 4, 5, 6, 7])
def test_enum_rows_are_lexicographic_permutations(T):
    for c, perm in enumerate(itertools.permutations(range(T))):
        assert tuple(O.enum_row(c, T)) == perm


@pytest.mark.parametrize("T", [1, 2, 5, 71, 300, 1055])
def test_random_rows_are_permutations(T):
    for c in [0, 1, 2, 12345, 2**33 + 7]:
        row = O.random_row(1, c, T)
        assert sorted(row.tolist()) == list(range(T))


def test_random_rows_uniform_over_permutations():
    # Fisher-Yates with independent uniform indices gives every permutation
    # probability 1/T!; chi-square over the 24 permutations of T = 4.
    T, N = 4, 24000
    counts = {}
    for c in range(N):
        key = tuple(O.random_row(7, c, T))
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 24
    chi2 = sum((v - N / 24) ** 2 / (N / 24) for v in counts.values())
    assert stats.chi2.sf(chi2, 23) > 1e-3
    # the seed changes the stream
    assert [tuple(O.random_row(1, c, 20)) for c in range(5)] != \
           [tuple(O.random_row(2, c, 20)) for c in range(5)]


@pytest.mark.parametrize("T", [200, 300])
def test_random_rows_first_position_uniform(T):
    # row[0] after the whole Fisher-Yates is the first step's target j_0, which
    # must be uniform on [0, T): chi-square over 60k rows, both draw widths
    # (16-bit halves for T <= 256, 32-bit words above; R10)
    N = 60000
    first = np.array([O.random_row(3, c, T)[0] for c in range(N)])
    counts = np.bincount(first, minlength=T)
    chi2 = float(((counts - N / T) ** 2 / (N / T)).sum())
    assert stats.chi2.sf(chi2, T - 1) > 1e-3


@pytest.mark.parametrize("T", [2, 3, 71, 255, 256])
def test_random_row_16bit_draw_is_multiply_shift_of_philox_R10(T):
    # The oracle's first Fisher-Yates step for T <= 256 is exactly
    # j0 = floor(u * T / 2^16), u = the low 16 bits of word 0 of the KAT-pinned
    # Philox block (ctr = (0, lo32 c, hi32 c, 'QLM\0'), key = seed): row[0] == j0
    # after the whole shuffle (later steps never touch position 0)
    seed = 0x1234_5678_9ABC
    for c in range(0, 4000, 7):
        w = O.philox4x32_10([0, c & 0xFFFFFFFF, c >> 32, 0x514C4D00], [seed & 0xFFFFFFFF, seed >> 32])
        u = int(w[0]) & 0xFFFF
        assert O.random_row(seed, c, T)[0] == (u * T) >> 16


def test_random_row_16bit_draw_bias_exact_R10():
    # Exact bias of R10's 16-bit multiply-shift draws (no rejection): for every
    # step range m = T - i in [2, 256], enumerate all 2^16 draws u and count the
    # preimages of each index j = floor(u m / 2^16).  Each j gets floor(2^16/m)
    # or ceil(2^16/m) draws, so a step's index probability is within a factor
    # (ceil or floor)(2^16/m) * m / 2^16 of 1/m: relative bias <= m / 2^16,
    # largest at m = 255 (1/257 = 0.389 %), zero when m divides 2^16.
    u = np.arange(1 << 16, dtype=np.int64)
    worst = 0.0
    for m in range(2, 257):
        cnt = np.bincount((u * m) >> 16, minlength=m)
        fl, ce = (1 << 16) // m, -(-(1 << 16) // m)
        assert cnt.sum() == 1 << 16 and set(np.unique(cnt)) <= {fl, ce}
        assert int(cnt.max()) * m - (1 << 16) < m and (1 << 16) - int(cnt.min()) * m < m
        worst = max(worst, (int(cnt.max()) - int(cnt.min())) * m / (1 << 16))
    assert worst == 255 / 65536
    # whole-row consequence (DESIGN R10): a C3 row (T = 71) has probability
    # within [0.9830, 1.0203] x 1/71!; T = 256 within [0.8056, 1.3204] x 1/256!
    for T, lo_b, hi_b in ((71, 0.9830, 1.0203), (256, 0.8056, 1.3204)):
        lo = math.prod(((1 << 16) // m) * m / (1 << 16) for m in range(2, T + 1))
        hi = math.prod((-(-(1 << 16) // m)) * m / (1 << 16) for m in range(2, T + 1))
        assert lo_b <= lo < 1.0 < hi <= hi_b and abs(lo - lo_b) < 1e-4 and abs(hi - hi_b) < 1e-4


# ---------------------------------------------------------------- SPEC worked examples
def test_wait_mean_and_std_S279():
    g = gold("spec_examples.json")["wait_S279"]
    # group A (25 requests) ahead of group B, same model = resident, one queue
    p = hand_problem([0, 0], [g["requests_ahead"], 1], g["mu"], g["sigma"] ** 2, [1e9, 5.5],
                     theta=g["theta"])
    o = O.Oracle(p)
    e = o.estimate([0, 1])
    assert e["wt"][1] == pytest.approx(g["mean"], abs=1e-12)
    assert math.sqrt(e["V"][1]) == pytest.approx(g["std"], abs=1e-12)
    assert e["wt"][0] == 0.0 and e["V"][0] == 0.0       # empty queue ahead
    # slo = mean + 1 std -> Phi-bar(1) (textbook)
    tb = dict((z, v) for z, v in gold("phibar_textbook.json")["values"])
    s1, s2, _ = o.score([0, 1])
    assert s1 * 26 == pytest.approx(tb[1.0], abs=1e-14)   # n_B = 1 of 26 requests


def test_serve_time_S306():
    g = gold("spec_examples.json")["serve_S306"]
    p = hand_problem([0, 0], [g["n"], 1], g["mu"], 0.0, 100.0, theta=g["theta"])
    assert O.Oracle(p).estimate([0, 1])["wt"][1] == pytest.approx(g["serve_time"], abs=1e-12)


def test_transition_tail_S287_S296():
    g1 = gold("spec_examples.json")["decode_S287"]
    g2 = gold("spec_examples.json")["completion_S296"]
    # X group (8 s of work) then a Y group: the Y group waits W_X + C_X - W_X + swap
    # = 8 + P + max_out*eps*d + S  (Eq. 1/4/10, readings R1/R2)
    S = 20.0
    p = hand_problem([0, 1], [40, 1], 200.0, 0.0, 1000.0, theta=1000.0, prefill=g2["prefill"],
                     eps=g1["eps"], dtok=g1["d"], max_out=g1["max_out"], swap=S, M=2)
    e = O.Oracle(p).estimate([0, 1])
    assert e["wt"][1] == pytest.approx(8.0 + g2["completion"] + S, abs=1e-9)
    assert g2["completion"] == pytest.approx(g2["prefill"] + g1["decode"])
    # reverse order: the Y group is first in a queue whose resident is X -> swap only (R4)
    e = O.Oracle(p).estimate([1, 0])
    assert e["wt"][1] == pytest.approx(S, abs=0)
    # and the X group behind it pays Y's tail + swap back
    assert e["wt"][0] == pytest.approx(S + 1 * 200.0 / 1000.0 + g2["completion"] + S,
                                       abs=1e-9)


def test_slack_and_step_violation_S315():
    g = gold("spec_examples.json")["slack_S315"]
    # A: 8 s of work (n=40, mu=200, Theta=1000), sigma = 0 -> V = 0 -> step function
    p = hand_problem([0, 0], [40, 10], 200.0, 0.0, [g["slo_A"], g["slo_B"]], theta=1000.0)
    o = O.Oracle(p)
    e = o.estimate([0, 1])
    assert e["wt"][1] == g["predicted_B"]
    assert g["slo_B"] - e["wt"][1] == g["slack_B"]
    s1, s2, n_over = o.score([0, 1])
    assert s1 == 10 / 50 and n_over == 1
    assert s2 == (0 - g["slo_A"]) + (g["predicted_B"] - g["slo_B"])
    # boundary: ttft == slo is met
    p2 = hand_problem([0, 0], [40, 10], 200.0, 0.0, [10.0, 8.0], theta=1000.0)
    assert O.Oracle(p2).score([0, 1])[0] == 0.0


def test_objective_tie_S375():
    g = gold("spec_examples.json")["tie_S375"]
    # serve 5 s each: n = 25, mu = 200, Theta = 1000, sigma = 0
    p = hand_problem([0, 0], [25, 25], 200.0, 0.0, g["slos"], theta=1000.0)
    o = O.Oracle(p)
    r = o.score_range(O.ENUM, 0, 2)
    assert list(r["s2"]) == [g["objective"], g["objective"]]
    assert O.argmin_key(r["s1"], r["s2"]) == 0          # tie -> lowest index (tighter first)
    e = o.estimate([0, 1])
    assert list(e["wt"] - np.asarray(g["slos"])) == g["penalties_tighter_first"]


# ---------------------------------------------------------------- hand-derived goldens
def test_xyx_example_P6():
    g = gold("p6_xyx.json")
    p = hand_problem([0, 1, 0], 25, 200.0, 0.0, 100.0, theta=1000.0, prefill=0.5, eps=1.0,
                     dtok=0.5, max_out=1.0, swap=20.0, M=2)
    o = O.Oracle(p)
    r = o.score_range(O.ENUM, 0, 6)
    for k, want in g["orders"].items():
        k = int(k)
        assert rank_of(want["order"]) == k
        assert list(o.estimate(want["order"])["wt"]) == want["wt_by_group"]
        assert r["s2"][k] == want["S2"]
        assert r["s1"][k] == 0.0
    assert O.argmin_key(r["s1"], r["s2"]) == g["argmin"]


def test_c1_golden_P7():
    g = gold("p7_c1.json")
    p = make_config("C1")
    o = O.Oracle(p)
    r = o.score_range(O.ENUM, 0, 24)
    assert O.argmin_key(r["s1"], r["s2"]) == g["argmin"] == rank_of(g["argmin_order"])
    e = o.estimate(g["argmin_order"])
    np.testing.assert_allclose(e["wt"], g["argmin_wt_by_group"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(e["V"], g["argmin_V_by_group"], rtol=0, atol=1e-12)
    assert r["s1"][12] == g["argmin_S1"]
    assert r["s2"][12] == pytest.approx(g["argmin_S2"], abs=1e-12)
    assert rank_of(g["runner_up_order"]) == g["runner_up"]
    s1_ru = 40 * 0.5 * math.erfc(3 / math.sqrt(0.85) / math.sqrt(2)) / 125
    assert r["s1"][13] == pytest.approx(s1_ru, rel=1e-12)
    assert r["s2"][13] == pytest.approx(g["runner_up_S2"], abs=1e-12)
    assert r["s1"].max() == pytest.approx(g["worst_S1"], abs=1e-15)
    assert r["s1"][rank_of(g["worst_order"])] == pytest.approx(g["worst_S1"], abs=1e-15)


def test_phibar_textbook_P16():
    for z, want in gold("phibar_textbook.json")["values"]:
        assert O.violation(0.0, 1.0, z) == pytest.approx(want, abs=2e-16 + 1e-14 * want)
        # scale invariance: only the z-score matters
        assert O.violation(100.0, 4.0, 100.0 + 2 * z) == pytest.approx(want, abs=1e-14)
    assert O.violation(0.0, 1.0, 8.5) == 0.0          # clamp (R9)
    assert O.violation(0.0, 1.0, -8.5) == 1.0
    assert 0.0 < O.violation(0.0, 1.0, 7.9) < 1e-14
    assert O.violation(5.0, 0.0, 5.0) == 0.0          # V = 0: met iff wt <= slo
    assert O.violation(5.0, 0.0, 4.999) == 1.0


# ---------------------------------------------------------------- closed forms
def test_identical_groups_closed_form_P8():
    # Eq. 2/3 with q-1 identical groups ahead: wt = s*n*mu/Theta, V = s*n*sigma^2/Theta^2
    G, n, mu, var, th = 40, 37, 311.0, 5000.0, 1700.0
    p = hand_problem([0] * G, n, mu, var, 1e6, theta=th)
    rng = np.random.default_rng(3)
    order = rng.permutation(G)
    e = O.Oracle(p).estimate(order)
    for s, i in enumerate(order):
        assert e["wt"][i] == pytest.approx(s * n * mu / th, rel=1e-13, abs=0)
        assert e["V"][i] == pytest.approx(s * n * var / th**2, rel=1e-13, abs=0)
        assert e["pos"][i] == s and e["queue"][i] == 0


def test_insight3_interleaving_costs_extra_transitions():
    # PAPER.md L351-357 (Insight 3): interleaved X,Y,X,Y vs grouped X,X,Y,Y costs
    # the extra model transitions.  Each transition costs tail + S here: Eq. 10
    # charges the completion C = W + tail of the group ahead at a model boundary
    # (reading R1, P:L705 / P:L743-746).  SPEC.md charges S
    # only; that is a recorded divergence from SPEC (R1), not a
    # SPEC pin.
    tail, S = 1.0, 20.0
    p = hand_problem([0, 1, 0, 1], 25, 200.0, 0.0, 1e4, theta=1000.0, prefill=0.5, eps=1.0,
                     dtok=0.5, max_out=1.0, swap=S, M=2)
    o = O.Oracle(p)
    inter = o.estimate([0, 1, 2, 3])["wt"]   # X1 Y1 X2 Y2: 3 transitions
    group = o.estimate([0, 2, 1, 3])["wt"]   # X1 X2 Y1 Y2: 1 transition
    assert inter[3] - group[3] == pytest.approx(2 * (tail + S), abs=1e-12)
    assert inter.sum() - group.sum() == pytest.approx(4 * (tail + S), abs=1e-12)


def _brute(o, G):
    return o.score_range(O.ENUM, 0, math.factorial(G))


@pytest.mark.parametrize("seed", range(12))
def test_spt_minimises_total_penalty_P9(seed):
    # sigma = 0, one queue, one model: S2 = sum_j wt_j - sum slo is total start time,
    # minimised by shortest-processing-time order (textbook 1||sum C_j).
    rng = np.random.default_rng(100 + seed)
    G = int(rng.integers(2, 8))
    n = rng.integers(1, 300, G)
    mu = rng.uniform(10, 500, G)
    slo = rng.uniform(1, 100, G)
    p = hand_problem([0] * G, n, mu, 0.0, slo, theta=1234.0)
    a = np.sort(n * mu / 1234.0)
    spt = sum(a[k] * (G - 1 - k) for k in range(G)) - slo.sum()
    r = _brute(O.Oracle(p), G)
    assert r["s2"].min() == pytest.approx(spt, rel=1e-12, abs=1e-9)


def _moore_hodgson(p_times, due):
    order = np.argsort(due, kind="stable")
    sched, t, late = [], 0.0, 0
    for j in order:
        sched.append(j)
        t += p_times[j]
        if t > due[j]:
            k = max(sched, key=lambda x: p_times[x])
            sched.remove(k)
            t -= p_times[k]
            late += 1
    return late


@pytest.mark.parametrize("seed", range(12))
def test_moore_hodgson_minimises_violations_P10(seed):
    # sigma = 0, equal n: S1 * G = #late; late iff start > slo iff C > slo + W
    # (due dates slo + W, textbook 1||sum U_j).
    rng = np.random.default_rng(200 + seed)
    G = int(rng.integers(2, 8))
    mu = rng.uniform(10, 500, G)
    p_times = 50 * mu / 1000.0
    slo = rng.uniform(0.5, 1.0, G) * p_times.sum() * rng.uniform(0.2, 1.0)
    p = hand_problem([0] * G, 50, mu, 0.0, slo, theta=1000.0)
    r = _brute(O.Oracle(p), G)
    assert round(r["s1"].min() * G, 9) == _moore_hodgson(p_times, slo + p_times)


# ---------------------------------------------------------------- invariants (P11)
@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_invariants_app_b(cfg):
    p = make_config(cfg)
    o = O.Oracle(p)
    for c in range(40):
        row = O.random_row(1, c, p.T)
        e = o.estimate(row)
        for q in range(p.Q):
            idx = np.where(e["queue"] == q)[0]
            idx = idx[np.argsort(e["pos"][idx])]
            assert np.all(np.diff(e["wt"][idx]) >= 0)          # monotone wt
            assert np.all(np.diff(e["V"][idx]) >= 0)
        s1, s2, _ = o.score(row)
        assert 0.0 <= s1 <= 1.0
        assert s2 == pytest.approx((e["wt"] - p.slo).sum(), rel=1e-12)
        # expected-violation mass is an integer when every v is 0 or 1
        v = np.array([O.violation(e["wt"][i], e["V"][i], p.slo[i]) for i in range(p.G)])
        if np.all((v == 0) | (v == 1)):
            assert (s1 * p.n_req.sum()) == pytest.approx(round(s1 * p.n_req.sum()), abs=1e-9)


def test_zero_swap_within_one_model_and_separability():
    rng = np.random.default_rng(5)
    # all groups of the resident model: no transition cost anywhere
    p = hand_problem([0] * 9, rng.integers(1, 100, 9), rng.uniform(50, 300, 9),
                     rng.uniform(0, 1e4, 9), 50.0, Q=3, swap=1e6, prefill=1e6)
    o = O.Oracle(p)
    row = O.random_row(3, 11, p.T)
    e = o.estimate(row)
    a = p.n_req * p.mu / 1000.0
    for q in range(3):
        idx = np.where(e["queue"] == q)[0]
        idx = idx[np.argsort(e["pos"][idx])]
        if len(idx) == 0:
            continue
        np.testing.assert_allclose(e["wt"][idx], np.concatenate([[0], np.cumsum(a[idx])[:-1]]),
                                   rtol=1e-13, atol=0)
    # separability: S2 of the row = sum over queues of each queue scored alone
    pr = make_config("C2")
    o2 = O.Oracle(pr)
    row = O.random_row(1, 5, pr.T)
    s1, s2, _ = o2.score(row)
    e = o2.estimate(row)
    tot = 0.0
    for q in range(pr.Q):
        idx = np.where(e["queue"] == q)[0]
        tot += (e["wt"][idx] - pr.slo[idx]).sum()
    assert s2 == pytest.approx(tot, rel=1e-12)


def test_queue_label_symmetry():
    # two queues with identical (device, resident, backlog): swapping their contents
    # leaves the multiset of (wt, V) and both scores unchanged.
    rng = np.random.default_rng(9)
    p = make_random_problem(rng, 10, 2, 3, 1)
    p.q_resident[:] = 1
    p.q_device[:] = 0
    o = O.Oracle(p)
    row = O.random_row(4, 1, p.T)
    bar = int(np.where(row >= p.G)[0][0])
    swapped = np.concatenate([row[bar + 1:], [row[bar]], row[:bar]])
    a, b = o.score(row), o.score(swapped)
    assert a[0] == pytest.approx(b[0], abs=1e-15)
    assert a[1] == pytest.approx(b[1], rel=1e-12)
    ea, eb = o.estimate(row), o.estimate(swapped)
    np.testing.assert_array_equal(ea["wt"], eb["wt"])
    np.testing.assert_array_equal(ea["V"], eb["V"])


def test_backlog_makes_first_switch_pay_tail():
    # R12: a pinned in-flight backlog of the resident model must drain (its tail)
    # before a different model can be swapped in.
    p = hand_problem([1], 10, 100.0, 0.0, 1e3, M=2, theta=1000.0, prefill=0.5, eps=1.0,
                     dtok=0.5, max_out=1.0, swap=7.0, backlog_mean=[3.0], backlog_var=[0.25])
    e = O.Oracle(p).estimate([0])
    assert e["wt"][0] == 3.0 + 1.0 + 7.0 and e["V"][0] == 0.25


def test_invalid_rows_rejected():
    p = make_config("C1")
    o = O.Oracle(p)
    with pytest.raises(ValueError):
        o.estimate([0, 1, 1, 3])
    with pytest.raises(ValueError):
        o.estimate([0, 1, 2, 4])


# ---------------------------------------------------------------- Monte-Carlo (P14/P15)
def test_mc_constant_table_closed_form():
    L = 123
    tabs = np.full((2, 256), L, np.uint16)
    tabs[1] = 7
    p = hand_problem([0, 0, 0], [5, 17, 300], 123.0, 0.0, [1.0, 3.0, 4.0], theta=1000.0,
                     len_tables=tabs, dist=[0, 1, 0])
    X = O.Oracle(p).mc_sample(2, 0, 5)
    assert np.all(X[:, 0] == 5 * L) and np.all(X[:, 1] == 17 * 7) and np.all(X[:, 2] == 300 * L)


def test_mc_two_value_table_parity_and_mean():
    tab = np.array([[1] * 512 + [3] * 512], np.uint16)
    n = 400
    p = hand_problem([0], n, 2.0, 1.0, 1.0, len_tables=tab, dist=[0])
    X = O.Oracle(p).mc_sample(9, 0, 2000)[:, 0].astype(np.int64)
    assert np.all((X - n) % 2 == 0) and X.min() >= n and X.max() <= 3 * n
    # Binomial(n, 1/2) upper-half draws: mean 2n, sd = 2*sqrt(n/4) = sqrt(n)
    assert abs(X.mean() - 2 * n) < 5 * math.sqrt(n) / math.sqrt(2000)


def test_mc_clt_normality_P15():
    # Appendix A: sums of n i.i.d. table draws are ~Normal.
    p = make_config("C4")
    tab = p.len_tables[int(p.dist[0])].astype(np.float64)
    mu, var = tab.mean(), tab.var()
    n = 200
    q = hand_problem([0], n, mu, var, 1.0, len_tables=p.len_tables, dist=[p.dist[0]])
    X = O.Oracle(q).mc_sample(2, 0, 3000)[:, 0].astype(np.float64)
    z = (X - n * mu) / math.sqrt(n * var)
    assert abs(z.mean()) < 4 / math.sqrt(3000)
    assert abs(z.std() - 1) < 0.06
    assert stats.kstest(z, "norm").pvalue > 0.01


def test_mc_deterministic_table_is_step_function():
    # constant lengths L: X/Theta is exactly n*L/Theta, so the MC walk equals the
    # Gaussian walk with sigma = 0 and counts are T_mc * [wt > slo].
    L = 64
    tabs = np.full((1, 64), L, np.uint16)
    rng = np.random.default_rng(1)
    p = make_random_problem(rng, 12, 3, 2, 2, sigma_zero=True)
    p.mu[:] = L
    p.len_tables = tabs
    p.dist = np.zeros(p.G, np.int32)
    o = O.Oracle(p)
    X = o.mc_sample(5, 0, 7)
    for c in range(10):
        row = O.random_row(1, c, p.T)
        e = o.estimate(row)
        cnt = o.mc_count(O.EXPLICIT, 0, 1, X, rows=row[None, :].astype(np.uint8))[0]
        np.testing.assert_array_equal(cnt, 7 * (e["wt"] > p.slo))


def test_mc_vs_gaussian_within_clt_scale():
    # statistical sanity (not parity): MC violation frequency vs the Gaussian
    # estimate on the C4 balanced ordering, within Edgeworth scale + 5 s.e.
    p = make_config("C4")
    o = O.Oracle(p)
    row = balanced_row(p.G, p.Q)
    T_mc = 400
    X = o.mc_sample(2, 0, T_mc)
    cnt = o.mc_count(O.EXPLICIT, 0, 1, X, rows=row[None, :])[0]
    e = o.estimate(row.astype(np.int32))
    v = np.array([O.violation(e["wt"][i], e["V"][i], p.slo[i]) for i in range(p.G)])
    vmc = cnt / T_mc
    se = np.sqrt(np.maximum(v * (1 - v), 1e-4) / T_mc)
    assert np.all(np.abs(vmc - v) <= 0.03 + 5 * se)


# ------------------------------------------------------- NEIGHBOR rows (R18, N1)
@pytest.mark.parametrize("T", [4, 17, 71])
def test_neighbor_rows_are_nearby_permutations(T):
    base = O.random_row(3, 5, T)
    assert np.array_equal(O.neighbor_row(base, 9, 123, 0), base)      # k = 0: the base row
    for k in (1, 2, 5):
        for c in range(200):
            row = O.neighbor_row(base, 9, c, k)
            assert sorted(row) == list(range(T))
            assert np.count_nonzero(row != base) <= 2 * k
            assert np.count_nonzero(row != base) != 1                  # a transposition moves 0 or 2


def test_neighbor_single_move_uniform_over_pairs():
    # k = 1: positions i, j uniform and independent -> P(i == j) = 1/T, and each
    # unordered pair {i, j}, i != j, has probability 2/T^2.
    T, N = 5, 20000
    base = np.arange(T)
    counts = {}
    for c in range(N):
        d = tuple(np.nonzero(O.neighbor_row(base, 4, c, 1) != base)[0])
        counts[d] = counts.get(d, 0) + 1
    pairs = list(itertools.combinations(range(T), 2))
    obs = [counts.get((), 0)] + [counts.get(p, 0) for p in pairs]
    exp = [N / T] + [N * 2 / T**2] * len(pairs)
    assert sum(obs) == N
    assert stats.chisquare(obs, exp).pvalue > 1e-3


@pytest.mark.parametrize("seed", range(8))
def test_local_search_reaches_brute_force_optimum(seed):
    # SURVEY 8(f) N1 on instances small enough for exhaustive search (ENUM over
    # all T! rows): iterated best-of-N over 2-move neighbourhoods, started from
    # the identity row, ends at the brute-force minimum of the (S1, S2) key.
    rng = np.random.default_rng(300 + seed)
    G, Q = int(rng.integers(4, 7)), int(rng.integers(1, 3))
    p = make_random_problem(rng, G, Q, 2, 1, backlog=bool(seed % 2))
    o = O.Oracle(p)
    T = p.T
    r = o.score_range(O.ENUM, 0, math.factorial(T))
    best = O.key32(*min(zip(r["s1"], r["s2"]), key=lambda x: O.key32(*x)))
    row, key, adopted = O.local_search(o, np.arange(T), seed=seed + 1, moves=2, per_iter=48, iters=40)
    assert key == best
    s1, s2, _ = o.score(row)
    assert O.key32(s1, s2) == key
    assert sorted(row) == list(range(T))


# ------------------------------------------- request-level violations (R19, N2)
def test_request_violations_single_request_groups_equal_group_level():
    # n_i = 1: the only request is the group's first, so f_i = v_i and S1_req = S1.
    rng = np.random.default_rng(5)
    p = make_random_problem(rng, 12, 3, 3, 2, backlog=True)
    p.n_req[:] = 1
    o = O.Oracle(p)
    for c in range(20):
        row = O.random_row(2, c, p.T)
        e = o.estimate(row)
        f, s1 = o.request_violations(row)
        v = np.array([O.violation(e["wt"][i], e["V"][i], p.slo[i]) for i in range(p.G)])
        assert np.array_equal(f, v)
        assert s1 == pytest.approx(o.score(row)[0], abs=1e-15)


@pytest.mark.parametrize("seed", range(6))
def test_request_violations_deterministic_step_count(seed):
    # sigma = 0: request r violates iff wt + r * mu/Theta > slo, so the fraction
    # is a closed-form count of the requests past the deadline.
    rng = np.random.default_rng(40 + seed)
    G = int(rng.integers(2, 9))
    n = rng.integers(1, 400, G)
    mu = rng.uniform(10, 500, G)
    theta = 1500.0
    slo = rng.uniform(0.5, 60.0, G)
    p = hand_problem([0] * G, n, mu, 0.0, slo, theta=theta)
    o = O.Oracle(p)
    row = rng.permutation(G)
    e = o.estimate(row)
    f, _ = o.request_violations(row)
    for i in range(G):
        a = mu[i] / theta
        ok = (slo[i] - e["wt"][i]) / a          # requests r <= ok meet the SLO
        met = 0 if ok < 0 else min(n[i], int(np.floor(ok)) + 1)
        assert f[i] == pytest.approx((n[i] - met) / n[i], abs=1e-12)


def test_request_violations_bounds():
    p = make_config("C3")
    o = O.Oracle(p)
    for c in range(10):
        row = O.random_row(1, c, p.T)
        e = o.estimate(row)
        f, s1r = o.request_violations(row)
        v = np.array([O.violation(e["wt"][i], e["V"][i], p.slo[i]) for i in range(p.G)])
        assert np.all(f >= v - 1e-15) and np.all(f <= 1.0)     # later requests wait longer
        assert s1r >= o.score(row)[0] - 1e-15


# ---------------------------------------------------------------- N3: two-tier swapping (R20)
def _tier_hand():
    p = hand_problem([1, 2, 1, 3, 0], 25, 200.0, 0.0, 1e4, theta=1000.0, prefill=0.5, eps=1.0,
                     dtok=0.5, max_out=1.0, swap=20.0, M=4)
    tiers = dict(mem=np.array([5, 2, 3, 1], np.int32), cap=np.array([4], np.int32),
                 load=np.array([[10.0, 20.0, 30.0, 40.0]]))
    return p, tiers


def test_tiers_hand_golden_N3():
    g = gold("n3_tiers.json")
    p, tiers = _tier_hand()
    o = O.Oracle(p)
    row = [0, 1, 2, 3, 4]
    e = o.estimate_tiered(row, tiers)
    assert list(e["wt"]) == g["wt_by_group"]
    assert list(e["cold"]) == g["cold_by_group"]
    assert list(o.estimate(row)["wt"]) == g["wt_untiered"]
    big = dict(tiers, cap=np.array([11], np.int32))          # every model fits: all warm
    assert list(o.estimate_tiered(row, big)["wt"]) == g["wt_all_warm"]
    zero = dict(tiers, cap=np.array([0], np.int32))          # no CPU memory: all cold
    assert list(o.estimate_tiered(row, zero)["wt"]) == g["wt_all_cold"]


def _rand_tier_case(seed):
    rng = np.random.default_rng(9000 + seed)
    G, Q, M, D = int(rng.integers(4, 24)), int(rng.integers(1, 5)), int(rng.integers(2, 6)), int(rng.integers(1, 3))
    p = make_random_problem(rng, G, Q, M, D, backlog=bool(seed % 2))
    from workloads.synth import make_random_tiers
    return rng, p, make_random_tiers(rng, M, D)


@pytest.mark.parametrize("seed", range(8))
def test_tiers_reduce_to_untiered_when_all_warm_or_free(seed):
    # cap >= sum(mem): every target warm -> the R1-R7 estimator, bit for bit;
    # load = 0: the tier never changes the cost -> the same.
    rng, p, tiers = _rand_tier_case(seed)
    o = O.Oracle(p)
    allwarm = dict(tiers, cap=np.full(p.D, int(tiers["mem"].sum()), np.int32))
    free = dict(tiers, load=np.zeros_like(tiers["load"]))
    for c in range(20):
        row = o.random_row(7, c)
        base = o.estimate(row)
        for t in (allwarm, free):
            e = o.estimate_tiered(row, t)
            assert np.array_equal(e["wt"], base["wt"]) and np.array_equal(e["V"], base["V"])
        assert o.score_tiered(row, allwarm) == o.score(row)


@pytest.mark.parametrize("seed", range(8))
def test_tiers_all_cold_equals_folded_swap_table(seed):
    # cap = 0: every transition is cold, i.e. the untiered estimator with
    # swap'[d][a][b] = swap[d][a][b] + load[d][b] (same single addition).
    import dataclasses
    rng, p, tiers = _rand_tier_case(seed)
    cold = dict(tiers, cap=np.zeros(p.D, np.int32))
    sw = p.swap + tiers["load"][:, None, :]
    for d in range(p.D):
        np.fill_diagonal(sw[d], 0.0)
    o, of = O.Oracle(p), O.Oracle(dataclasses.replace(p, swap=sw))
    for c in range(20):
        row = o.random_row(11, c)
        e, f = o.estimate_tiered(row, cold), of.estimate(row)
        assert np.array_equal(e["wt"], f["wt"]) and np.array_equal(e["V"], f["V"])


@pytest.mark.parametrize("seed", range(6))
def test_tiers_wait_monotone_in_cpu_memory(seed):
    # More CPU memory only lengthens the warm prefix: no wait can grow.
    rng, p, tiers = _rand_tier_case(seed)
    o = O.Oracle(p)
    total = int(tiers["mem"].sum())
    for c in range(10):
        row = o.random_row(5, c)
        prev = None
        for cap in range(0, total + 2, max(1, total // 12)):
            e = o.estimate_tiered(row, dict(tiers, cap=np.full(p.D, cap, np.int32)))
            if prev is not None:
                assert np.all(e["wt"] <= prev + 1e-9 * np.maximum(1.0, prev))
            prev = e["wt"]
            assert np.all(e["cold"] <= 1)


# ---------------------------------------------------------------- N4: group formation (R21)
def _req(model, slo, out, feat):
    return dict(model=np.asarray(model, np.int32), slo=np.asarray(slo, np.float64),
                out=np.asarray(out, np.int32), feat=np.asarray(feat, np.int32).reshape(len(model), -1))


def test_groups_spec_identical_requests_split_in_half():
    # S:L199 (Alg. 1 split rule): 8 identical requests, threshold 4 -> two groups of 4
    r = _req([0] * 8, [20.0] * 8, [100] * 8, [[7, 7]] * 8)
    g = O.form_groups(r, 1, [3], limit=4)
    assert g["k_eff"][0] == 1                      # no distinct point for a second centre
    assert g["n_groups"] == 2 and list(g["n"]) == [4, 4]
    assert list(g["group_of"]) == [0, 0, 0, 0, 1, 1, 1, 1]   # arrival-order halves
    assert list(g["mu"]) == [100.0, 100.0] and list(g["var"]) == [0.0, 0.0]


def test_groups_spec_models_are_a_hard_partition():
    # requests of 2 models, k = 2 -> >= 2 groups, none mixing models
    rng = np.random.default_rng(3)
    n = 60
    model = rng.integers(0, 2, n)
    feat = rng.integers(0, 1000, (n, 2))
    g = O.form_groups(_req(model, np.full(n, 20.0), rng.integers(1, 500, n), feat), 2, [2, 2], limit=100)
    assert g["n_groups"] >= 2
    for k in range(g["n_groups"]):
        assert len(set(model[g["group_of"] == k])) == 1
        assert g["model"][k] == model[g["group_of"] == k][0]


def test_groups_spec_slo_classes_do_not_overlap():
    # 100 requests, SLOs {20 s, 3600 s}, k = 2 -> SLO ranges do not overlap
    rng = np.random.default_rng(4)
    slo = rng.choice([20.0, 3600.0], 100)
    feat = np.rint(4096 * np.log2(slo)).astype(np.int32)[:, None]
    g = O.form_groups(_req(np.zeros(100), slo, np.full(100, 10), feat), 1, [2], limit=1000)
    assert g["n_groups"] == 2
    a, b = slo[g["group_of"] == 0], slo[g["group_of"] == 1]
    assert a.max() < b.min() or b.max() < a.min()


def _farthest_point_ok(feat, model, init, k_eff):
    """Each chosen centre is a farthest point (exact int64) from the centres before it."""
    off = 0
    for m, k in enumerate(k_eff):
        idx = np.where(model == m)[0]
        if k == 0:
            continue
        assert init[off] == idx[0]                           # first request of the model
        X = feat[idx].astype(np.int64)
        for j in range(1, k):
            C = feat[init[off:off + j]].astype(np.int64)
            mind = ((X[:, None, :] - C[None]) ** 2).sum(-1).min(1)
            assert mind.max() > 0
            best = idx[np.flatnonzero(mind == mind.max())[0]]   # lowest index on ties
            assert init[off + j] == best
        off += k


@pytest.mark.parametrize("seed", range(6))
def test_groups_lloyd_matches_sklearn_from_the_same_start(seed):
    # Lloyd's algorithm (textbook) as implemented by scikit-learn, started from
    # the oracle's farthest-point centres: same final partition per model.
    from sklearn.cluster import KMeans
    from workloads.synth import make_requests
    r = make_requests(3000, seed=100 + seed)
    M, k = 4, [3, 4, 5, 6]
    g = O.form_groups(r, M, k, limit=32768, max_iter=300)
    _farthest_point_ok(r["feat"], r["model"], g["init"], g["k_eff"])
    assert g["iters"] < 300                               # converged: labels stable
    off = 0
    for m in range(M):
        idx = np.where(r["model"] == m)[0]
        X = r["feat"][idx].astype(np.float64)
        init = r["feat"][g["init"][off:off + g["k_eff"][m]]].astype(np.float64)
        km = KMeans(n_clusters=len(init), init=init, n_init=1, max_iter=300, tol=0.0,
                    algorithm="lloyd").fit(X)
        ours = g["label"][idx] - off
        # same partition (labels index the same initial centres)
        assert np.array_equal(km.labels_, ours)
        off += g["k_eff"][m]


@pytest.mark.parametrize("seed", range(4))
def test_groups_fixed_point_split_and_stats(seed):
    from workloads.synth import make_requests
    r = make_requests(5000, seed=200 + seed)
    L = 97
    g = O.form_groups(r, 4, [5, 5, 5, 5], limit=L, max_iter=200)
    feat, model = r["feat"].astype(np.float64), r["model"]
    lab = g["label"]
    # Lloyd fixed point: every request sits at its nearest centre of its model,
    # the centres being the means of the final clusters
    K = int(g["k_eff"].sum())
    cent = np.array([feat[lab == j].mean(0) if np.any(lab == j) else np.full(feat.shape[1], np.nan)
                     for j in range(K)])
    off = np.concatenate([[0], np.cumsum(g["k_eff"])])
    for m in range(4):
        idx = np.where(model == m)[0]
        d = ((feat[idx][:, None, :] - cent[off[m]:off[m + 1]][None]) ** 2).sum(-1)
        assert np.all(d[np.arange(len(idx)), lab[idx] - off[m]] <= d.min(1) * (1 + 1e-12))
    # splitHalf: groups are consecutive arrival-order runs of one cluster, numbered
    # cluster by cluster; no group exceeds L; halves of a split cluster keep >= ceil(L/2)
    gid = 0
    for j in range(K):
        mem = np.where(lab == j)[0]
        if len(mem) == 0:
            continue
        gs = g["group_of"][mem]
        assert np.all(np.diff(gs) >= 0) and gs[0] == gid
        sizes = np.bincount(gs - gid)
        assert sizes.max() <= L and sizes.sum() == len(mem)
        if len(mem) > L:
            assert sizes.min() >= (L + 1) // 2
        if len(mem) in (L * 2, L * 4):
            assert np.all(sizes == L)
        gid += len(sizes)
    assert gid == g["n_groups"]
    # group statistics: numpy's mean / population variance / min over the members
    for k in range(g["n_groups"]):
        mem = g["group_of"] == k
        o = r["out"][mem].astype(np.float64)
        assert g["n"][k] == mem.sum() and g["model"][k] == model[mem][0]
        assert g["slo"][k] == r["slo"][mem].min()
        assert g["mu"][k] == pytest.approx(o.mean(), rel=1e-14)
        assert g["var"][k] == pytest.approx(o.var(), rel=1e-12, abs=1e-9)


@pytest.mark.parametrize("seed", range(4))
def test_mc_tiered_reduces_to_untiered_and_folded_table(seed):
    # tiered MC counts: cap >= sum(mem) (all warm) equals or_mc_count; cap = 0
    # (all cold) equals or_mc_count with swap + load folded into the table
    import dataclasses
    from workloads.synth import make_random_tiers
    rng = np.random.default_rng(4400 + seed)
    G, Q, M, D = int(rng.integers(4, 16)), int(rng.integers(1, 4)), int(rng.integers(2, 5)), int(rng.integers(1, 3))
    p = make_random_problem(rng, G, Q, M, D, backlog=bool(seed % 2), with_tables=True)
    tiers = make_random_tiers(rng, M, D)
    o = O.Oracle(p)
    X = o.mc_sample(3, 0, 40)
    allwarm = dict(tiers, cap=np.full(D, int(tiers["mem"].sum()), np.int32))
    cold = dict(tiers, cap=np.zeros(D, np.int32))
    base = o.mc_count(O.RANDOM, 0, 30, X, seed=2)
    assert np.array_equal(o.mc_count_tiered(allwarm, O.RANDOM, 0, 30, X, seed=2), base)
    sw = p.swap + tiers["load"][:, None, :]
    for d in range(D):
        np.fill_diagonal(sw[d], 0.0)
    of = O.Oracle(dataclasses.replace(p, swap=sw))
    assert np.array_equal(o.mc_count_tiered(cold, O.RANDOM, 0, 30, X, seed=2),
                          of.mc_count(O.RANDOM, 0, 30, X, seed=2))
