"""qlm_large.cu (D = 1 thread-per-candidate scorer over the 16-bit rows of the
two-phase large-T RANDOM path): bit-identical to the general scan kernel on
the same rows -- every candidate's S1, S2, n_over and the argmin record -- and
equal to the oracle on a ragged tail (objective P:L761-767, R11; Eq. 10 slot
arithmetic R1-R9, R22)."""
import os

import numpy as np
import pytest
import torch

import oracle as O
from tests.parity import argmin_ok, check_scores
from workloads.synth import make_config, make_random_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()


def hi_only(p):
    """The same problem with every SLO rounded to a zero low 32-bit word (the
    record layout of the D = 1 kernels keeps the high word only)."""
    u = p.slo.astype(np.float64).view(np.uint64) & np.uint64(0xFFFFFFFF00000000)
    p.slo = u.view(np.float64).copy()
    return p


def run(p, first, n, seed, no_large, cap=0):
    from paper_2407_00047_b200 import RwtEstimator, kernel_overrides
    kernel_overrides(no_large=no_large, no_wide=True, ilv_cap=cap)
    try:
        e = RwtEstimator(p, device=0)
        rec = torch.empty(2, dtype=torch.int64, device="cuda")
        s1, s2, nov = e.score_orderings(e.random(first, n, seed=seed))
        rec2 = e.best_ordering_async(e.random(first, n, seed=seed), rec)
        torch.cuda.synchronize()
        return s1.clone(), s2.clone(), nov.clone(), rec2.clone()
    finally:
        kernel_overrides()


CASES = [
    # (G, Q, M, backlog): T = G + Q - 1 from 257 (odd) to 2060 (even)
    (250, 8, 4, False),
    (256, 2, 3, True),
    (300, 33, 6, True),
    (1024, 32, 4, False),
    (2029, 32, 2, True),
]


@pytest.mark.parametrize("G,Q,M,backlog", CASES)
def test_large_kernel_equals_scan_kernel(G, Q, M, backlog):
    p = hi_only(make_random_problem(np.random.default_rng(G * 7 + Q), G, Q, M, backlog=backlog))
    n = 3 * 4096 + 45                                    # several chunks + a ragged batch
    a = run(p, 11, n, 5, no_large=False, cap=4096)
    b = run(p, 11, n, 5, no_large=True, cap=4096)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    lo, cnt = n - 9, 9
    ref = O.Oracle(p).score_range(O.RANDOM, 11 + lo, cnt, seed=5)
    check_scores(a[0][lo:].cpu().numpy(), a[1][lo:].cpu().numpy(), ref, p)


def test_large_kernel_C5_vs_oracle_sample():
    # C5 (1024 groups, 32 queues, D = 1): a strided sample re-scored by the
    # oracle, and the argmin of a 20000-candidate range
    p = make_config("C5")
    n = 20000
    s1, s2, nov, rec = run(p, 777, n, 1, no_large=False)
    o = O.Oracle(p)
    ref = o.score_range(O.RANDOM, 777, n, seed=1)
    check_scores(s1.cpu().numpy(), s2.cpu().numpy(), ref, p)
    ok, cstar = argmin_ok(int(rec[1]), ref["s1"], ref["s2"], p, first=777)
    assert ok, (int(rec[1]) - 777, cstar)


def test_large_kernel_is_chosen_for_C5():
    # the library's own log names the kernel that ran (QLM_LOG is read once per
    # process, so a child process checks it)
    import subprocess
    import sys
    code = ("import torch, __graft_entry__; __graft_entry__.build();"
            "from paper_2407_00047_b200 import RwtEstimator; from workloads.synth import make_config;"
            "e = RwtEstimator(make_config('C5')); e.best_ordering_async(e.random(0, 8192, seed=1));"
            "torch.cuda.synchronize()")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, QLM_LOG="1"), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "large_kernel<score=" in r.stderr, r.stderr[-2000:]


def unclamped_problem(G, Q, M, seed):
    """A D = 1 problem where most slots have |z| < z_clamp: large output
    variance and each SLO at the median waiting time of its group over a
    sample of orderings, so the deferred-Phi-bar FIFOs of ws2_kernel /
    large_kernel fill and flush many times per row (R8/R9)."""
    rng = np.random.default_rng(seed)
    p = make_random_problem(rng, G, Q, M, backlog=True)
    p.n_req = rng.integers(1, 4, G).astype(np.int32)         # few requests: sd ~ mean per group
    p.var = (3.0 * p.mu) ** 2
    p.q_backlog_var = np.maximum(p.q_backlog_var, 4.0)      # sd > 0 at every queue head
    p.dtok, p.prefill, p.swap = p.dtok * 1e-3, p.prefill * 1e-3, p.swap * 1e-3   # small fixed terms
    wt = O.Oracle(p).estimate_range(O.RANDOM, 0, 64, seed=11)["wt"]   # [count][G]
    p.slo = np.median(wt, axis=0) * rng.uniform(0.9, 1.1, G)
    return hi_only(p)


@pytest.mark.parametrize("G,Q,seed", [(60, 5, 1), (120, 9, 2), (300, 7, 3)])
def test_deferred_fifo_stress(G, Q, seed):
    # most slots unclamped: ws2 (T <= 256) / large_kernel (T > 256) equal the
    # general kernels bit for bit (bulk for ws2, scores for both) and the
    # oracle on a tail; S1 is dominated by the FIFO's Phi-bar terms
    from paper_2407_00047_b200 import RwtEstimator, kernel_overrides
    p = unclamped_problem(G, Q, 4, seed)
    n = 4096 + 61
    o = O.Oracle(p)
    ref = o.score_range(O.RANDOM, 3 + n - 24, 24, seed=4)
    est = o.estimate_range(O.RANDOM, 3 + n - 24, 24, seed=4)
    frac_open = np.mean(np.abs(p.slo[None, :] - est["wt"]) < 8.0 * est["sd"])   # |z| < z_clamp
    assert frac_open > 0.5, frac_open                  # the stress is real
    res = {}
    for path in ("fast", "general"):
        kernel_overrides(no_ws2=path == "general", no_large=path == "general", no_wide=True)
        try:
            e = RwtEstimator(p, device=0)
            cand = e.random(3, n, seed=4)
            rec = torch.empty(2, dtype=torch.int64, device="cuda")
            if p.T <= 256:
                bufs = {k: torch.empty((p.G, n), dtype=torch.float32, device="cuda") for k in ("wt", "sd", "v")}
                bufs["n_over"] = torch.empty(n, dtype=torch.int32, device="cuda")
                out = e.score_estimate(cand, out=bufs, rec=rec)
                res[path] = [out[k].clone() for k in ("wt", "sd", "v", "s1", "s2", "n_over")] + [rec.clone()]
            else:
                s1, s2, nov = e.score_orderings(cand)
                rec = e.best_ordering_async(cand, rec)
                res[path] = [s1.clone(), s2.clone(), nov.clone(), rec.clone()]
            torch.cuda.synchronize()
        finally:
            kernel_overrides()
    for a, b in zip(res["fast"], res["general"]):
        assert torch.equal(a, b)
    s1 = res["fast"][3 if p.T <= 256 else 0]
    s2 = res["fast"][4 if p.T <= 256 else 1]
    check_scores(s1[n - 24:].cpu().numpy(), s2[n - 24:].cpu().numpy(), ref, p)


@pytest.mark.parametrize("G,Q,M", [(40, 150, 3), (100, 157, 6), (9, 200, 2)])
def test_ws2_many_queues(G, Q, M):
    # byte rows near T = 256 with many separators (T = 189, 256 -- no padding
    # byte -- and 208): the seven-pair plan shrinks to fewer pairs; ws2 equals
    # the general warp-specialised kernel and the scan bit for bit, and the oracle
    from paper_2407_00047_b200 import RwtEstimator, kernel_overrides
    p = hi_only(make_random_problem(np.random.default_rng(G + Q + M), G, Q, M, backlog=True))
    assert p.T <= 256
    n = 4096 + 33
    res = {}
    for path in ("ws2", "ws", "scan"):
        kernel_overrides(no_ws2=path == "ws", no_ws=path == "scan")
        try:
            e = RwtEstimator(p, device=0)
            rec = torch.empty(2, dtype=torch.int64, device="cuda")
            bufs = {k: torch.empty((p.G, n), dtype=torch.float32, device="cuda") for k in ("wt", "sd", "v")}
            bufs["n_over"] = torch.empty(n, dtype=torch.int32, device="cuda")
            out = e.score_estimate(e.random(1, n, seed=2), out=bufs, rec=rec)
            torch.cuda.synchronize()
            res[path] = [out[k].clone() for k in ("wt", "sd", "v", "s1", "s2", "n_over")] + [rec.clone()]
        finally:
            kernel_overrides()
    for path in ("ws", "scan"):
        for a, b in zip(res["ws2"], res[path]):
            assert torch.equal(a, b), path
    ref = O.Oracle(p).score_range(O.RANDOM, 1 + n - 16, 16, seed=2)
    check_scores(res["ws2"][3][n - 16:].cpu().numpy(), res["ws2"][4][n - 16:].cpu().numpy(), ref, p)
