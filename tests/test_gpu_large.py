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
