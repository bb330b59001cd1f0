"""GPU edge cases the oracle pins hold for the device too, and full-range
argmin parity at C5 / C5h ("parity on a strided subsample +
a 1e6-prefix argmin").

* S:L62-70 boundary: wt == slo with V = 0 is MET (v = 0), wt > slo by one ulp
  is violated (v = 1) -- on the thread-per-candidate scan and on the
  warp-specialised kernel (>= 4096 candidates).
* S:L375 tie: two orderings with identical (S1, S2) -> the lowest candidate
  index wins (R14), on both kernels.
* C5 / C5h argmin over a contiguous 1e6 / 2e5 range equals the oracle's
  argmin (rule of tests/parity.argmin_ok); the oracle runs split over the
  host cores inside the test."""
import json
import math
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
from tests.handmade import hand_problem
from tests.parity import argmin_ok
from workloads.synth import make_config

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "spec_examples.json")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()


def est_of(p):
    from paper_2407_00047_b200 import RwtEstimator
    return RwtEstimator(p, device=0)


def explicit_rows(e, rows, copies):
    """`copies` repetitions of the given rows as a u8 EXPLICIT candidate set."""
    rows = np.asarray(rows, np.uint8)
    buf = np.zeros((len(rows) * copies, 16), np.uint8)
    buf[:, :rows.shape[1]] = np.tile(rows, (copies, 1))
    return e.explicit(torch.tensor(buf, device="cuda"))


@pytest.mark.parametrize("copies", [1, 4096])           # scan kernel / warp-specialised kernel
def test_boundary_wt_equal_slo_is_met_S62(copies):
    # A: 40 x 200 tokens at 1000 tok/s = 8 s, sigma = 0 -> B waits exactly 8 s
    # with V = 0: the step [wt > slo] (R9); slo_B = 8 s is met, 7.5 s is not
    for slo_b, v_b in ((8.0, 0.0), (7.5, 1.0)):
        p = hand_problem([0, 0], [40, 10], 200.0, 0.0, [10.0, slo_b], theta=1000.0)
        e = est_of(p)
        cand = explicit_rows(e, [[0, 1]], copies)
        out = e.score_estimate(cand, out={k: torch.empty((2, copies), device="cuda") for k in ("wt", "sd", "v")},
                               rec=torch.empty(2, dtype=torch.int64, device="cuda"))
        assert float(out["wt"][1, 0]) == 8.0 and float(out["sd"][1, 0]) == 0.0
        assert float(out["v"][1, 0]) == v_b
        assert torch.all(out["v"][1] == v_b)
        assert float(out["s1"][0]) == float(np.float32(v_b * 10 / 50))
        ref = O.Oracle(p).score([0, 1])
        assert float(out["s1"][0]) == np.float32(ref[0])


@pytest.mark.parametrize("copies", [1, 2048])
def test_objective_tie_lowest_index_S375(copies):
    g = json.load(open(GOLD))["tie_S375"]
    p = hand_problem([0, 0], [25, 25], 200.0, 0.0, g["slos"], theta=1000.0)
    e = est_of(p)
    # both orders tie on (S1, S2); candidates alternate [0,1], [1,0], ...
    cand = explicit_rows(e, [[0, 1], [1, 0]], copies)
    out = e.score_estimate(cand, out={k: torch.empty((2, 2 * copies), device="cuda") for k in ("wt", "sd", "v")},
                           rec=torch.empty(2, dtype=torch.int64, device="cuda"))
    s2 = out["s2"].cpu().numpy()
    assert np.all(s2 == np.float32(g["objective"]))
    rec = e.best_ordering_async(cand)
    assert int(rec[1]) == 0                            # R14: lowest global index
    en = e.best_ordering_async(e.enum(0, 2))
    assert int(en[1]) == 0


def _score_chunk(args):
    cfg, first, count = args
    r = O.Oracle(make_config(cfg)).score_range(O.RANDOM, first, count, seed=1)
    return r["s1"], r["s2"]


@pytest.mark.parametrize("cfg,first,n", [("C5", 12_345_678, 1_000_000), ("C5h", 98_765, 200_000)])
def test_large_G_argmin_vs_oracle_full_range(cfg, first, n):
    p = make_config(cfg)
    e = est_of(p)
    rec = e.best_ordering_async(e.random(first, n, seed=1))
    torch.cuda.synchronize()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    parts = max(cores, 1) * 4
    step = math.ceil(n / parts)
    jobs = [(cfg, first + a, min(step, n - a)) for a in range(0, n, step)]
    with mp.get_context("fork").Pool(max(cores, 1)) as pool:
        res = pool.map(_score_chunk, jobs)
    s1 = np.concatenate([r[0] for r in res])
    s2 = np.concatenate([r[1] for r in res])
    ok, cstar = argmin_ok(int(rec[1]), s1, s2, p, first=first)
    assert ok, (int(rec[1]) - first, cstar, s1[cstar], s2[cstar])


def test_launch_limits_are_named_errors():
    # one-block-per-row launches refuse counts that do not fit a grid dimension
    # instead of wrapping (qlm_check_rows)
    from paper_2407_00047_b200 import _lib as L
    p = make_config("C2")
    e = est_of(p)
    buf = torch.zeros((4, 32), dtype=torch.uint8, device="cuda")
    cand = e.explicit(buf)
    c = cand.c()
    c.count = (1 << 31) + 5
    import ctypes as C
    n = C.c_int64()
    rc = L.lib().qlm_check_rows(e._h, C.byref(c), C.byref(n), None)
    assert rc == L.QLM_ECUDA and "invalid argument" in L.lib().qlm_last_error().decode()


def test_calls_restore_the_current_device():
    # every entry point makes the context's device current and restores the
    # caller's on return; with two GPUs the second context must not leak
    p = make_config("C2")
    n_dev = torch.cuda.device_count()
    torch.cuda.set_device(0)
    from paper_2407_00047_b200 import RwtEstimator
    ests = [RwtEstimator(p, device=d) for d in range(min(n_dev, 2))]
    for est in ests:
        torch.cuda.set_device(0)
        rec = est.best_ordering_async(est.random(0, 8192, seed=1))
        assert torch.cuda.current_device() == 0
        out = {k: torch.empty((p.G, 8192), device=est.device) for k in ("wt", "sd", "v")}
        est.score_estimate(est.random(0, 8192, seed=1), out=out)       # opts the bulk kernels in per device
        assert torch.cuda.current_device() == 0
        assert int(rec[1]) >= 0
    if len(ests) == 2:
        torch.cuda.synchronize(1)
        a = ests[0].best_ordering_async(ests[0].random(0, 8192, seed=1)).cpu()
        b = ests[1].best_ordering_async(ests[1].random(0, 8192, seed=1)).cpu()
        assert torch.equal(a, b)


@pytest.mark.parametrize("cap", [0, 4096])
def test_tiered_large_T_two_phase_equals_direct(cap):
    # tiered RANDOM scoring with T > 256 and G > 256 generates its rows per chunk
    # with fy_rows_kernel (two-phase); it must equal the lane-per-queue kernel
    # generating rows itself bit for bit, across chunks, and match the oracle
    from paper_2407_00047_b200 import RwtEstimator, kernel_overrides
    from workloads.synth import make_tiers
    from tests.parity import check_estimates, check_scores
    p = make_config("C5h")
    t = make_tiers(dev_rows=(0, 1))
    n = 9000
    res = {}
    for mode in ("direct", "two_phase"):
        kernel_overrides(no_two_phase=mode == "direct", ilv_cap=cap)
        e = RwtEstimator(p, device=0)
        e.set_tiers(t)
        cand = e.random(123, n, seed=1)
        out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
        rec = torch.empty(2, dtype=torch.int64, device="cuda")
        r = e.tiered_score_estimate(cand, out=out, rec=rec)
        torch.cuda.synchronize()
        res[mode] = (r, rec.clone())
        kernel_overrides()
    (a, ra), (b, rb) = res["direct"], res["two_phase"]
    for k in ("wt", "sd", "v", "s1", "s2"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(ra, rb)
    o = O.Oracle(p)
    lo, cnt = n - 40, 40
    ref = o.tiered_range(t, O.RANDOM, 123 + lo, cnt, seed=1)
    check_estimates({k: b[k][:, lo:lo + cnt] for k in ("wt", "sd", "v")}, ref)
    check_scores(b["s1"][lo:].cpu().numpy(), b["s2"][lo:].cpu().numpy(), ref, p)



@pytest.mark.parametrize("G,Q", [(250, 8), (300, 33), (1024, 32), (1990, 11), (3500, 2)])
def test_large_T_two_phase_rows_equal_direct_scan(G, Q):
    # large-T RANDOM: rows materialised by fy_rows_kernel and scored from the
    # interleaved scratch (two-phase) equal the scan kernel generating rows
    # itself, bit for bit -- every candidate's scores and the argmin -- and the
    # oracle on a ragged tail (T = 257 .. 3501)
    from paper_2407_00047_b200 import RwtEstimator, kernel_overrides
    from tests.parity import check_scores
    from workloads.synth import make_random_problem
    p = make_random_problem(np.random.default_rng(G + Q), G, Q, 4)
    n = 4096 + 77
    res = {}
    for direct in (False, True):
        kernel_overrides(no_two_phase=direct, no_wide=True)
        e = RwtEstimator(p, device=0)
        rec = torch.empty(2, dtype=torch.int64, device="cuda")
        out = e.score_estimate(e.random(5, n, seed=3), rec=rec)
        torch.cuda.synchronize()
        res[direct] = (out["s1"].clone(), out["s2"].clone(), rec.clone())
        kernel_overrides()
    for a, b in zip(res[False], res[True]):
        assert torch.equal(a, b)
    lo, cnt = n - 12, 12
    ref = O.Oracle(p).score_range(O.RANDOM, 5 + lo, cnt, seed=3)
    check_scores(res[False][0][lo:].cpu().numpy(), res[False][1][lo:].cpu().numpy(), ref, p)
