"""The library's own NCCL communicator through the C ABI (SURVEY 8(b)/(e):
qlm_comm_unique_id / qlm_comm_attach), on one GPU as a single-rank
communicator: every collective path (global argmin record, owner-decoded
best ordering, summed MC counts, sharded local search) runs through NCCL and
must return exactly what the same calls return without a communicator.
Multi-rank exchange logic is covered by tests/test_dist_gloo.py on CPU."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from workloads.synth import balanced_row, make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()


def pair(cfg):
    from paper_2407_00047_b200 import RwtEstimator
    p = make_config(cfg)
    a, b = RwtEstimator(p, device=0), RwtEstimator(p, device=0)
    b.comm_attach(RwtEstimator.comm_unique_id(), 0, 1)
    return p, a, b


def test_attach_info_and_detach():
    p, a, b = pair("C2")
    info = b.comm_info()
    assert info["world"] == 1 and info["rank"] == 0 and info["nccl_version"] > 20000
    assert a.comm_info()["world"] == 1 and not a.comm_attached and b.comm_attached
    b.comm_detach()
    assert not b.comm_attached
    from paper_2407_00047_b200 import RwtEstimator
    b.comm_attach(RwtEstimator.comm_unique_id(), 0, 1)       # re-attach
    assert b.comm_attached


@pytest.mark.parametrize("cfg,n", [("C2", 50_000), ("C3", 20_000)])
def test_global_record_paths_equal_local(cfg, n):
    p, a, b = pair(cfg)
    ca, cb = a.random(7, n, seed=1), b.random(7, n, seed=1)
    ra, rb = a.best_ordering_async(ca), b.best_ordering_async(cb)
    assert torch.equal(ra, rb)
    out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
    xa, xb = torch.empty(2, dtype=torch.int64, device="cuda"), torch.empty(2, dtype=torch.int64, device="cuda")
    a.score_estimate(ca, out=out, rec=xa)
    b.score_estimate(cb, out={k: torch.empty_like(v) for k, v in out.items()}, rec=xb)
    assert torch.equal(xa, xb) and torch.equal(xa, ra)
    # empty range: the "none" record still goes through the collective
    e = b.best_ordering_async(b.random(0, 0, seed=1))
    assert e.tolist() == [-1, -1]


@pytest.mark.parametrize("kind", ["random", "explicit"])
def test_best_ordering_owner_decode(kind):
    p, a, b = pair("C3")
    if kind == "random":
        ca, cb = a.random(100, 30_000, seed=3), b.random(100, 30_000, seed=3)
    else:
        rows = a.rows(a.random(0, 5000, seed=9)).cpu().numpy().astype(np.uint8)
        buf = np.zeros((5000, 80), np.uint8)
        buf[:, :p.T] = rows
        t = torch.tensor(buf, device="cuda")
        ca, cb = a.explicit(t, first=1000), b.explicit(t, first=1000)
    x, y = a.best_ordering(ca), b.best_ordering(cb)
    assert x["index"] == y["index"] and x["s1"] == y["s1"] and x["s2"] == y["s2"]
    assert x["n_over"] == y["n_over"]
    assert np.array_equal(x["queue_of_group"], y["queue_of_group"])
    assert np.array_equal(x["pos_of_group"], y["pos_of_group"])


def test_mc_counts_summed_through_nccl():
    p, a, b = pair("C4")
    row = balanced_row(p.G, p.Q)
    buf = np.zeros((1, p.row_stride // 2), np.int16)
    buf[0, :p.T] = row
    t = torch.tensor(buf, device="cuda")
    ca = a.mc_estimate(a.explicit(t), mc_seed=2, trials=300)
    cb = b.mc_estimate(b.explicit(t), mc_seed=2, trials=300)
    assert torch.equal(ca, cb) and int(ca.sum()) > 0


def test_local_search_sharded_by_the_library():
    p, a, b = pair("C3")
    start = np.arange(p.T)
    ba, ia = a.local_search(start, moves=2, per_iter=4096, iters=6, seed=11)
    bb, ib = b.local_search(start, moves=2, per_iter=4096, iters=6, seed=11)
    assert torch.equal(ba, bb) and torch.equal(ia, ib)


def test_local_search_graph_equals_direct_launches():
    # qlm_local_search captures its launches into a CUDA graph on a real
    # stream; the direct launches (override) give the same row and record,
    # and a second call (graph updated in place, new seed) matches too
    from paper_2407_00047_b200 import RwtEstimator, kernel_overrides
    p = make_config("C3")
    e = RwtEstimator(p, device=0)
    start = np.arange(p.T)
    s = torch.cuda.Stream()
    for stream in (s, torch.cuda.default_stream()):     # a side stream; the legacy default stream
      with torch.cuda.stream(stream):
        for seed in (5, 6):
            kernel_overrides()
            g_row, g_inc = e.local_search(start, moves=2, per_iter=8192, iters=12, seed=seed)
            kernel_overrides(no_graph=True)
            d_row, d_inc = e.local_search(start, moves=2, per_iter=8192, iters=12, seed=seed)
            kernel_overrides()
            torch.cuda.synchronize()
            assert torch.equal(g_row, d_row) and torch.equal(g_inc, d_inc)


@pytest.mark.parametrize("pinned", [True, False])
def test_winner_reads_the_record_into_host_buffers(pinned):
    # qlm_winner: the record's candidate scored + decoded on the stream, written
    # into host buffers (pinned: by the device directly; pageable: copies) --
    # equal to the synchronous qlm_best_ordering
    from paper_2407_00047_b200 import RwtEstimator
    p = make_config("C3")
    e = RwtEstimator(p, device=0)
    cand = e.random(0, 50_000, seed=2)
    rec = e.best_ordering_async(cand)
    mk = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
    host = {"best": mk(torch.full((24,), 0xAB, dtype=torch.uint8)),
            "qo": mk(torch.full((p.G,), -7, dtype=torch.int32)),
            "po": mk(torch.full((p.G,), -7, dtype=torch.int32))}
    e.winner(e.from_record(rec, seed=2), host)
    torch.cuda.synchronize()
    got = RwtEstimator.best_of(host["best"])
    ref = e.best_ordering(cand)
    assert got["index"] == ref["index"] and got["s1"] == ref["s1"] and got["s2"] == ref["s2"]
    assert got["n_over"] == ref["n_over"]
    assert np.array_equal(host["qo"].numpy(), ref["queue_of_group"])
    assert np.array_equal(host["po"].numpy(), ref["pos_of_group"])
