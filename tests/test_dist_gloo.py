"""World-size-2 gloo tests of the data-parallel plumbing (CPU, no GPU).

Each rank scores its contiguous shard of candidates (here with the oracle,
standing in for the kernel's per-rank record), the ranks exchange 16-byte
records with paper_2407_00047_b200.dist.global_best, and the merged winner
must equal the single-process argmin over all candidates.  MC counts of
disjoint trial ranges summed with dist.sum_counts must equal one full run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2407_00047_b200.dist import global_best, shard_range, sum_counts
from workloads.synth import make_config, balanced_row


def pack_key(s1, s2):
    """Host mirror of the record key (fp32 S1 bits, order-preserving fp32 S2)."""
    b1 = np.float32(s1).view(np.uint32).astype(np.uint64)
    f2 = np.float32(s2) + np.float32(0.0)
    b2 = int(np.float32(f2).view(np.uint32))
    b2 = (~b2 & 0xFFFFFFFF) if b2 & 0x80000000 else (b2 | 0x80000000)
    return int((int(b1) << 32) | b2)


def to_i64(u):
    return u - (1 << 64) if u >= 1 << 63 else u


def cpu_reduce(recs):
    """Lexicographic (unsigned key, index) min over gathered records."""
    r = recs.view(-1, 2).tolist()
    best = min(r, key=lambda kv: (kv[0] & ((1 << 64) - 1), kv[1] & ((1 << 64) - 1)))
    return torch.tensor(best, dtype=torch.int64)


def local_record(p, first, count):
    r = O.Oracle(p).score_range(O.RANDOM, first, count, seed=1)
    i = O.argmin_key(r["s1"], r["s2"])
    return torch.tensor([to_i64(pack_key(r["s1"][i], r["s2"][i])), first + i], dtype=torch.int64)


def _worker(rank, world, port, N, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = make_config("C2")
        first, count = shard_range(N, rank, world)
        rec = local_record(p, first, count)
        g = global_best(rec, cpu_reduce)
        # MC: disjoint trial ranges, counts summed across ranks
        p4 = make_config("C4")
        o4 = O.Oracle(p4)
        row = balanced_row(p4.G, p4.Q)[None, :]
        t0, nt = shard_range(60, rank, world)
        X = o4.mc_sample(2, t0, nt)
        cnt = torch.tensor(o4.mc_count(O.EXPLICIT, 0, 1, X, rows=row).astype(np.int64))
        sum_counts(cnt)
        q.put((rank, g.tolist(), cnt.numpy()))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_range_partitions():
    for N in [0, 1, 7, 1000, 10**8 + 3]:
        for W in [1, 2, 3, 4, 8]:
            parts = [shard_range(N, r, W) for r in range(W)]
            assert parts[0][0] == 0
            assert sum(c for _, c in parts) == N
            for (f0, c0), (f1, _) in zip(parts, parts[1:]):
                assert f0 + c0 == f1
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def test_pack_key_orders_lexicographically():
    rng = np.random.default_rng(0)
    s1 = rng.choice([0.0, 0.25, 0.5, 1.0], 200)
    s2 = rng.normal(0, 1e4, 200)
    s2[:5] = [0.0, -0.0, 1e-30, -1e-30, 5.0]
    keys = [pack_key(a, b) for a, b in zip(s1, s2)]
    order_k = sorted(range(200), key=lambda i: (keys[i], i))
    order_v = sorted(range(200), key=lambda i: (np.float32(s1[i]), np.float32(s2[i]) + np.float32(0), i))
    assert order_k == order_v


def test_two_rank_gloo_global_argmin_and_mc_sum():
    N, world = 6000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = make_config("C2")
    full = O.Oracle(p).score_range(O.RANDOM, 0, N, seed=1)
    want = O.argmin_key(full["s1"], full["s2"])
    for _, g, _ in res:
        assert g[1] == want
        assert g[0] == to_i64(pack_key(full["s1"][want], full["s2"][want]))
    p4 = make_config("C4")
    o4 = O.Oracle(p4)
    row = balanced_row(p4.G, p4.Q)[None, :]
    ref = o4.mc_count(O.EXPLICIT, 0, 1, o4.mc_sample(2, 0, 60), rows=row)
    for _, _, cnt in res:
        np.testing.assert_array_equal(cnt, ref.astype(np.int64))


# ------------------------------------------------- sharded local search (R18)
class OracleEstimator:
    """CPU stand-in for RwtEstimator in the plumbing test: the same method
    names dist.local_search calls, each computed with the oracle."""

    def __init__(self, p):
        self.p, self.o, self.T = p, O.Oracle(p), p.T

    def row_buffer(self, row):
        return torch.tensor(np.asarray(row, np.int64))

    def explicit(self, rows):
        return ("explicit", rows)

    def neighbor(self, base, first, count, seed, moves):
        return ("neighbor", base, first, count, seed, moves)

    def best_ordering_async(self, cand):
        if cand[0] == "explicit":
            s1, s2, _ = self.o.score(cand[1][0].numpy())
            return torch.tensor([to_i64(pack_key(s1, s2)), 0], dtype=torch.int64)
        _, base, first, count, seed, moves = cand
        if count == 0:
            return torch.tensor([-1, -1], dtype=torch.int64)
        r = self.o.score_range(O.NEIGHBOR, first, count, seed=seed, rows=base.numpy(), moves=moves)
        i = O.argmin_key(r["s1"], r["s2"])
        return torch.tensor([to_i64(pack_key(r["s1"][i], r["s2"][i])), first + i], dtype=torch.int64)

    def reduce_records(self, recs):
        return cpu_reduce(recs)

    def adopt_best(self, cand, rec, inc):
        _, base, _, _, seed, moves = cand
        u = lambda v: v & ((1 << 64) - 1)                                     # noqa: E731
        if rec[1] >= 0 and u(int(rec[0])) < u(int(inc[0])):
            base[:] = torch.tensor(O.neighbor_row(base.numpy(), seed, int(rec[1]), moves))
            inc[:] = rec


def _search_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_00047_b200.dist import local_search
        p = make_config("C1r")
        buf, inc = local_search(OracleEstimator(p), np.arange(p.T), moves=2, per_iter=13, iters=12,
                                seed=5)
        q.put((rank, buf.tolist(), inc.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_local_search():
    """Each iteration's candidates split over 2 ranks + global min-loc + the
    same adoption on every rank == the single-process oracle local search."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_search_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = make_config("C1r")
    row, key, _ = O.local_search(O.Oracle(p), np.arange(p.T), seed=5, moves=2, per_iter=13, iters=12)
    for _, b, inc in res:
        assert b == row.tolist()
        s1, s2, _ = O.Oracle(p).score(np.array(b))
        assert O.key32(s1, s2) == key


# ------------------------------------------------- sharded two-tier scoring (R20)
def _tier_worker(rank, world, port, N, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from workloads.synth import make_tiers
        p = make_config("C3")
        t = make_tiers()
        first, count = shard_range(N, rank, world)
        r = O.Oracle(p).tiered_range(t, O.RANDOM, first, count, seed=1, estimates=False)
        i = O.argmin_key(r["s1"], r["s2"])
        rec = torch.tensor([to_i64(pack_key(r["s1"][i], r["s2"][i])), first + i], dtype=torch.int64)
        g = global_best(rec, cpu_reduce)
        q.put((rank, g.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_tiered_argmin():
    """Two-tier scoring shards like plain scoring: per-rank records + one
    16-B min-loc exchange == the single-process tiered argmin."""
    N, world = 3000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_tier_worker, args=(r, world, port, N, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from workloads.synth import make_tiers
    p = make_config("C3")
    full = O.Oracle(p).tiered_range(make_tiers(), O.RANDOM, 0, N, seed=1, estimates=False)
    want = O.argmin_key(full["s1"], full["s2"])
    for _, g in res:
        assert g[1] == want


# ------------------------------------- the library's communicator: id plumbing
class _FakeCommEstimator:
    """Stands in for RwtEstimator: records what comm_attach receives."""

    def __init__(self):
        self.got = None
        self.comm_attached = False

    def comm_attach(self, uid, rank, world):
        self.got = (uid, rank, world)
        self.comm_attached = True


def _attach_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_00047_b200.dist import attach_comm
        est = _FakeCommEstimator()
        attach_comm(est, unique_id=lambda: bytes(range(7, 135)))
        rec = torch.tensor([1, 2], dtype=torch.int64)
        same = global_best(rec, cpu_reduce, est=est)        # records already global: identity
        cnt = torch.ones(3, dtype=torch.int64)
        sum_counts(cnt, est=est)                             # summed inside the C ABI: identity
        q.put((rank, est.got, same.tolist(), cnt.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_comm_id_broadcast():
    """attach_comm: rank 0's 128-byte NCCL unique id reaches every rank intact
    (torch.distributed carries only that), each rank attaches with its own
    (rank, world), and the Python exchange helpers become pass-throughs."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_attach_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, (uid, r, w), same, cnt in res:
        assert uid == bytes(range(7, 135)) and r == rank and w == world
        assert same == [1, 2] and cnt == [1, 1, 1]
