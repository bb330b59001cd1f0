"""Seeded synthetic QLM scheduling problems.

Only raw problem descriptions are drawn here -- nothing of the RWT estimator's
arithmetic.  Every number the paper does not give is [SYNTHETIC]; the
structure follows the paper's workloads:

* three SLO classes, 20 s / 1 min / 1 h p99 TTFT,
  mixed 0.2 / 0.3 / 0.5 [SYNTHETIC mix];
* request-group sizes by class: interactive U{16..64}, batch-1 U{64..256},
  batch-2 U{256..1024}; delta = 4 x batch 64 = 256 for the MC config
  (PAPER.md L1063-1070);
* models 7B / 13B / 70B-a / 70B-b on A100-like
  and A10-like devices;
* ShareGPT-shaped output lengths (histogram only):
  truncated lognormal quantile tables, K = 4096 entries, clamp [1, 2048]
  (SPEC.md L161), mean 300 * s_model * s_class, cv 0.83;
* profile constants P, eps, d, max_out per (device, model) (PAPER.md
  Table tab:symbols_rwt L568-588; SPEC.md L287 uses eps 1.2, d 0.025,
  max_out 2048) and swap times with ~20 s for a 70B model.

The group statistics mu / var are the exact mean / population variance of the
group's length table: that is workload profiling ("fitted from the request
input-output history dataset"), which is outside the hot path.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
from scipy.special import ndtri

WORKLOAD_SEED = 20240701
CANDIDATE_SEED = 1
MC_SEED = 2

SLO_CLASSES = (20.0, 60.0, 3600.0)
SLO_MIX = (0.2, 0.3, 0.5)
N_RANGE = ((16, 64), (64, 256), (256, 1024))

# App. B of SURVEY.md -- [SYNTHETIC] A100-like (d0) and A10-like (d1) rows.
THETA = np.array([[3000.0, 1800.0, 900.0, 900.0],
                  [1000.0, 500.0, 150.0, 150.0]])
DTOK = np.array([[0.015, 0.025, 0.050, 0.050],
                 [0.030, 0.050, 0.100, 0.100]])
PREFILL = np.array([[0.1, 0.2, 0.5, 0.5],
                    [0.2, 0.4, 1.0, 1.0]])
EPS = 1.2
MAX_OUT = 2048.0
SWAP_TO = np.array([[2.0, 4.0, 20.0, 20.0],
                    [3.0, 6.0, 30.0, 30.0]])
S_MODEL = (1.0, 1.0, 1.2, 1.2)
S_CLASS = (0.5, 1.0, 1.5)
LEN_K = 4096
LEN_CV = 0.83


@dataclasses.dataclass
class Problem:
    """Raw inputs of one scheduling problem (Table 3)."""
    name: str
    model: np.ndarray        # int32 [G]   model of request group i (Eq. 7)
    n_req: np.ndarray        # int32 [G]   requests in group i
    slo: np.ndarray          # f64  [G]   TTFT deadline, s (Def. 2, Eq. 8)
    mu: np.ndarray           # f64  [G]   mean output tokens (Eq. 3)
    var: np.ndarray          # f64  [G]   variance of output tokens (Eq. 3)
    dist: np.ndarray         # int32 [G]  length-table id for MC, -1 = none
    q_device: np.ndarray     # int32 [Q]  device-type row of each queue
    q_resident: np.ndarray   # int32 [Q]  model loaded at t = 0 (Def. 3)
    q_backlog_mean: np.ndarray  # f64 [Q] in-flight work pinned ahead, s
    q_backlog_var: np.ndarray   # f64 [Q]
    theta: np.ndarray        # f64 [D, M] tokens/s (Eq. 2)
    prefill: np.ndarray      # f64 [D, M] P, s (Eq. 1)
    eps: np.ndarray          # f64 [D, M] inefficiency factor (Eq. 4)
    dtok: np.ndarray         # f64 [D, M] decode time per token d, s (Eq. 4)
    max_out: np.ndarray      # f64 [D, M] max output tokens (Eq. 4 bound)
    swap: np.ndarray         # f64 [D, M, M] swap time from -> to, s
    len_tables: np.ndarray | None = None  # uint16 [n_tables, K]

    @property
    def G(self) -> int:
        return int(self.model.shape[0])

    @property
    def Q(self) -> int:
        return int(self.q_device.shape[0])

    @property
    def D(self) -> int:
        return int(self.theta.shape[0])

    @property
    def M(self) -> int:
        return int(self.theta.shape[1])

    @property
    def T(self) -> int:
        """Tokens per candidate row: G group tokens + (Q-1) queue separators."""
        return self.G + self.Q - 1

    @property
    def token_bytes(self) -> int:
        return 1 if self.T <= 256 else 2

    @property
    def row_stride(self) -> int:
        return -(-self.T * self.token_bytes // 16) * 16


def length_table(mean: float, cv: float = LEN_CV, K: int = LEN_K,
                 lo: int = 1, hi: int = 2048) -> np.ndarray:
    """Quantile table of a truncated lognormal, uint16 [K]."""
    s2 = math.log1p(cv * cv)
    m = math.log(mean) - 0.5 * s2
    p = (np.arange(K, dtype=np.float64) + 0.5) / K
    x = np.exp(m + math.sqrt(s2) * ndtri(p))
    return np.clip(np.rint(x), lo, hi).astype(np.uint16)


def all_length_tables() -> np.ndarray:
    """12 tables, id = model * 3 + slo_class."""
    return np.stack([length_table(300.0 * sm * sc) for sm in S_MODEL for sc in S_CLASS])


def table_moments(tab: np.ndarray) -> tuple[float, float]:
    x = tab.astype(np.float64)
    mu = float(x.mean())
    return mu, float(((x - mu) ** 2).mean())


def _profile(D_rows, models):
    D_rows = list(D_rows)
    models = list(models)
    theta = THETA[np.ix_(D_rows, models)].copy()
    dtok = DTOK[np.ix_(D_rows, models)].copy()
    prefill = PREFILL[np.ix_(D_rows, models)].copy()
    eps = np.full_like(theta, EPS)
    max_out = np.full_like(theta, MAX_OUT)
    M = len(models)
    swap = np.zeros((len(D_rows), M, M))
    for di, d in enumerate(D_rows):
        for a in range(M):
            for b in range(M):
                if a != b:
                    swap[di, a, b] = SWAP_TO[d, models[b]]
    return theta, prefill, eps, dtok, max_out, swap


def make_problem(G: int, Q: int, models=(0, 1, 2, 3), *, seed: int = WORKLOAD_SEED,
                 n_fixed: int | None = None, q_devices=None, name: str = "",
                 backlog: bool = False) -> Problem:
    """App. B workload: G groups over len(models) models, Q A100-like queues.

    ``q_devices`` maps each queue to a device row (0 = A100-like, 1 = A10-like).
    """
    rng = np.random.default_rng(seed)
    M = len(models)
    q_devices = np.zeros(Q, np.int32) if q_devices is None else np.asarray(q_devices, np.int32)
    dev_rows = sorted(set(int(d) for d in q_devices))
    dev_index = {d: i for i, d in enumerate(dev_rows)}
    theta, prefill, eps, dtok, max_out, swap = _profile(dev_rows, models)
    tabs = all_length_tables()
    cls = rng.choice(3, size=G, p=SLO_MIX)
    model = rng.integers(0, M, size=G).astype(np.int32)
    if n_fixed is None:
        n = np.array([rng.integers(N_RANGE[c][0], N_RANGE[c][1] + 1) for c in cls], np.int32)
    else:
        n = np.full(G, n_fixed, np.int32)
    dist = (np.array([models[m] for m in model]) * 3 + cls).astype(np.int32)
    mom = [table_moments(tabs[k]) for k in dist]
    mu = np.array([m for m, _ in mom])
    var = np.array([v for _, v in mom])
    slo = np.array([SLO_CLASSES[c] for c in cls])
    bm = np.zeros(Q)
    bv = np.zeros(Q)
    if backlog:
        bm = rng.uniform(0.0, 30.0, Q) * (rng.random(Q) < 0.5)
        bv = np.where(bm > 0, rng.uniform(0.0, 4.0, Q), 0.0)
    return Problem(
        name=name or f"G{G}Q{Q}M{M}",
        model=model, n_req=n, slo=slo, mu=mu, var=var, dist=dist,
        q_device=np.array([dev_index[int(d)] for d in q_devices], np.int32),
        q_resident=(np.arange(Q) % M).astype(np.int32),
        q_backlog_mean=bm, q_backlog_var=bv,
        theta=theta, prefill=prefill, eps=eps, dtok=dtok, max_out=max_out, swap=swap,
        len_tables=tabs,
    )


def make_golden_c1() -> Problem:
    """C1 hand-checkable instance: 1 model, 1 queue.

    Theta 1000 tok/s, mu 200, sigma^2 1e4, n = (25, 40, 10, 50),
    slo = (12, 20, 4, 30) s.  Profile constants are SPEC.md L287's.
    """
    G = 4
    return Problem(
        name="C1",
        model=np.zeros(G, np.int32), n_req=np.array([25, 40, 10, 50], np.int32),
        slo=np.array([12.0, 20.0, 4.0, 30.0]), mu=np.full(G, 200.0), var=np.full(G, 1e4),
        dist=np.full(G, -1, np.int32),
        q_device=np.zeros(1, np.int32), q_resident=np.zeros(1, np.int32),
        q_backlog_mean=np.zeros(1), q_backlog_var=np.zeros(1),
        theta=np.array([[1000.0]]), prefill=np.array([[0.5]]), eps=np.array([[1.2]]),
        dtok=np.array([[0.025]]), max_out=np.array([[2048.0]]), swap=np.zeros((1, 1, 1)),
        len_tables=None,
    )


def make_random_problem(rng: np.random.Generator, G: int, Q: int, M: int, D: int = 1, *,
                        sigma_zero: bool = False, backlog: bool = False,
                        with_tables: bool = False, name: str = "rand") -> Problem:
    """Generic random instance with random (not App. B) profile constants.

    Used by parity tests to exercise shapes and corner cases the App. B
    configs do not reach (several device types, backlogs, sigma = 0).
    """
    theta = rng.uniform(100.0, 4000.0, (D, M))
    prefill = rng.uniform(0.05, 1.0, (D, M))
    eps = rng.uniform(1.0, 1.5, (D, M))
    dtok = rng.uniform(0.005, 0.06, (D, M))
    max_out = rng.choice([512.0, 1024.0, 2048.0, 4096.0], (D, M))
    swap = rng.uniform(0.5, 30.0, (D, M, M))
    for d in range(D):
        np.fill_diagonal(swap[d], 0.0)
    model = rng.integers(0, M, G).astype(np.int32)
    n = rng.integers(1, 600, G).astype(np.int32)
    mu = rng.uniform(20.0, 600.0, G)
    var = np.zeros(G) if sigma_zero else (rng.uniform(0.1, 1.0, G) * mu) ** 2
    slo = rng.choice([20.0, 60.0, 3600.0], G) * rng.uniform(0.2, 2.0, G)
    tabs = None
    dist = np.full(G, -1, np.int32)
    if with_tables:
        tabs = np.stack([length_table(float(m), cv=0.8, K=1024) for m in (80.0, 200.0, 450.0)])
        dist = rng.integers(0, 3, G).astype(np.int32)
        mom = [table_moments(tabs[k]) for k in dist]
        mu = np.array([a for a, _ in mom])
        var = np.array([b for _, b in mom])
    bm = np.zeros(Q)
    bv = np.zeros(Q)
    if backlog:
        bm = rng.uniform(0.0, 40.0, Q) * (rng.random(Q) < 0.6)
        bv = np.where(bm > 0, rng.uniform(0.0, 9.0, Q), 0.0)
    return Problem(
        name=name, model=model, n_req=n, slo=slo, mu=mu, var=var, dist=dist,
        q_device=rng.integers(0, D, Q).astype(np.int32),
        q_resident=rng.integers(0, M, Q).astype(np.int32),
        q_backlog_mean=bm, q_backlog_var=bv,
        theta=theta, prefill=prefill, eps=eps, dtok=dtok, max_out=max_out, swap=swap,
        len_tables=tabs,
    )


def balanced_row(G: int, Q: int) -> np.ndarray:
    """Token row placing group i in queue i mod Q, ascending within a queue.

    Tokens < G are group ids; tokens >= G are queue separators ("bars").
    """
    toks = []
    for q in range(Q):
        toks.extend(range(q, G, Q))
        if q < Q - 1:
            toks.append(G + q)
    T = G + Q - 1
    dt = np.uint8 if T <= 256 else np.uint16
    return np.asarray(toks, dtype=dt)


def queue_row(order, G: int, Q: int, queue_of=None) -> np.ndarray:
    """Token row from a group order: group order[k] goes to queue queue_of[k]
    (default k mod Q), keeping the order within each queue."""
    qs = [[] for _ in range(Q)]
    for k, g in enumerate(order):
        qs[(k % Q) if queue_of is None else int(queue_of[k])].append(int(g))
    toks = []
    for q in range(Q):
        toks.extend(qs[q])
        if q < Q - 1:
            toks.append(G + q)
    T = G + Q - 1
    return np.asarray(toks, dtype=np.uint8 if T <= 256 else np.uint16)


def fcfs_row(p: "Problem") -> np.ndarray:
    """Comparator: groups in arrival (index) order, dealt round-robin over the
    queues (FCFS baseline of P:L790-791)."""
    return queue_row(range(p.G), p.G, p.Q)


def edf_row(p: "Problem") -> np.ndarray:
    """Comparator: earliest deadline (SLO) first, dealt round-robin over the
    queues (EDF baseline of P:L790-791)."""
    return queue_row(np.argsort(p.slo, kind="stable"), p.G, p.Q)


# Two-tier model swapping (R20) [SYNTHETIC]:
# fp16 weights (2 B/param) of the 7B / 13B / 70B-like models, the host CPU
# memory an A100-like / A10-like instance can give to warm models, and the
# registry (storage) read bandwidth that a cold model pays before its swap.
MODEL_MEM_GB = (14, 26, 140, 140)
CPU_CAP_GB = (200, 96)
DISK_GBPS = (2.0, 1.0)


def make_tiers(models=(0, 1, 2, 3), dev_rows=(0,)) -> dict:
    """Tier inputs of qlm_set_tiers / the oracle: mem int32 [M] (GB), cap int32
    [D] (GB), load f64 [D, M] = mem / disk bandwidth (s)."""
    mem = np.array([MODEL_MEM_GB[m] for m in models], np.int32)
    cap = np.array([CPU_CAP_GB[d] for d in dev_rows], np.int32)
    load = np.array([[MODEL_MEM_GB[m] / DISK_GBPS[d] for m in models] for d in dev_rows])
    return dict(mem=mem, cap=cap, load=load)


def make_random_tiers(rng: np.random.Generator, M: int, D: int) -> dict:
    """Random tier inputs: sizes 1..40 units, budgets 0..(sum of sizes), loads 0..60 s."""
    mem = rng.integers(1, 41, M).astype(np.int32)
    cap = rng.integers(0, int(mem.sum()) + 1, D).astype(np.int32)
    load = rng.uniform(0.0, 60.0, (D, M))
    return dict(mem=mem, cap=cap, load=load)


# Request-group formation (R21; Alg. 1) [SYNTHETIC]:
# requests in arrival order with a model, an SLO class, an input length and
# an output length drawn from the (model, class) length table (the
# "input-output history").  Features (Def. P:L443-447: SLO, input /
# output token distribution) are quantised logs: round(4096 * log2(x)),
# which keeps every coordinate in [0, 65535] for x <= 2^15.
FEAT_SCALE = 4096.0
GROUP_LIMIT = 256          # delta = 4 x average batch 64


def make_requests(n: int, models=(0, 1, 2, 3), *, seed: int = WORKLOAD_SEED) -> dict:
    rng = np.random.default_rng(seed + 17)
    tabs = all_length_tables()
    M = len(models)
    model = rng.integers(0, M, n).astype(np.int32)
    cls = rng.choice(3, size=n, p=SLO_MIX)
    slo = np.array(SLO_CLASSES)[cls]
    in_len = np.clip(np.rint(np.exp(rng.normal(math.log(400.0), 0.9, n))), 1, 8192)
    dist = np.array(models)[model] * 3 + cls
    out = tabs[dist, rng.integers(0, tabs.shape[1], n)].astype(np.int32)
    cls_mean = np.array([table_moments(tabs[k])[0] for k in range(len(tabs))])[dist]
    feat = np.stack([np.rint(FEAT_SCALE * np.log2(x)) for x in (slo, in_len, cls_mean)], 1).astype(np.int32)
    return dict(model=model, slo=slo, out=out, feat=feat, in_len=in_len.astype(np.int32))


# name -> (problem factory, candidate kind, candidate count / trials)
CONFIGS = {
    "C1": dict(desc="4 groups, 1 model, 1 queue: all 24 orderings (ENUM)",
               kind="enum", count=24),
    "C1r": dict(desc="C1 shape with seeded App. B values", kind="enum", count=24),
    "C2": dict(desc="16 groups x 2 models x 2 queues, 1e5 RANDOM candidates",
               kind="random", count=100_000),
    "C3": dict(desc="64 groups, 4 models, 8 queues, 1e6 RANDOM candidates",
               kind="random", count=1_000_000),
    "C4": dict(desc="MC: 256 groups (n=256), 8 queues, 1221 trials on the balanced ordering",
               kind="mc", count=1, trials=1221),
    "C5": dict(desc="1024 groups, 32 queues, 1e8 RANDOM candidates", kind="random",
               count=100_000_000),
    "C5h": dict(desc="C5 with queues 24-31 A10-like", kind="random", count=100_000_000),
}


def make_config(name: str) -> Problem:
    if name == "C1":
        return make_golden_c1()
    if name == "C1r":
        return make_problem(4, 1, models=(0,), name="C1r")
    if name == "C2":
        return make_problem(16, 2, models=(0, 2), name="C2")
    if name == "C3":
        return make_problem(64, 8, name="C3")
    if name == "C4":
        return make_problem(256, 8, n_fixed=256, name="C4")
    if name == "C5":
        return make_problem(1024, 32, name="C5")
    if name == "C5h":
        return make_problem(1024, 32, q_devices=[0] * 24 + [1] * 8, name="C5h")
    raise KeyError(name)
