"""ctypes wrapper of the plain C fp64 oracle (oracle/qlm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg -- never by the product
package ``paper_2407_00047_b200``.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qlm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

EXPLICIT, RANDOM, ENUM, NEIGHBOR = 0, 1, 2, 3
Z_CLAMP = 8.0
ALPHA = 0.01


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Problem(C.Structure):
    _fields_ = [
        ("G", C.c_int32), ("Q", C.c_int32), ("D", C.c_int32), ("M", C.c_int32),
        ("model", C.c_void_p), ("n_req", C.c_void_p), ("slo", C.c_void_p),
        ("mu", C.c_void_p), ("var", C.c_void_p), ("dist", C.c_void_p),
        ("q_device", C.c_void_p), ("q_resident", C.c_void_p),
        ("q_bmean", C.c_void_p), ("q_bvar", C.c_void_p),
        ("theta", C.c_void_p), ("prefill", C.c_void_p), ("eps", C.c_void_p),
        ("dtok", C.c_void_p), ("max_out", C.c_void_p), ("swap", C.c_void_p),
        ("K", C.c_int32), ("n_tables", C.c_int32), ("len", C.c_void_p),
        ("z_clamp", C.c_double), ("alpha", C.c_double),
    ]


class _Tiers(C.Structure):
    _fields_ = [("mem", C.c_void_p), ("cap", C.c_void_p), ("load", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER(_Problem)
        vp, i32, i64, u64, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
        _lib.or_philox4x32_10.argtypes = [vp, vp, vp]
        _lib.or_random_row.argtypes = [u64, u64, i32, vp]
        _lib.or_enum_row.argtypes = [u64, i32, vp]
        _lib.or_neighbor_row.argtypes = [vp, i32, u64, u64, i32, vp]
        _lib.or_estimate_row.argtypes = [P, vp, dp, dp, vp, vp]
        _lib.or_estimate_row.restype = C.c_int
        _lib.or_violation.argtypes = [C.c_double] * 4
        _lib.or_violation.restype = C.c_double
        _lib.or_score_row.argtypes = [P, vp, dp, dp, vp]
        _lib.or_score_row.restype = C.c_int
        _lib.or_score_range.argtypes = [P, C.c_int, vp, i32, i64, u64, u64, i64, dp, dp, vp]
        _lib.or_score_range.restype = i64
        _lib.or_estimate_range.argtypes = [P, C.c_int, vp, i32, i64, u64, u64, i64, dp, dp, dp]
        _lib.or_estimate_range.restype = i64
        _lib.or_mc_sample.argtypes = [P, u64, i64, i64, vp]
        _lib.or_request_violations_row.argtypes = [P, vp, dp, dp]
        _lib.or_request_violations_row.restype = C.c_int
        _lib.or_request_violations_range.argtypes = [P, C.c_int, vp, i32, i64, u64, u64, i64, dp, dp]
        _lib.or_request_violations_range.restype = i64
        _lib.or_mc_count.argtypes = [P, C.c_int, vp, i32, i64, u64, u64, i64, vp, i64, vp]
        _lib.or_mc_count.restype = i64
        T = C.POINTER(_Tiers)
        _lib.or_estimate_row_tiered.argtypes = [P, T, vp, dp, dp, vp]
        _lib.or_estimate_row_tiered.restype = C.c_int
        _lib.or_score_row_tiered.argtypes = [P, T, vp, dp, dp, vp, dp, dp]
        _lib.or_score_row_tiered.restype = C.c_int
        _lib.or_tiered_range.argtypes = [P, T, C.c_int, vp, i32, i64, u64, u64, i64, dp, dp, vp, dp, dp]
        _lib.or_tiered_range.restype = i64
        _lib.or_mc_count_tiered.argtypes = [P, T, C.c_int, vp, i32, i64, u64, u64, i64, vp, i64, vp]
        _lib.or_mc_count_tiered.restype = i64
        _lib.or_form_groups.argtypes = [i32, i32, vp, vp, vp, vp, i32, vp, i32, i32,
                                        vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp]
        _lib.or_form_groups.restype = i32
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Oracle bound to one workloads.Problem (arrays kept alive here)."""

    def __init__(self, prob, z_clamp: float = Z_CLAMP, alpha: float = ALPHA):
        self.prob = prob
        c = np.ascontiguousarray
        self._keep = dict(
            model=c(prob.model, np.int32), n_req=c(prob.n_req, np.int32),
            slo=c(prob.slo, np.float64), mu=c(prob.mu, np.float64), var=c(prob.var, np.float64),
            dist=c(prob.dist, np.int32), q_device=c(prob.q_device, np.int32),
            q_resident=c(prob.q_resident, np.int32), q_bmean=c(prob.q_backlog_mean, np.float64),
            q_bvar=c(prob.q_backlog_var, np.float64), theta=c(prob.theta, np.float64),
            prefill=c(prob.prefill, np.float64), eps=c(prob.eps, np.float64),
            dtok=c(prob.dtok, np.float64), max_out=c(prob.max_out, np.float64),
            swap=c(prob.swap, np.float64),
        )
        tabs = prob.len_tables
        if tabs is not None:
            tabs = c(tabs, np.uint16)
            self._keep["len"] = tabs
        k = self._keep
        self.p = _Problem(
            prob.G, prob.Q, prob.D, prob.M,
            *[_ptr(k[n]) for n in ("model", "n_req", "slo", "mu", "var", "dist", "q_device",
                                   "q_resident", "q_bmean", "q_bvar", "theta", "prefill", "eps",
                                   "dtok", "max_out", "swap")],
            0 if tabs is None else tabs.shape[1], 0 if tabs is None else tabs.shape[0],
            _ptr(tabs), z_clamp, alpha)
        self.G, self.Q, self.T = prob.G, prob.Q, prob.T

    # -- rows --------------------------------------------------------------
    def random_row(self, seed: int, c: int) -> np.ndarray:
        return random_row(seed, c, self.T)

    def enum_row(self, c: int) -> np.ndarray:
        return enum_row(c, self.T)

    # -- single ordering -----------------------------------------------------
    def estimate(self, row):
        row = np.ascontiguousarray(row, np.int32)
        G = self.G
        wt, V = np.zeros(G), np.zeros(G)
        q, pos = np.zeros(G, np.int32), np.zeros(G, np.int32)
        rc = lib().or_estimate_row(C.byref(self.p), _ptr(row), _ptr(wt), _ptr(V), _ptr(q), _ptr(pos))
        if rc != 0:
            raise ValueError("row is not a permutation of 0..T-1 (Eq. 6)")
        return dict(wt=wt, V=V, queue=q, pos=pos)

    def score(self, row):
        row = np.ascontiguousarray(row, np.int32)
        s1, s2, no = C.c_double(), C.c_double(), C.c_int32()
        rc = lib().or_score_row(C.byref(self.p), _ptr(row), C.byref(s1), C.byref(s2), C.byref(no))
        if rc != 0:
            raise ValueError("row is not a permutation of 0..T-1 (Eq. 6)")
        return s1.value, s2.value, no.value

    # -- ranges --------------------------------------------------------------
    def _rows_args(self, kind, rows, moves=0):
        if kind == EXPLICIT:
            rows = np.ascontiguousarray(rows)
            return rows, rows.dtype.itemsize, rows.strides[0]
        if kind == NEIGHBOR:         # rows = base row (uint8 / uint16), stride slot = moves
            rows = np.ascontiguousarray(rows, np.uint16)
            return rows, 2, int(moves)
        return None, 1, 0

    def neighbor_row(self, base, seed: int, c: int, moves: int) -> np.ndarray:
        return neighbor_row(base, seed, c, moves)

    def score_range(self, kind, first, count, seed=0, rows=None, moves=0):
        rows, tb, stride = self._rows_args(kind, rows, moves)
        s1, s2, no = np.zeros(count), np.zeros(count), np.zeros(count, np.int32)
        bad = lib().or_score_range(C.byref(self.p), kind, _ptr(rows), tb, stride, seed, first,
                                   count, _ptr(s1), _ptr(s2), _ptr(no))
        return dict(s1=s1, s2=s2, n_over=no, bad=bad)

    def estimate_range(self, kind, first, count, seed=0, rows=None, moves=0):
        rows, tb, stride = self._rows_args(kind, rows, moves)
        G = self.G
        wt, sd, v = np.zeros((count, G)), np.zeros((count, G)), np.zeros((count, G))
        bad = lib().or_estimate_range(C.byref(self.p), kind, _ptr(rows), tb, stride, seed, first,
                                      count, _ptr(wt), _ptr(sd), _ptr(v))
        return dict(wt=wt, sd=sd, v=v, bad=bad)

    def request_violations(self, row):
        """R19: per-group violating fraction over the group's requests, and S1_req."""
        row = np.ascontiguousarray(row, np.int32)
        frac, s1 = np.zeros(self.G), C.c_double()
        if lib().or_request_violations_row(C.byref(self.p), _ptr(row), _ptr(frac), C.byref(s1)) != 0:
            raise ValueError("row is not a permutation of 0..T-1 (Eq. 6)")
        return frac, s1.value

    def request_violations_range(self, kind, first, count, seed=0, rows=None, moves=0):
        rows, tb, stride = self._rows_args(kind, rows, moves)
        frac, s1 = np.zeros((count, self.G)), np.zeros(count)
        bad = lib().or_request_violations_range(C.byref(self.p), kind, _ptr(rows), tb, stride, seed,
                                                first, count, _ptr(frac), _ptr(s1))
        return dict(frac=frac, s1=s1, bad=bad)

    # -- two-tier model swapping (R20) -------------------------
    def _tiers(self, tiers):
        """tiers: dict(mem=int32 [M], cap=int32 [D], load=f64 [D, M]) (workloads.make_tiers)."""
        k = (np.ascontiguousarray(tiers["mem"], np.int32), np.ascontiguousarray(tiers["cap"], np.int32),
             np.ascontiguousarray(tiers["load"], np.float64))
        return k, _Tiers(*[_ptr(a) for a in k])

    def estimate_tiered(self, row, tiers):
        row = np.ascontiguousarray(row, np.int32)
        keep, t = self._tiers(tiers)
        wt, V, cold = np.zeros(self.G), np.zeros(self.G), np.zeros(self.G, np.int32)
        if lib().or_estimate_row_tiered(C.byref(self.p), C.byref(t), _ptr(row), _ptr(wt), _ptr(V),
                                        _ptr(cold)) != 0:
            raise ValueError("row is not a permutation of 0..T-1 (Eq. 6)")
        return dict(wt=wt, V=V, cold=cold)

    def score_tiered(self, row, tiers):
        row = np.ascontiguousarray(row, np.int32)
        keep, t = self._tiers(tiers)
        s1, s2, no = C.c_double(), C.c_double(), C.c_int32()
        if lib().or_score_row_tiered(C.byref(self.p), C.byref(t), _ptr(row), C.byref(s1), C.byref(s2),
                                     C.byref(no), None, None) != 0:
            raise ValueError("row is not a permutation of 0..T-1 (Eq. 6)")
        return s1.value, s2.value, no.value

    def tiered_range(self, tiers, kind, first, count, seed=0, rows=None, moves=0, estimates=True):
        rows, tb, stride = self._rows_args(kind, rows, moves)
        keep, t = self._tiers(tiers)
        G = self.G
        s1, s2, no = np.zeros(count), np.zeros(count), np.zeros(count, np.int32)
        wt = np.zeros((count, G)) if estimates else None
        V = np.zeros((count, G)) if estimates else None
        bad = lib().or_tiered_range(C.byref(self.p), C.byref(t), kind, _ptr(rows), tb, stride, seed,
                                    first, count, _ptr(s1), _ptr(s2), _ptr(no), _ptr(wt), _ptr(V))
        out = dict(s1=s1, s2=s2, n_over=no, bad=bad)
        if estimates:
            out.update(wt=wt, V=V, sd=np.sqrt(V),
                       v=np.array([[violation(wt[k, i], V[k, i], self.prob.slo[i]) for i in range(G)]
                                   for k in range(count)]) if count * G <= 2000000 else None)
        return out

    def mc_count_tiered(self, tiers, kind, first, count, X, seed=0, rows=None, moves=0):
        """MC counts under two-tier swapping (R13 + R20)."""
        rows, tb, stride = self._rows_args(kind, rows, moves)
        keep, t = self._tiers(tiers)
        X = np.ascontiguousarray(X, np.uint32)
        counts = np.zeros((count, self.G), np.uint32)
        bad = lib().or_mc_count_tiered(C.byref(self.p), C.byref(t), kind, _ptr(rows), tb, stride, seed,
                                       first, count, _ptr(X), X.shape[0], _ptr(counts))
        if bad:
            raise ValueError(f"{bad} invalid rows")
        return counts

    def mc_sample(self, mc_seed, trial_first, trial_count):
        X = np.zeros((trial_count, self.G), np.uint32)
        lib().or_mc_sample(C.byref(self.p), mc_seed, trial_first, trial_count, _ptr(X))
        return X

    def mc_count(self, kind, first, count, X, seed=0, rows=None, moves=0):
        rows, tb, stride = self._rows_args(kind, rows, moves)
        X = np.ascontiguousarray(X, np.uint32)
        counts = np.zeros((count, self.G), np.uint32)
        bad = lib().or_mc_count(C.byref(self.p), kind, _ptr(rows), tb, stride, seed, first, count,
                                _ptr(X), X.shape[0], _ptr(counts))
        if bad:
            raise ValueError(f"{bad} invalid rows")
        return counts


def form_groups(req: dict, M: int, k_per_model, limit: int, max_iter: int = 50) -> dict:
    """Alg. 1 under reading R21: k-means per model + recursive
    splitHalf.  req: dict(model int32 [n], slo f64 [n], out int32 [n],
    feat int32 [n, dims]) in arrival order (workloads.make_requests)."""
    c = np.ascontiguousarray
    model, slo = c(req["model"], np.int32), c(req["slo"], np.float64)
    out, feat = c(req["out"], np.int32), c(req["feat"], np.int32)
    n, dims = feat.shape
    k = c(k_per_model, np.int32)
    label, gof = np.zeros(n, np.int32), np.zeros(n, np.int32)
    cap = n
    gm, gn = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    gs, gmu, gvar = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    iters, keff = C.c_int32(), np.zeros(M, np.int32)
    init = np.full(max(1, int(np.sum(k))), -1, np.int32)
    G = lib().or_form_groups(n, dims, _ptr(model), _ptr(slo), _ptr(out), _ptr(feat), M, _ptr(k), limit,
                             max_iter, _ptr(label), _ptr(gof), _ptr(gm), _ptr(gn), _ptr(gs), _ptr(gmu),
                             _ptr(gvar), cap, C.byref(iters), _ptr(keff), _ptr(init))
    if G < 0:
        raise ValueError("invalid requests (model or feature out of range)")
    return dict(n_groups=G, label=label, group_of=gof, model=gm[:G], n=gn[:G], slo=gs[:G], mu=gmu[:G],
                var=gvar[:G], iters=iters.value, k_eff=keff, init=init[:int(keff.sum())])


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def random_row(seed: int, c: int, T: int) -> np.ndarray:
    row = np.zeros(T, np.int32)
    lib().or_random_row(seed, c, T, _ptr(row))
    return row


def neighbor_row(base, seed: int, c: int, moves: int) -> np.ndarray:
    """R18: the base row with `moves` Philox-drawn transpositions."""
    b = np.ascontiguousarray(base, np.int32)
    row = np.zeros(len(b), np.int32)
    lib().or_neighbor_row(_ptr(b), len(b), seed, c, moves, _ptr(row))
    return row


def key32(s1: float, s2: float):
    """The objective key of R11 as a comparable tuple (fp32 S1, fp32 S2)."""
    return (float(np.float32(s1)), float(np.float32(s2)))


def local_search(o: "Oracle", start_row, seed: int, moves: int, per_iter: int, iters: int):
    """SURVEY 8(f) N1 as plain iterated best-of-N: each iteration scores the
    per_iter NEIGHBOR candidates [it*per_iter, (it+1)*per_iter) of the
    incumbent (R18) and adopts the lexicographic argmin (R11/R14) if its key
    beats the incumbent's.  Returns (row, key, number of adoptions)."""
    inc = np.ascontiguousarray(start_row, np.int32)
    s1, s2, _ = o.score(inc)
    inc_key = key32(s1, s2)
    adopted = 0
    for it in range(iters):
        r = o.score_range(NEIGHBOR, it * per_iter, per_iter, seed=seed, rows=inc, moves=moves)
        i = argmin_key(r["s1"], r["s2"])
        k = key32(r["s1"][i], r["s2"][i])
        if k < inc_key:
            inc = neighbor_row(inc, seed, it * per_iter + i, moves)
            inc_key = k
            adopted += 1
    return inc, inc_key, adopted


def enum_row(c: int, T: int) -> np.ndarray:
    row = np.zeros(T, np.int32)
    lib().or_enum_row(c, T, _ptr(row))
    return row


def violation(wt, V, slo, z_clamp=Z_CLAMP):
    return lib().or_violation(wt, V, slo, z_clamp)


def argmin_key(s1: np.ndarray, s2: np.ndarray) -> int:
    """Lexicographic argmin over (fp32(S1), fp32(S2), index) -- R11/R14."""
    f1 = s1.astype(np.float32)
    f2 = s2.astype(np.float32)
    order = np.lexsort((np.arange(len(f1)), f2, f1))
    return int(order[0])
