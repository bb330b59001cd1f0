"""Python binding of libqlm: bulk RWT estimation over candidate queue orderings.

Thin marshalling over include/qlm.h -- every step of the path runs in the
CUDA kernels of csrc/.  torch provides device memory and streams only.

    est = RwtEstimator(problem, device=0)          # qlm_create (a0)
    cand = est.random(first=0, count=10**6, seed=1)
    best = est.best_ordering(cand)                  # a1-a5, a7, a9
    wt, sd, v = est.rwt_estimate(cand)              # a6 bulk per-(candidate, group)
    counts = est.mc_estimate(est.from_record(rec), mc_seed=2, trials=1221)   # a10-a11

Citations: PAPER.md Sec. 6 (RWT estimator, L564-664) and Sec. 7 (global
scheduler objective, L665-767); readings R1-R14 in DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np
import torch

from . import _lib as L


@dataclasses.dataclass
class Cand:
    """A set of candidate orderings (qlm_candidates, R10)."""
    kind: int
    first: int = 0
    count: int = 0
    seed: int = 0
    rows: torch.Tensor | None = None        # EXPLICIT: uint8/int16 device [count, stride]
                                            # NEIGHBOR: the base row, uint8/int16 device [>= T]
    first_from: torch.Tensor | None = None  # device record (int64[2]); count must be 1
    moves: int = 0                          # NEIGHBOR: transpositions per candidate (R18)

    def c(self) -> L.Candidates:
        tb, stride, rows = 1, 0, None
        if self.kind == L.CAND_EXPLICIT:
            r = self.rows
            tb = r.element_size()
            stride = r.stride(0) * tb
            rows = r.data_ptr()
        elif self.kind == L.CAND_NEIGHBOR:
            tb = self.rows.element_size()
            rows = self.rows.data_ptr()
        ff = None if self.first_from is None else self.first_from.data_ptr()
        return L.Candidates(self.kind, tb, rows, stride, self.seed, self.first, self.count, ff,
                            self.moves, 0)


def groups_array(model, n_req, slo, mu, var, dist=None) -> np.ndarray:
    G = len(model)
    g = np.zeros(G, L.GROUP_DTYPE)
    g["model"], g["n_req"], g["slo_s"], g["mu_out"], g["var_out"] = model, n_req, slo, mu, var
    g["dist_id"] = -1 if dist is None else dist
    return g


def queues_array(device, resident, backlog_mean=None, backlog_var=None) -> np.ndarray:
    Q = len(device)
    q = np.zeros(Q, L.QUEUE_DTYPE)
    q["device"], q["resident_model"] = device, resident
    q["backlog_mean_s"] = 0.0 if backlog_mean is None else backlog_mean
    q["backlog_var_s2"] = 0.0 if backlog_var is None else backlog_var
    return q


def kernel_overrides(no_ws=False, no_ws2=False, no_two_phase=False, no_wide=False, no_tier_warp=False,
                     no_graph=False, no_large=False, ilv_cap=0):
    """Testing: restrict the library's kernel choice process-wide
    (qlm_set_kernel_overrides); call with no arguments to restore the default."""
    kw = dict(no_ws=no_ws, no_ws2=no_ws2, no_two_phase=no_two_phase, no_wide=no_wide,
              no_tier_warp=no_tier_warp, no_graph=no_graph, no_large=no_large)
    flags = sum(L.OVERRIDE[k] for k, v in kw.items() if v)
    L.check(L.lib().qlm_set_kernel_overrides(flags, int(ilv_cap)), "qlm_set_kernel_overrides")


class RwtEstimator:
    """One qlm_ctx: a scheduling problem resident on one sm_100a GPU."""

    def __init__(self, problem, device: int = 0, z_clamp: float = 8.0, alpha: float = 0.01,
                 with_tables: bool | None = None):
        p = problem
        self.device = torch.device("cuda", device)
        self.groups = groups_array(p.model, p.n_req, p.slo, p.mu, p.var, p.dist)
        self.queues = queues_array(p.q_device, p.q_resident, p.q_backlog_mean, p.q_backlog_var)
        c = np.ascontiguousarray
        self._prof_arrays = [c(a, np.float64) for a in
                             (p.theta, p.prefill, p.eps, p.dtok, p.max_out, p.swap)]
        D, M = self._prof_arrays[0].shape
        prof = L.Profile(D, M, *[a.ctypes.data for a in self._prof_arrays])
        tabs = None
        use_tabs = p.len_tables is not None if with_tables is None else with_tables
        if use_tabs:
            self._len = c(p.len_tables, np.uint16)
            tabs = L.LenTables(self._len.shape[1], self._len.shape[0], self._len.ctypes.data)
        else:
            self.groups["dist_id"] = -1
        opt = L.Options(z_clamp, alpha, device, 0)
        h = C.c_void_p()
        L.check(L.lib().qlm_create(self.groups.ctypes.data, len(self.groups),
                                   self.queues.ctypes.data, len(self.queues), C.byref(prof),
                                   C.byref(tabs) if tabs is not None else None, C.byref(opt),
                                   C.byref(h)), "qlm_create")
        self._h = h
        self.G, self.Q, self.D, self.M = len(self.groups), len(self.queues), D, M
        self.T = self.G + self.Q - 1

    def close(self):
        if getattr(self, "_h", None):
            L.lib().qlm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- multi-GPU: the library's own NCCL communicator (include/qlm.h) -----------
    @staticmethod
    def comm_unique_id() -> bytes:
        """A fresh 128-byte NCCL unique id (rank 0; broadcast it to the others)."""
        buf = (C.c_uint8 * L.COMM_ID_BYTES)()
        L.check(L.lib().qlm_comm_unique_id(buf), "qlm_comm_unique_id")
        return bytes(buf)

    def comm_attach(self, uid: bytes, rank: int, world: int):
        """Collective: attach this context to the communicator `uid` as `rank` of
        `world`; argmin records become global and MC counts sums over ranks."""
        if len(uid) != L.COMM_ID_BYTES:
            raise ValueError(f"unique id must be {L.COMM_ID_BYTES} bytes, got {len(uid)}")
        buf = (C.c_uint8 * L.COMM_ID_BYTES).from_buffer_copy(uid)
        torch.cuda.synchronize(self.device)
        L.check(L.lib().qlm_comm_attach(self._h, buf, rank, world), "qlm_comm_attach")
        self._comm = (rank, world)

    def comm_detach(self):
        L.check(L.lib().qlm_comm_detach(self._h), "qlm_comm_detach")
        self._comm = None

    def comm_info(self) -> dict:
        r, w, v = C.c_int32(), C.c_int32(), C.c_int32()
        L.check(L.lib().qlm_comm_info(self._h, C.byref(r), C.byref(w), C.byref(v)), "qlm_comm_info")
        return dict(rank=r.value, world=w.value, nccl_version=v.value)

    @property
    def comm_attached(self) -> bool:
        return getattr(self, "_comm", None) is not None

    # -- helpers --------------------------------------------------------------
    def _stream(self, stream):
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        return C.c_void_p(s.cuda_stream)

    def _empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def random(self, first: int, count: int, seed: int) -> Cand:
        return Cand(L.CAND_RANDOM, first, count, seed)

    def enum(self, first: int, count: int) -> Cand:
        return Cand(L.CAND_ENUM, first, count)

    def explicit(self, rows: torch.Tensor, first: int = 0) -> Cand:
        """rows: device uint8 (T <= 256) or int16 tensor [count, >= T], row stride a multiple of 16 B."""
        return Cand(L.CAND_EXPLICIT, first, rows.shape[0], rows=rows)

    def neighbor(self, base: torch.Tensor, first: int, count: int, seed: int, moves: int) -> Cand:
        """NEIGHBOR candidates (R18): `base` with `moves` Philox-drawn transpositions each.
        base: device uint8 (T <= 256) / int16 tensor of >= T tokens, 16-B aligned, padded
        to a multiple of 16 B (see row_buffer)."""
        return Cand(L.CAND_NEIGHBOR, first, count, seed, rows=base, moves=moves)

    def row_buffer(self, row, token_bytes: int | None = None) -> torch.Tensor:
        """A device row in the layout NEIGHBOR / qlm_local_search expect (padded to 16 B)."""
        tb = token_bytes or (1 if self.T <= 256 else 2)
        n = -(-self.T * tb // 16) * 16 // tb
        buf = torch.zeros(n, dtype=torch.uint8 if tb == 1 else torch.int16, device=self.device)
        r = torch.as_tensor(np.asarray(row, np.int64))
        buf[: self.T] = r.to(buf.dtype).to(self.device)
        return buf

    def request_violations(self, cand: Cand, stream=None):
        """R19: (frac [G, count], s1_req [count]) -- per-group fraction of SLO-violating
        requests and the request-granular S1 of each candidate."""
        frac = self._empty((self.G, cand.count), torch.float32)
        s1r = self._empty(cand.count, torch.float32)
        L.check(L.lib().qlm_request_violations(self._h, C.byref(cand.c()), frac.data_ptr(), s1r.data_ptr(),
                                               self._stream(stream)), "qlm_request_violations")
        return frac, s1r

    def set_tiers(self, tiers: dict | None):
        """Two-tier model swapping (R20): tiers = dict(mem=int32 [M], cap=int32 [D],
        load=f64 [D, M]) or None to clear."""
        if tiers is None:
            L.check(L.lib().qlm_set_tiers(self._h, None), "qlm_set_tiers")
            return
        arrs = (np.ascontiguousarray(tiers["mem"], np.int32), np.ascontiguousarray(tiers["cap"], np.int32),
                np.ascontiguousarray(tiers["load"], np.float64))
        t = L.Tiers(*[a.ctypes.data for a in arrs])
        L.check(L.lib().qlm_set_tiers(self._h, C.byref(t)), "qlm_set_tiers")

    def tiered_score_estimate(self, cand: Cand, out=None, scores=True, rec: torch.Tensor | None = None,
                              stream=None):
        """qlm_tiered_score_estimate: score_estimate under two-tier swapping (R20)."""
        out = {} if out is None else out
        if scores and out.get("s1") is None:
            out["s1"] = self._empty(cand.count, torch.float32)
            out["s2"] = self._empty(cand.count, torch.float32)
        ptr = {k: (out[k].data_ptr() if out.get(k) is not None else None)
               for k in ("wt", "sd", "v", "s1", "s2", "n_over")}
        L.check(L.lib().qlm_tiered_score_estimate(self._h, C.byref(cand.c()), ptr["wt"], ptr["sd"], ptr["v"],
                                                  ptr["s1"], ptr["s2"], ptr["n_over"],
                                                  None if rec is None else rec.data_ptr(),
                                                  self._stream(stream)), "qlm_tiered_score_estimate")
        return out

    def tiered_mc_count(self, cand: Cand, trials: int, counts: torch.Tensor | None = None, stream=None):
        """qlm_tiered_mc_count: MC counts with the warm/cold swap costs (R13 + R20)."""
        counts = self._empty((cand.count, self.G), torch.int32) if counts is None else counts
        L.check(L.lib().qlm_tiered_mc_count(self._h, C.byref(cand.c()), trials, counts.data_ptr(),
                                            self._stream(stream)), "qlm_tiered_mc_count")
        return counts

    def adopt_best(self, cand: Cand, rec: torch.Tensor, incumbent: torch.Tensor, stream=None):
        """Device-side local-search step: cand.rows <- winner row if rec beats incumbent."""
        L.check(L.lib().qlm_adopt_best(self._h, C.byref(cand.c()), rec.data_ptr(), incumbent.data_ptr(),
                                       self._stream(stream)), "qlm_adopt_best")

    def local_search(self, row, moves: int = 2, per_iter: int = 1 << 16, iters: int = 16,
                     seed: int = 1, stream=None):
        """Iterated best-of-N over NEIGHBOR candidates (R18), asynchronous on the stream.
        row: start ordering (host sequence or a row_buffer tensor, updated in place).
        Returns (row buffer, incumbent record int64[2] = (key bits, adopted index))."""
        buf = row if isinstance(row, torch.Tensor) else self.row_buffer(row)
        inc = self._empty(2, torch.int64)
        L.check(L.lib().qlm_local_search(self._h, C.c_void_p(buf.data_ptr()), buf.element_size(), moves,
                                         per_iter, iters, seed, C.c_void_p(inc.data_ptr()),
                                         self._stream(stream)), "qlm_local_search")
        return buf, inc

    def from_record(self, rec: torch.Tensor, kind: int = L.CAND_RANDOM, seed: int = 0,
                    base: torch.Tensor | None = None, moves: int = 0) -> Cand:
        """The single candidate named by a device record (no host sync); NEIGHBOR
        records also need the base row and the number of moves."""
        return Cand(kind, 0, 1, seed, rows=base, first_from=rec, moves=moves)

    # -- hot path -------------------------------------------------------------
    def update_groups(self, groups: np.ndarray | torch.Tensor, stream=None):
        ptr = groups.data_ptr() if isinstance(groups, torch.Tensor) else groups.ctypes.data
        L.check(L.lib().qlm_update_groups(self._h, C.c_void_p(ptr), self._stream(stream)),
                "qlm_update_groups")

    def score_orderings(self, cand: Cand, with_n_over: bool = True, stream=None):
        s1 = self._empty(cand.count, torch.float32)
        s2 = self._empty(cand.count, torch.float32)
        no = self._empty(cand.count, torch.int32) if with_n_over else None
        L.check(L.lib().qlm_score_orderings(self._h, C.byref(cand.c()), s1.data_ptr(), s2.data_ptr(),
                                            None if no is None else no.data_ptr(),
                                            self._stream(stream)), "qlm_score_orderings")
        return s1, s2, no

    def best_ordering_async(self, cand: Cand, rec: torch.Tensor | None = None, stream=None):
        """Device record int64[2] = (key as int64 bits, global index)."""
        rec = self._empty(2, torch.int64) if rec is None else rec
        L.check(L.lib().qlm_best_ordering_async(self._h, C.byref(cand.c()), rec.data_ptr(),
                                                self._stream(stream)), "qlm_best_ordering_async")
        return rec

    def reduce_records(self, recs: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        out = self._empty(2, torch.int64) if out is None else out
        n = recs.numel() // 2
        L.check(L.lib().qlm_reduce_records(self._h, recs.data_ptr(), n, out.data_ptr(),
                                           self._stream(stream)), "qlm_reduce_records")
        return out

    def best_ordering(self, cand: Cand, stream=None) -> dict:
        b = L.Best()
        qo = np.zeros(self.G, np.int32)
        po = np.zeros(self.G, np.int32)
        L.check(L.lib().qlm_best_ordering(self._h, C.byref(cand.c()), C.byref(b), qo.ctypes.data,
                                          po.ctypes.data, self._stream(stream)), "qlm_best_ordering")
        return dict(index=b.index, s1=b.s1, s2=b.s2, n_over=b.n_over, queue_of_group=qo,
                    pos_of_group=po)

    def winner(self, one: Cand, host: dict, stream=None):
        """qlm_winner: the record's candidate scored and decoded on the stream and
        written into host tensors (pinned: by the device directly, one kernel;
        pageable: one copy per field): host["best"] a uint8[24]
        qlm_best image, host["qo"] / host["po"] int32[G].  Asynchronous."""
        L.check(L.lib().qlm_winner(self._h, C.byref(one.c()), host["best"].data_ptr(),
                                   host["qo"].data_ptr() if "qo" in host else None,
                                   host["po"].data_ptr() if "po" in host else None,
                                   self._stream(stream)), "qlm_winner")

    @staticmethod
    def best_of(best_bytes: torch.Tensor) -> dict:
        """Decode a host qlm_best image (qlm_winner) into a dict."""
        b = L.Best.from_buffer_copy(bytes(best_bytes.numpy().tobytes()))
        return dict(index=b.index, s1=b.s1, s2=b.s2, n_over=b.n_over)

    def rwt_estimate(self, cand: Cand, want=("wt", "sd", "v"), out=None, stream=None):
        """Per-(group, candidate) expected wait, its std and violation probability.

        Group-major: out[k] has shape [G, count]; out["v"][g, k] is group g in
        candidate first + k.
        """
        if out is None:
            out = {k: self._empty((self.G, cand.count), torch.float32) for k in want}
        ptr = {k: (out[k].data_ptr() if k in out else None) for k in ("wt", "sd", "v")}
        L.check(L.lib().qlm_rwt_estimate(self._h, C.byref(cand.c()), ptr["wt"], ptr["sd"], ptr["v"],
                                         self._stream(stream)), "qlm_rwt_estimate")
        return out

    def score_estimate(self, cand: Cand, out=None, scores=True, rec: torch.Tensor | None = None,
                       stream=None):
        """The fused single pass: bulk estimates + per-candidate scores + argmin record."""
        out = {} if out is None else out
        ptr = {k: (out[k].data_ptr() if out.get(k) is not None else None)
               for k in ("wt", "sd", "v", "s1", "s2", "n_over")}
        if scores and ptr["s1"] is None:
            out["s1"] = self._empty(cand.count, torch.float32)
            out["s2"] = self._empty(cand.count, torch.float32)
            ptr["s1"], ptr["s2"] = out["s1"].data_ptr(), out["s2"].data_ptr()
        L.check(L.lib().qlm_score_estimate(self._h, C.byref(cand.c()), ptr["wt"], ptr["sd"], ptr["v"],
                                           ptr["s1"], ptr["s2"], ptr["n_over"],
                                           None if rec is None else rec.data_ptr(),
                                           self._stream(stream)), "qlm_score_estimate")
        return out

    def mc_estimate(self, cand: Cand, mc_seed: int, trials: int, trial_first: int = 0,
                    counts: torch.Tensor | None = None, stream=None):
        """counts[k, g] = #{trials t: sampled W_g > slo_g} (uint32 stored as int32)."""
        counts = self._empty((cand.count, self.G), torch.int32) if counts is None else counts
        L.check(L.lib().qlm_mc_estimate(self._h, C.byref(cand.c()), mc_seed, trial_first, trials,
                                        counts.data_ptr(), self._stream(stream)), "qlm_mc_estimate")
        return counts

    def mc_sample(self, mc_seed: int, trials: int, trial_first: int = 0, stream=None):
        """Candidate-independent MC half (may overlap scan calls on another stream)."""
        L.check(L.lib().qlm_mc_sample(self._h, mc_seed, trial_first, trials, self._stream(stream)),
                "qlm_mc_sample")

    def mc_count(self, cand: Cand, trials: int, counts: torch.Tensor | None = None, stream=None):
        counts = self._empty((cand.count, self.G), torch.int32) if counts is None else counts
        L.check(L.lib().qlm_mc_count(self._h, C.byref(cand.c()), trials, counts.data_ptr(),
                                     self._stream(stream)), "qlm_mc_count")
        return counts

    def decode(self, cand: Cand, stream=None, out=None):
        """qlm_decode: queue and position of every group (int32 [count][G] each);
        `out` = (qo, po) preallocated on the device (e.g. for another stream)."""
        if out is not None:
            qo, po = out
            assert qo.shape == (cand.count, self.G) and po.shape == qo.shape and qo.dtype == po.dtype == torch.int32
        else:
            qo = self._empty((cand.count, self.G), torch.int32)
            po = self._empty((cand.count, self.G), torch.int32)
        L.check(L.lib().qlm_decode(self._h, C.byref(cand.c()), qo.data_ptr(), po.data_ptr(),
                                   self._stream(stream)), "qlm_decode")
        return qo, po

    def rows(self, cand: Cand, stream=None) -> torch.Tensor:
        r = self._empty((cand.count, self.T), torch.int16)
        L.check(L.lib().qlm_rows(self._h, C.byref(cand.c()), r.data_ptr(), self._stream(stream)),
                "qlm_rows")
        return r

    def check_rows(self, cand: Cand, stream=None) -> int:
        n = C.c_int64()
        L.check(L.lib().qlm_check_rows(self._h, C.byref(cand.c()), C.byref(n), self._stream(stream)),
                "qlm_check_rows")
        return n.value


def form_groups(req: dict, M: int, k_per_model, limit: int = 256, max_iter: int = 50,
                device: int = 0, stream=None) -> dict:
    """Alg. 1 on the GPU under reading R21 (qlm_form_groups).

    req: dict(model int32 [n], slo f64 [n], out int32 [n], feat int32 [n, dims])
    in arrival order (host arrays or device tensors).  Returns dict(n_groups,
    iters, label / group_of: device int32 [n], groups: numpy qlm_group records
    ready for RwtEstimator / qlm_create)."""
    dev = torch.device("cuda", device)
    t = {k: torch.as_tensor(np.ascontiguousarray(req[k]) if not isinstance(req[k], torch.Tensor) else req[k])
         .to(dev).contiguous() for k in ("model", "slo", "out", "feat")}
    t["model"], t["out"], t["feat"] = (t["model"].to(torch.int32), t["out"].to(torch.int32),
                                       t["feat"].to(torch.int32))
    t["slo"] = t["slo"].to(torch.float64)
    n = t["model"].numel()
    dims = t["feat"].shape[1] if t["feat"].dim() == 2 else 1
    r = L.Requests(n, dims, t["model"].data_ptr(), t["slo"].data_ptr(), t["out"].data_ptr(), t["feat"].data_ptr())
    k = np.ascontiguousarray(k_per_model, np.int32)
    label = torch.empty(n, dtype=torch.int32, device=dev)
    gof = torch.empty(n, dtype=torch.int32, device=dev)
    # groups <= clusters + 2n / ceil(limit / 2): a split leaf keeps >= ceil(limit / 2) members
    cap = int(min(n, int(k.sum()) + (2 * n) // max(1, (limit + 1) // 2) + 1))
    groups = torch.empty(cap * L.GROUP_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    G, it = C.c_int32(), C.c_int32()
    s = torch.cuda.current_stream(dev) if stream is None else stream
    L.check(L.lib().qlm_form_groups(C.byref(r), M, k.ctypes.data, limit, max_iter, label.data_ptr(),
                                    gof.data_ptr(), groups.data_ptr(), cap, C.byref(G), C.byref(it), device,
                                    C.c_void_p(s.cuda_stream)), "qlm_form_groups")
    recs = groups[: G.value * L.GROUP_DTYPE.itemsize].cpu().numpy().view(L.GROUP_DTYPE)
    return dict(n_groups=G.value, iters=it.value, label=label, group_of=gof, groups=recs)


def kernel_launches() -> int:
    return int(L.lib().qlm_kernel_launches())


def decode_key(key: int) -> tuple[float, float]:
    """(fp32 S1, fp32 S2) from a record key (inverse of the kernel's packing)."""
    key &= (1 << 64) - 1
    b1 = np.uint32(key >> 32)
    b2 = np.uint32(key & 0xFFFFFFFF)
    b2 = np.uint32(b2 ^ 0x80000000) if b2 & 0x80000000 else np.uint32(~b2 & 0xFFFFFFFF)
    return float(b1.view(np.float32)), float(b2.view(np.float32))
