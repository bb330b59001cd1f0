"""Local search (DESIGN R18) on a config: quality and speed.

    python tools/search_bench.py C3 [per_iter] [iters]
Starts from the FCFS and the EDF comparator rows, runs
qlm_local_search (2 transpositions per candidate), and prints the objective
(S1 = expected violating fraction, S2 = sum of slacks, and the request-level
S1_req of R19) of the comparators,
of the best of as many RANDOM candidates, and of the search result, plus
candidates/s of the search timed with CUDA events.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator, decode_key  # noqa: E402
from workloads.synth import edf_row, fcfs_row, make_config  # noqa: E402


def main():
    __graft_entry__.build()
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    per_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    p = make_config(cfg)
    e = RwtEstimator(p)

    def score(row):
        b = e.row_buffer(row)
        ex = e.explicit(b.view(1, -1))
        s1, s2, _ = e.score_orderings(ex)
        _, s1r = e.request_violations(ex)          # request-granular S1 (R19)
        return float(s1[0]), float(s2[0]), float(s1r[0])

    out = {"config": cfg, "per_iter": per_iter, "iters": iters}
    for name, row in (("fcfs", fcfs_row(p)), ("edf", edf_row(p))):
        out[name] = score(row)
    rec = e.best_ordering_async(e.random(0, per_iter * iters, seed=1))
    out["best_random"] = decode_key(int(rec.cpu().numpy()[0]))
    for name, row in (("search_from_fcfs", fcfs_row(p)), ("search_from_edf", edf_row(p))):
        e.local_search(row, moves=2, per_iter=per_iter, iters=2, seed=7)       # warm-up
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        buf, inc = e.local_search(row, moves=2, per_iter=per_iter, iters=iters, seed=7)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        res = buf.cpu().numpy()[: p.T].astype(np.int64)
        out[name] = score(res)
        out[name + "_ms"] = round(ms, 3)
        out[name + "_cand_per_s"] = per_iter * iters / ms * 1e3
    # request-level evaluation rate (R19) over 65536 RANDOM candidates
    cand = e.random(0, 65536, seed=3)
    e.request_violations(cand)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    e.request_violations(cand)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    out["request_violations_65536_ms"] = round(ms, 3)
    out["request_evals_per_s"] = 65536 * float(p.n_req.sum()) / ms * 1e3
    print(out)


if __name__ == "__main__":
    main()
