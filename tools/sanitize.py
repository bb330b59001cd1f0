"""Small invocations of every kernel family for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import balanced_row, make_config, make_requests, make_tiers  # noqa: E402


def main():
    __graft_entry__.build()
    for cfg in ("C2", "C3", "C4", "C5"):
        p = make_config(cfg)
        e = RwtEstimator(p)
        n = 4100 if cfg != "C5" else 4104
        cand = e.random(3, n, seed=1)
        bufs = {k: torch.empty((p.G, n), dtype=torch.float32, device="cuda") for k in ("wt", "sd", "v")}
        e.score_estimate(cand, out=bufs, rec=torch.empty(2, dtype=torch.int64, device="cuda"))
        e.score_orderings(e.random(0, 5000, seed=2))
        rec = e.best_ordering_async(cand)
        e.decode(e.from_record(rec, seed=1))
        base = e.row_buffer(balanced_row(p.G, p.Q).astype(np.int64))
        nb = e.neighbor(base, 0, 4200, seed=4, moves=3)
        e.score_orderings(nb)
        e.rows(e.neighbor(base, 0, 40, seed=4, moves=3))
        e.local_search(balanced_row(p.G, p.Q).astype(np.int64), moves=2, per_iter=4096, iters=2, seed=1)
        e.request_violations(e.random(0, 40, seed=5))
        if p.len_tables is not None:
            e.mc_estimate(e.from_record(rec, seed=1), mc_seed=2, trials=100)
        # two-tier swapping (R20): warp-specialised TIER path, thread kernel, lane-per-queue kernel
        e.set_tiers(make_tiers((0, 1, 2, 3)[: p.M], tuple(range(p.D))))
        e.tiered_score_estimate(cand, out=bufs, rec=torch.empty(2, dtype=torch.int64, device="cuda"))
        e.tiered_score_estimate(e.random(0, 300, seed=2))
        e.tiered_score_estimate(e.from_record(rec, seed=1))
        if p.len_tables is not None:
            e.mc_sample(mc_seed=2, trials=64)
            e.tiered_mc_count(e.from_record(rec, seed=1), 64)
        torch.cuda.synchronize()
        print(cfg, "ok", flush=True)
    # request-group formation (R21)
    from paper_2407_00047_b200 import form_groups
    form_groups(make_requests(20000, seed=1), 4, [5, 3, 1, 8], limit=64, max_iter=20)
    form_groups(make_requests(3000, seed=2), 4, [2, 2, 2, 2], limit=1, max_iter=5)
    torch.cuda.synchronize()
    print("groups ok", flush=True)


if __name__ == "__main__":
    main()
