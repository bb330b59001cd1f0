"""Two-tier swapping (R20) throughput and effect per config.

    python tools/tier_bench.py [C3] [count]
Times qlm_tiered_score_estimate (bulk wt/sd/v + scores + argmin) and the
untiered qlm_score_estimate on the same RANDOM candidates with CUDA events,
reports candidates/s and achieved HBM GB/s of the bulk outputs (12 B per
(candidate, group)), and the best S1 with and without the warm/cold costs.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator, decode_key  # noqa: E402
from workloads.synth import make_config, make_tiers  # noqa: E402


def main():
    __graft_entry__.build()
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    p = make_config(cfg)
    e = RwtEstimator(p)
    devs = (0, 1) if cfg == "C5h" else (0,)
    models = (0, 2) if cfg == "C2" else (0, 1, 2, 3)
    e.set_tiers(make_tiers(models, devs))
    cand = e.random(0, N, seed=1)
    out = {k: torch.empty((p.G, N), dtype=torch.float32, device="cuda") for k in ("wt", "sd", "v")}
    rec = torch.empty(2, dtype=torch.int64, device="cuda")
    res = {"config": cfg, "candidates": N}
    for name, fn in (("tiered", e.tiered_score_estimate), ("untiered", e.score_estimate)):
        for _ in range(3):
            fn(cand, out=out, rec=rec)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record()
        for _ in range(reps):
            fn(cand, out=out, rec=rec)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        s1, s2 = decode_key(int(rec[0]))
        res[name] = dict(ms=round(ms, 4), candidates_per_s=N / ms * 1e3,
                         bulk_GBps=12 * p.G * N / ms / 1e6, best_index=int(rec[1]), best_s1=s1, best_s2=s2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
