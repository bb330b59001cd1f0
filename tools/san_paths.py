"""Small launches of the bulk kernels for compute-sanitizer (memcheck /
racecheck / synccheck): ws2_kernel (plain and tiered), wide_kernel and
tier_warp_kernel on the two-phase rows, and the score-only large-T path
(fy_rows_kernel + large_kernel)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config, make_tiers  # noqa: E402


def run(cfg, n, tiered):
    p = make_config(cfg)
    e = RwtEstimator(p)
    if tiered:
        e.set_tiers(make_tiers(dev_rows=tuple(range(p.theta.shape[0]))))
    cand = e.random(0, n, seed=1)
    out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
    rec = torch.empty(2, dtype=torch.int64, device="cuda")
    (e.tiered_score_estimate if tiered else e.score_estimate)(cand, out=out, rec=rec)
    torch.cuda.synchronize()
    print(cfg, n, "tiered" if tiered else "plain", rec.tolist())


def score_only(cfg, n):
    p = make_config(cfg)
    e = RwtEstimator(p)
    s1, s2, nov = e.score_orderings(e.random(0, n, seed=1))
    rec = e.best_ordering_async(e.random(0, n, seed=1))
    torch.cuda.synchronize()
    print(cfg, n, "score-only", rec.tolist())


if __name__ == "__main__":
    run("C3", 8192, False)
    run("C3", 8192, True)
    run("C5", 4096, False)
    run("C5h", 4096, True)
    score_only("C5", 4096 + 77)
