"""C5 / C5h bulk (wt, sd, v for every group) + argmin over N RANDOM candidates:
CUDA-event time of one call (after warm-up).   python tools/c5_bulk.py [N] [cfg] [tiered]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config, make_tiers  # noqa: E402

__graft_entry__.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
cfg = sys.argv[2] if len(sys.argv) > 2 else "C5"
tiered = len(sys.argv) > 3 and sys.argv[3] == "tiered"
p = make_config(cfg)
e = RwtEstimator(p)
if tiered:
    e.set_tiers(make_tiers(dev_rows=(0, 1) if cfg == "C5h" else (0,)))
cand = e.random(0, N, seed=1)
out = {k: torch.empty((p.G, N), device="cuda") for k in ("wt", "sd", "v")}
rec = torch.empty(2, dtype=torch.int64, device="cuda")
f = (lambda: e.tiered_score_estimate(cand, out=out, scores=False, rec=rec)) if tiered else \
    (lambda: e.score_estimate(cand, out=out, scores=False, rec=rec))
for _ in range(2):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
f()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b)
print("ms", ms, "GBps", 12 * p.G * N / ms / 1e6, "rec", rec.tolist())
