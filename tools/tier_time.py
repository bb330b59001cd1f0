"""Time the tiered C3 bulk pass (qlm_tiered_score_estimate, 1e6 RANDOM
candidates) with CUDA events; QLM_LIB_PATH selects a library build."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config, make_tiers  # noqa: E402

p = make_config("C3")
e = RwtEstimator(p)
e.set_tiers(make_tiers())
N = 1_000_000
cand = e.random(0, N, seed=1)
out = {k: torch.empty((p.G, N), device="cuda") for k in ("wt", "sd", "v")}
rec = torch.empty(2, dtype=torch.int64, device="cuda")
for _ in range(5):
    e.tiered_score_estimate(cand, out=out, rec=rec)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    e.tiered_score_estimate(cand, out=out, rec=rec)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(json.dumps(dict(lib=os.path.basename(os.environ.get("QLM_LIB_PATH", "libqlm.so")), median_ms=round(ts[15], 4),
                      rec=rec.tolist())))
