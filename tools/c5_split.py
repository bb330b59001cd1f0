"""C5 score-only (two-phase) under ncu: per-kernel time / instructions / DRAM.

    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
smsp__issue_active.avg.pct_of_peak_sustained_active --csv python tools/c5_split.py [N]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config  # noqa: E402

__graft_entry__.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = sys.argv[2] if len(sys.argv) > 2 else "C5"
e = RwtEstimator(make_config(cfg))
rec = torch.empty(2, dtype=torch.int64, device="cuda")
cand = e.random(0, N, seed=1)
for _ in range(2):
    e.best_ordering_async(cand, rec)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
e.best_ordering_async(cand, rec)
b.record()
torch.cuda.synchronize()
print("ms", a.elapsed_time(b), "rate", N / a.elapsed_time(b) * 1e3, "rec", rec.tolist())
