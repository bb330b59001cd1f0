"""Score-only (argmin) throughput per config: python tools/score_rate.py C5 1000000"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config
__graft_entry__.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
est = RwtEstimator(make_config(cfg))
cand = est.random(0, N, seed=1)
rec = torch.empty(2, dtype=torch.int64, device="cuda")
for _ in range(2):
    est.best_ordering_async(cand, rec)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
reps = 5
for _ in range(reps):
    est.best_ordering_async(cand, rec)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"{cfg} score+argmin: {ms:.3f} ms for {N} candidates = {N / ms / 1e6:.3f} G candidates/s")
