"""Large-G probe: time row generation (qlm_rows) and EXPLICIT scoring separately.

    python tools/c5_probe.py C5 100000
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


__graft_entry__.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
est = RwtEstimator(make_config(cfg))
cand = est.random(0, N, seed=1)
T = est.T
ms_rows = timed(lambda: est.rows(cand))
rows = est.rows(cand)
stride = (T * 2 + 15) // 16 * 8
pad = torch.zeros((N, stride), dtype=torch.int16, device="cuda")
pad[:, :T] = rows
ex = est.explicit(pad)
rec = torch.empty(2, dtype=torch.int64, device="cuda")
ms_ex = timed(lambda: est.best_ordering_async(ex, rec))
ms_rnd = timed(lambda: est.best_ordering_async(cand, rec))
print(f"{cfg} N={N} T={T}: rows {ms_rows:.3f} ms ({N / ms_rows / 1e6:.3f} G/s) | "
      f"explicit score {ms_ex:.3f} ms ({N / ms_ex / 1e6:.3f} G/s) | random score {ms_rnd:.3f} ms "
      f"({N / ms_rnd / 1e6:.3f} G/s)")
