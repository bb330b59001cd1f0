"""Time the fused bulk pass (qlm_score_estimate, C3, 1e6 RANDOM candidates)
with CUDA events; QLM_LIB_PATH selects an experimental library build.

    QLM_LIB_PATH=... python tools/ws_time.py [cfg] [count] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_00047_b200 import RwtEstimator, decode_key  # noqa: E402
from workloads.synth import make_config  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    keys = sys.argv[4].split(",") if len(sys.argv) > 4 else ["wt", "sd", "v"]
    p = make_config(cfg)
    e = RwtEstimator(p)
    cand = e.random(0, N, seed=1)
    out = {k: torch.empty((p.G, N), dtype=torch.float32, device="cuda") for k in keys}
    rec = torch.empty(2, dtype=torch.int64, device="cuda")
    for _ in range(5):
        e.score_estimate(cand, out=out, rec=rec)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e.score_estimate(cand, out=out, rec=rec)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    s1, s2 = decode_key(int(rec[0]))
    print(json.dumps(dict(lib=os.path.basename(os.environ.get("QLM_LIB_PATH", "libqlm.so")), cfg=cfg, N=N,
                          median_ms=round(ms, 4), min_ms=round(ts[0], 4),
                          GBps=4 * len(keys) * p.G * N / ms / 1e6, outs=",".join(keys), best=int(rec[1]), s1=s1, s2=s2)))


if __name__ == "__main__":
    main()
