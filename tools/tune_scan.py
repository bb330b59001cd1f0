"""Time the fused scan kernel (qlm_score_estimate) on C3 under launch-config overrides.

    python tools/tune_scan.py            # sweep QLM_BLK x QLM_REP_SHIFT
Prints one line per config: ms per launch (CUDA events) and GB/s of outputs.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config  # noqa: E402


def time_it(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    __graft_entry__.build()
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    p = make_config(cfg)
    est = RwtEstimator(p)
    cand = est.random(0, N, seed=1)
    out = {k: torch.empty((p.G, N), dtype=torch.float32, device="cuda") for k in ("wt", "sd", "v")}
    rec = torch.empty(2, dtype=torch.int64, device="cuda")
    byts = 12 * p.G * N
    quick = os.environ.get("TUNE_QUICK")
    configs = [dict()] if quick else [dict()] + [dict(QLM_WS_PAIRS=w_, QLM_REP_SHIFT=r) for w_ in (7, 6) for r in (3, 0)] + \
        [dict(QLM_NO_WS=1, QLM_BLK=b, QLM_REP_SHIFT=r) for b in (128,) for r in (0,)]
    keys = ("QLM_WS_PAIRS", "QLM_REP_SHIFT", "QLM_NO_WS", "QLM_BLK")
    for cfgd in configs:
        blk, rs = cfgd, ""
        for k, v in ((k, cfgd.get(k)) for k in keys):
            if quick:
                break                       # quick mode: keep the caller's environment
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)
        try:
            ms = time_it(lambda: est.score_estimate(cand, out=out, scores=False, rec=rec))
            ms_s = time_it(lambda: est.best_ordering_async(cand, rec))
        except Exception as e:  # config does not fit
            print(f"{blk}: {e}")
            continue
        print(f"{cfg} {blk}: fused {ms:.4f} ms = {byts / ms / 1e6:.1f} GB/s "
              f"({N / ms / 1e6:.3f} Gcand/s) | score-only {ms_s:.4f} ms ({N / ms_s / 1e6:.3f} Gcand/s)",
              flush=True)


if __name__ == "__main__":
    main()
