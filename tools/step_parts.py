"""Time the C3 bench step with parts left out (CUDA events, 300 steps), to see
where the time outside the fused pass goes.   python tools/step_parts.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from paper_2407_00047_b200 import RwtEstimator  # noqa: E402
from workloads.synth import make_config  # noqa: E402

__graft_entry__.build()
p = make_config("C3")
e = RwtEstimator(p)
N = 1_000_000
cand = e.random(0, N, seed=1)
rec = torch.empty(2, dtype=torch.int64, device="cuda")
bulk = {k: torch.empty((p.G, N), device="cuda") for k in ("wt", "sd", "v")}
counts = torch.empty((1, p.G), dtype=torch.int32, device="cuda")
side = torch.cuda.Stream()
st = torch.cuda.current_stream()
ev_f, ev_s = torch.cuda.Event(), torch.cuda.Event()


def step(scan=True, sample=True, decode=True, count=True):
    ev_f.record(st)
    if scan:
        e.score_estimate(cand, out=bulk, scores=False, rec=rec)
    if sample:
        side.wait_event(ev_f)
        e.mc_sample(7, 1221, stream=side)
        ev_s.record(side)
    win = e.from_record(rec, seed=1)
    if decode:
        e.decode(win)
    if count:
        if sample:
            st.wait_event(ev_s)
        e.mc_count(win, 1221, counts=counts)


def timed(**kw):
    for _ in range(20):
        step(**kw)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(300):
        step(**kw)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 300 * 1000


e.mc_sample(7, 1221)
torch.cuda.synchronize()
for name, kw in [("full", {}), ("no decode", dict(decode=False)), ("no count", dict(count=False)),
                 ("no sample", dict(sample=False)), ("no decode/count", dict(decode=False, count=False)),
                 ("scan only", dict(sample=False, decode=False, count=False)),
                 ("decode+count only", dict(scan=False, sample=False)),
                 ("sample+decode+count", dict(scan=False))]:
    print(f"{name:22s} {timed(**kw):8.1f} us")
