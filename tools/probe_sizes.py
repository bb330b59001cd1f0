"""Size envelope of the C ABI: which entry points run for G up to T = 32768.

    python tools/probe_sizes.py
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_problem
import oracle as O
for G in [1500, 4000, 8000, 20000, 32700]:
    p = make_problem(G, 8, name=f"G{G}")
    try:
        e = RwtEstimator(p)
    except Exception as ex:
        print(G, "create", type(ex).__name__, str(ex)[:150]); continue
    for name, fn in [("score_random", lambda: e.score_orderings(e.random(0, 300, seed=1))),
                     ("best_random", lambda: e.best_ordering(e.random(0, 300, seed=1))),
                     ("bulk_random", lambda: e.rwt_estimate(e.random(0, 64, seed=1))),
                     ("rows", lambda: e.rows(e.random(0, 4, seed=1))),
                     ("reqviol", lambda: e.request_violations(e.random(0, 2, seed=1)))]:
        try:
            r = fn(); torch.cuda.synchronize()
            ok = ""
            if name == "score_random":
                ref = O.Oracle(p).score_range(O.RANDOM, 0, 20, seed=1)
                ok = f"maxdiff {np.max(np.abs(r[0][:20].cpu().numpy() - ref['s1'])):.2e}"
            print(G, name, "OK", ok, flush=True)
        except Exception as ex:
            print(G, name, "FAIL", type(ex).__name__, str(ex)[:200], flush=True)
