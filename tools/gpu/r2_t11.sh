cat > /tmp/c5b.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch, __graft_entry__, kernel_suite
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config
__graft_entry__.build()
p = make_config("C5"); e = RwtEstimator(p)
n = 100000
cand = e.random(0, n, seed=1)
out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
rec = torch.empty(2, dtype=torch.int64, device="cuda")
ms = kernel_suite._time(lambda: e.score_estimate(cand, out=out, scores=False, rec=rec), 20)
print(os.environ.get("QLM_WIDE_RS"), "C5 bulk ms", round(ms, 4), "GB/s", round(n * 12 * p.G / ms / 1e6, 1))
PY
for rs in 0 1 2; do QLM_WIDE_RS=$rs python /tmp/c5b.py; done
timeout 900 python -m pytest tests -m gpu -q -x -k "wide or large_G or c5" 2>&1 | tail -2
