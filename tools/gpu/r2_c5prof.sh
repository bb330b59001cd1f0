cat > /tmp/c5.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, __graft_entry__
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config
__graft_entry__.build()
p = make_config("C5"); e = RwtEstimator(p)
n = 100000
cand = e.random(0, n, seed=1)
out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
rec = torch.empty(2, dtype=torch.int64, device="cuda")
for _ in range(3):
    e.score_estimate(cand, out=out, scores=False, rec=rec)
    e.best_ordering_async(e.random(0, 200000, seed=1), rec)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:"fy_rows_kernel|wide_kernel|scan_kernel" -s 6 -c 4 -o gpurun_out/c5_full python /tmp/c5.py > gpurun_out/c5_ncu.txt 2>&1
tail -3 gpurun_out/c5_ncu.txt
