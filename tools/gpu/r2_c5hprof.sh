cat > /tmp/c5h.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, __graft_entry__
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config, make_tiers
__graft_entry__.build()
p = make_config("C5h"); e = RwtEstimator(p); e.set_tiers(make_tiers(dev_rows=(0, 1)))
n = 100000
cand = e.random(0, n, seed=1)
out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
rec = torch.empty(2, dtype=torch.int64, device="cuda")
for _ in range(3):
    e.tiered_score_estimate(cand, out=out, scores=False, rec=rec)
    e.score_estimate(cand, out=out, scores=False, rec=rec)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:"tier_warp_kernel|wide_kernel" -s 2 -c 2 -o gpurun_out/c5h_full python /tmp/c5h.py > gpurun_out/c5h_ncu.txt 2>&1
tail -2 gpurun_out/c5h_ncu.txt
