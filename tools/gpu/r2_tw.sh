set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -m gpu -k "tier" > gpurun_out/tw_tests.log 2>&1; tail -3 gpurun_out/tw_tests.log
python - <<'PY'
import json, subprocess, os
for lib in ("build/variants/libqlm_base.so", ""):
    env = dict(os.environ)
    if lib: env["QLM_LIB_PATH"] = lib
    code = r'''
import torch, json
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config, make_tiers
p = make_config("C5h"); e = RwtEstimator(p); e.set_tiers(make_tiers(dev_rows=tuple(range(p.theta.shape[0]))))
n = 100000; cand = e.random(0, n, seed=1)
out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
rec = torch.empty(2, dtype=torch.int64, device="cuda")
for _ in range(3): e.tiered_score_estimate(cand, out=out, scores=False, rec=rec)
torch.cuda.synchronize(); ts = []
for _ in range(15):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); e.tiered_score_estimate(cand, out=out, scores=False, rec=rec); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
ts.sort(); print(json.dumps({"ms": ts[len(ts)//2], "rec": rec.tolist()}))
'''
    print(lib or "new", subprocess.run(["python", "-c", code], env=env, capture_output=True, text=True).stdout.strip())
PY
