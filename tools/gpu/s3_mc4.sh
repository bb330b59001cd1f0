QLM_LIB_PATH=build/variants/libqlm_mcb4.so timeout 900 python -m pytest tests -q -m gpu -x -k "mc or MC or smoke or bench_step" 2>&1 | tail -1
for v in mcall mcb2 mcb3 mcb4 mcall mcb2 mcb3 mcb4; do echo "$v $(QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/step_parts.py 2>&1 | grep -E '^full' )"; QLM_LIB_PATH=build/variants/libqlm_$v.so python - <<'PY'
import sys, torch; sys.path.insert(0, ".")
import __graft_entry__; __graft_entry__.build()
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config
for cfg in ("C3", "C4"):
    e = RwtEstimator(make_config(cfg))
    for _ in range(3): e.mc_sample(2, 1221)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): e.mc_sample(2, 1221)
    b.record(); torch.cuda.synchronize()
    print("  ", cfg, "mc_sample us", round(a.elapsed_time(b) / 20 * 1000, 2))
PY
done
