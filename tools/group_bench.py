"""Request-group formation (Alg. 1, R21): GPU time vs the oracle.

    python tools/group_bench.py [n_requests] [k_per_model] [max_iter]
Times qlm_form_groups (validation, farthest-point init, Lloyd, splitHalf,
group records) with CUDA events on the calling stream (the call ends with a
stream sync), checks bit-exact parity with the oracle, and reports requests/s
and the Lloyd step's achieved bandwidth (16 B read per request per iteration:
model + 3 features, + 4 B label read/write).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
import oracle as O  # noqa: E402
from paper_2407_00047_b200 import form_groups  # noqa: E402
from workloads.synth import GROUP_LIMIT, make_requests  # noqa: E402


def main():
    __graft_entry__.build()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    it = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    req = make_requests(n, seed=7)
    dreq = {key: torch.as_tensor(np.ascontiguousarray(v)).cuda() for key, v in req.items() if key != "in_len"}
    for _ in range(2):
        g = form_groups(dreq, 4, [k] * 4, limit=GROUP_LIMIT, max_iter=it)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        g = form_groups(dreq, 4, [k] * 4, limit=GROUP_LIMIT, max_iter=it)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    t0 = time.perf_counter()
    ref = O.form_groups(req, 4, [k] * 4, limit=GROUP_LIMIT, max_iter=it)
    cpu_s = time.perf_counter() - t0
    exact = (np.array_equal(g["label"].cpu().numpy(), ref["label"]) and
             np.array_equal(g["group_of"].cpu().numpy(), ref["group_of"]) and g["n_groups"] == ref["n_groups"])
    print(json.dumps(dict(requests=n, k_per_model=k, max_iter=it, iters=g["iters"], n_groups=g["n_groups"],
                          gpu_ms=round(ms, 3), requests_per_s=n / ms * 1e3,
                          lloyd_GBps_lower_bound=20 * n * g["iters"] / ms / 1e6,
                          oracle_s=round(cpu_s, 3), oracle_cores=1, bit_exact=bool(exact))))


if __name__ == "__main__":
    main()
