"""Per-kernel roofline lines (a line per config against its
binding roof).  Imported by bench.py (the JSON line's `kernels` list) and run
standalone under ncu to refresh the instruction / DRAM counts it reports:

    python tools/kernel_suite.py                  # print the list (JSON)
    ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum --csv --log-file gpurun_out/suite.csv python tools/kernel_suite.py --once
    python tools/kernel_suite.py --ingest gpurun_out/suite.csv   # -> profiles/r2_kernels_ncu.json

Each item times one library call with CUDA events on its stream (median of
`reps` after warm-up).  HBM-bound items report algorithmic bytes / time
against the measured copy peak; issue-bound items (score-only scans, the MC
sampler and walk) report the ncu-measured warp instructions of their dominant
kernel / time against the SM issue roof (148 SMs x 4 schedulers x 1 warp
instruction per cycle at the sampled clock).
"""
from __future__ import annotations

import csv
import json
import os
import re
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NCU_JSON = os.path.join(ROOT, "profiles", "r2_kernels_ncu.json")


def _time(fn, reps, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def items():
    """(name, config, setup) triples; setup() -> (fn, units, unit, bytes or None, kernel regex)."""
    import numpy as np
    import torch
    from paper_2407_00047_b200 import RwtEstimator
    from workloads.synth import balanced_row, make_config, make_tiers

    def c3_explicit():
        p = make_config("C3")
        e = RwtEstimator(p)
        n = 1_000_000
        rows = e.rows(e.random(0, n, seed=1))                      # uint16 [n][T]
        buf = torch.zeros((n, 80), dtype=torch.uint8, device="cuda")
        buf[:, :p.T] = rows.to(torch.uint8)
        cand = e.explicit(buf)
        out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
        return (lambda: e.rwt_estimate(cand, out=out)), n, "orderings/s", n * (80 + 12 * p.G), \
            r"ws2_kernel<\(int\)0"

    def score_only(cfg, n):
        def setup():
            e = RwtEstimator(make_config(cfg))
            cand = e.random(0, n, seed=1)
            rec = torch.empty(2, dtype=torch.int64, device="cuda")
            return (lambda: e.best_ordering_async(cand, rec)), n, "orderings/s", None, \
                r"scan_kernel|fy_rows_kernel|large_kernel"
        return setup

    def c4_mc():
        p = make_config("C4")
        e = RwtEstimator(p)
        trials = 1221
        samples = trials * int(np.sum(p.n_req))
        return (lambda: e.mc_sample(2, trials)), samples, "samples/s", None, r"mc_sample_kernel"

    def c4_mc_count():
        p = make_config("C4")
        e = RwtEstimator(p)
        trials = 1221
        e.mc_sample(2, trials)
        row = balanced_row(p.G, p.Q)
        buf = np.zeros((1, p.row_stride // 2), np.int16)
        buf[0, :p.T] = row
        cand = e.explicit(torch.tensor(buf, device="cuda"))
        cnt = torch.empty((1, p.G), dtype=torch.int32, device="cuda")
        return (lambda: e.mc_count(cand, trials, counts=cnt)), trials * p.G, "slot-trials/s", None, \
            r"mc_count_kernel"

    def bulk(cfg, n, tiered=False):
        def setup():
            p = make_config(cfg)
            e = RwtEstimator(p)
            if tiered:
                e.set_tiers(make_tiers(dev_rows=tuple(range(p.theta.shape[0]))))
            cand = e.random(0, n, seed=1)
            out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
            rec = torch.empty(2, dtype=torch.int64, device="cuda")
            fn = (lambda: e.tiered_score_estimate(cand, out=out, scores=False, rec=rec)) if tiered else \
                (lambda: e.score_estimate(cand, out=out, scores=False, rec=rec))
            return fn, n, "orderings/s", n * 12 * p.G, r"tier_warp_kernel|tier_kernel" if tiered else \
                r"wide_kernel|fy_rows_kernel|scan_kernel"
        return setup

    def c2_step(graph):
        def setup():
            p = make_config("C2")
            e = RwtEstimator(p)
            n = 100_000
            cand = e.random(0, n, seed=1)
            out = {k: torch.empty((p.G, n), device="cuda") for k in ("wt", "sd", "v")}
            rec = torch.empty(2, dtype=torch.int64, device="cuda")

            def step():
                e.score_estimate(cand, out=out, scores=False, rec=rec)
                e.decode(e.from_record(rec, seed=1))
            if not graph:
                return step, n, "orderings/s", n * 12 * p.G, r"ws2_kernel<1, 32|row_warp_kernel"
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step()                                   # warm-up (opt-ins, tensor maps)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            keep = (e, cand, out, rec)                   # the graph replays into these: keep them alive

            def replay():
                g.replay()
                return keep
            return replay, n, "orderings/s", n * 12 * p.G, r"ws2_kernel<1, 32|row_warp_kernel"
        return setup

    def c3_search():
        p = make_config("C3")
        e = RwtEstimator(p)
        start = np.arange(p.T)
        per, iters = 65536, 64
        return (lambda: e.local_search(start, moves=2, per_iter=per, iters=iters, seed=3)), per * iters, \
            "orderings/s", None, r"scan_kernel|adopt_kernel"

    return [
        ("rwt_estimate EXPLICIT u8 rows (ws2_kernel, bulk only)", "C3", c3_explicit),
        ("best_ordering_async RANDOM (score + argmin only)", "C2", score_only("C2", 1_000_000)),
        ("best_ordering_async RANDOM (score + argmin only)", "C3", score_only("C3", 1_000_000)),
        ("best_ordering_async RANDOM (two-phase: fy_rows + large_kernel)", "C5", score_only("C5", 1_000_000)),
        ("mc_sample 1221 trials (Philox + length tables)", "C4", c4_mc),
        ("mc_count 1221 trials of one ordering", "C4", c4_mc_count),
        ("score_estimate RANDOM bulk + argmin (wide_kernel)", "C5", bulk("C5", 100_000)),
        ("tiered_score_estimate RANDOM bulk + argmin", "C5h", bulk("C5h", 100_000, tiered=True)),
        ("tiered_score_estimate RANDOM bulk + argmin (ws2 kernel, TIER)", "C3", bulk("C3", 1_000_000, tiered=True)),
        ("local_search 64 x 65536 NEIGHBOR (2 moves)", "C3", c3_search),
        ("step: score_estimate 1e5 + winner decode, direct launches", "C2", c2_step(False)),
        ("step: score_estimate 1e5 + winner decode, CUDA graph replay", "C2", c2_step(True)),
    ]


def _ncu_counts():
    try:
        with open(NCU_JSON) as f:
            return json.load(f)
    except Exception:
        return {}


def run(reps=20, hbm_peak=None, clk_mhz=1965.0, once=False):
    import torch
    out = []
    counts = _ncu_counts()
    ipeak = 148 * 4 * clk_mhz * 1e6
    for name, cfg, setup in items():
        print(f"# {cfg} {name}", file=sys.stderr, flush=True)
        fn, units, unit, nbytes, kre = setup()
        if once:
            fn()
            torch.cuda.synchronize()
            print(f"#suite {cfg} {name}", flush=True)
            continue
        ms = _time(fn, reps)
        line = {"name": name, "config": cfg, "value": units / (ms / 1e3), "unit": unit, "ms": ms}
        key = f"{cfg} | {name}"
        nc = counts.get(key)
        if nbytes is not None and hbm_peak:
            gbs = nbytes / (ms / 1e3) / 1e9
            line["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                                "frac": gbs / hbm_peak, "bytes_per_call": nbytes,
                                "traffic": nc.get("dram_bytes") if nc else None}
        elif nc and nc.get("inst"):
            # the dominant kernels' warp instructions over the call's duration
            ach = nc["inst"] / (ms / 1e3)
            line["roofline"] = {"bound": "issue", "achieved": ach, "peak": ipeak,
                                "unit": "warp instructions/s", "frac": ach / ipeak,
                                "inst_per_call": nc["inst"], "source": "profiles/r2_kernels_ncu.json"}
        else:
            line["roofline"] = None
        out.append(line)
    return out


def ingest(csv_path):
    """ncu launch CSV (--csv --log-file, the --once run) -> per-item totals of
    the kernels matching each item's regex, in item order."""
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    launches = {}
    order = []
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        lid = r[0]
        if lid not in launches:
            launches[lid] = {"kernel": r[ik]}
            order.append(lid)
        v = float(r[iv].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "usecond": 1e-6,
                 "msecond": 1e-3}.get(r[iu], 1)
        launches[lid][r[im]] = v * scale
    # the suite's --once run launches its items in order; walk them item by item
    res = {}
    pos = 0
    seq = [launches[i] for i in order]
    # group: an item's launches are those from after the previous item's kernels
    # up to its own matching kernels (matching by regex, in order)
    for name, cfg, setup in items_meta():
        kre = re.compile(setup)
        inst = dram = t = 0.0
        found = False
        while pos < len(seq):
            L = seq[pos]
            if kre.search(L["kernel"]):
                found = True
                inst += L.get("smsp__inst_executed.sum", 0.0)
                dram += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
                t += L.get("gpu__time_duration.sum", 0.0)
                pos += 1
            elif found:
                break
            else:
                pos += 1
        res[f"{cfg} | {name}"] = {"inst": inst, "dram_bytes": dram, "ncu_seconds": t,
                                  "kernels": setup}
    os.makedirs(os.path.dirname(NCU_JSON), exist_ok=True)
    json.dump(res, open(NCU_JSON, "w"), indent=1)
    print(json.dumps(res, indent=1))


def items_meta():
    # the dominant kernels of each item (ncu prints template arguments as <0, 64, 0>)
    return [
        ("rwt_estimate EXPLICIT u8 rows (ws2_kernel, bulk only)", "C3", r"ws2_kernel<0,"),
        ("best_ordering_async RANDOM (score + argmin only)", "C2", r"scan_kernel<1, unsigned char"),
        ("best_ordering_async RANDOM (score + argmin only)", "C3", r"scan_kernel<1, unsigned char"),
        ("best_ordering_async RANDOM (two-phase: fy_rows + large_kernel)", "C5", r"fy_rows_kernel|large_kernel|scan_kernel<7|reduce_records"),
        ("mc_sample 1221 trials (Philox + length tables)", "C4", r"mc_sample_kernel"),
        ("mc_count 1221 trials of one ordering", "C4", r"mc_count_kernel"),
        ("score_estimate RANDOM bulk + argmin (wide_kernel)", "C5", r"fy_rows_kernel|wide_kernel|reduce_records"),
        ("tiered_score_estimate RANDOM bulk + argmin", "C5h", r"tier_warp_kernel|tier_kernel|big_kernel"),
        ("tiered_score_estimate RANDOM bulk + argmin (ws2 kernel, TIER)", "C3", r"ws2_kernel<1, \d+, \d, (true|1)>|ws_kernel<1, unsigned char, 1, \d, 1>"),
        ("local_search 64 x 65536 NEIGHBOR (2 moves)", "C3", r"scan_kernel<[03], unsigned char|adopt_kernel"),
        ("step: score_estimate 1e5 + winner decode, direct launches", "C2", r"ws2_kernel<1, 32|row_warp_kernel"),
        ("step: score_estimate 1e5 + winner decode, CUDA graph replay", "C2", r"ws2_kernel<1, 32|row_warp_kernel"),
    ]


if __name__ == "__main__":
    import __graft_entry__
    if len(sys.argv) > 2 and sys.argv[1] == "--ingest":
        ingest(sys.argv[2])
        sys.exit(0)
    __graft_entry__.build()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    if "--once" in sys.argv:
        run(once=True)
    else:
        print(json.dumps(run(hbm_peak=peaks.get("hbm_gbs", 6650.0)), indent=1))
