#!/usr/bin/env python
"""Bench: RWT-scored queue orderings / s on 1..8 B200 (BASELINE.json metric).

One step = one pass of the whole hot path over one batch of
C3 (64 groups, 4 models, 8 virtual queues) on every GPU:
  a1-a7     qlm_score_estimate, ONE fused kernel: 1e6 RANDOM candidates
            generated on the device, Eq. 10 scan, violation probabilities,
            per-(group, candidate) wt / sd / v written to HBM (768 MB fp32),
            S1/S2 and the argmin record
  a8        global min-loc: NCCL all-gather of 16-B records + reduce kernel
  a9        decode of the global winner (queue, position per group)
  a10-a12   MC check of the winner: qlm_mc_sample (1221 Philox trials per
            GPU, candidate-independent: on a side stream, filling SMs as the
            fused pass drains and overlapping a8/a9) then qlm_mc_count of the
            winner; counts summed with one NCCL all-reduce.  (Running the sampler on a second
            stream concurrently with the fused scan was measured: the step
            gains ~2 % while the scan slows by the same SM time, so the step
            keeps them sequential for a clean per-kernel roofline.)
Weak scaling: rank r scores global indices [r*1e6, (r+1)*1e6).

`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded sample
of the same step on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = "C3"
N_PER_GPU = 1_000_000
MC_TRIALS = 1221
METRIC = "RWT-scored queue orderings/sec"
# the path's arithmetic: Eq. 10 waiting-time sums, slack and S2 in fp64; the
# variance sum, z, Phi-bar, S1 terms and every bulk output in fp32 (R22)
DTYPE = "f64+f32"
UNIT = "orderings/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel roofline list")
    ap.add_argument("--config", default="C3", choices=["C2", "C3", "C5", "C5h"],
                    help="workload (BASELINE.json configs); the metric is quoted on C3")
    ap.add_argument("--candidates", type=int, default=None,
                    help="candidates per GPU per step (default 1e6)")
    return ap.parse_args()


SHAPES = {"C2": (16, 2, 2), "C3": (64, 8, 4), "C5": (1024, 32, 4), "C5h": (1024, 32, 4)}


def workload_config(world):
    G, Q, M = SHAPES[CFG]
    return {
        "workload": f"{CFG}: {G} request groups, {M} models (7B/13B/70B-like), {Q} virtual queues "
                    f"(App. B profiles); per GPU per step {N_PER_GPU:.0e} RANDOM candidate "
                    f"orderings scored + argmin, bulk per-group wt/sd/v for all of them, "
                    f"MC ({MC_TRIALS} trials) of the global winner",
        "groups": G, "queues": Q, "models": M, "candidates_per_gpu": N_PER_GPU,
        "mc_trials_per_gpu": MC_TRIALS, "parallelism": f"dp{world}",
        "l2": f"not flushed explicitly: every step writes {12 * G * N_PER_GPU / 1e6:.0f} MB of bulk "
              "estimates per GPU (> the 126 MB L2), evicting it between steps",
    }


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {N.nvmlClocksThrottleReasonHwSlowdown: "hw_slowdown",
                     N.nvmlClocksThrottleReasonHwThermalSlowdown: "hw_thermal_slowdown",
                     N.nvmlClocksThrottleReasonSwThermalSlowdown: "sw_thermal_slowdown",
                     N.nvmlClocksThrottleReasonSwPowerCap: "sw_power_cap"}

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for bit, name in names.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(self.period)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML missing: report that instead of a number
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- oracle leg
def oracle_sample(n_cand: int, trials: int, first: int = 0):
    """One bounded sample of the step on the CPU oracle: candidates
    [first, first + n_cand) scored + argmin, their bulk estimates, the
    winner's estimate and `trials` MC trials of it; returns seconds."""
    import numpy as np
    import oracle as O
    from workloads.synth import make_config, CANDIDATE_SEED, MC_SEED
    p = make_config(CFG)
    o = O.Oracle(p)
    t0 = time.perf_counter()
    r = o.score_range(O.RANDOM, first, n_cand, seed=CANDIDATE_SEED)
    best = first + O.argmin_key(r["s1"], r["s2"])
    o.estimate_range(O.RANDOM, first, n_cand, seed=CANDIDATE_SEED)
    row = O.random_row(CANDIDATE_SEED, best, p.T)
    o.estimate(row)
    if trials > 0:
        X = o.mc_sample(MC_SEED, first, trials)
        o.mc_count(O.EXPLICIT, 0, 1, X, rows=row[None, :].astype(np.uint8))
    return time.perf_counter() - t0


def _oracle_chunk(args):
    return oracle_sample(*args)


def cpu_baseline(budget_s: float = 15.0):
    """Oracle on a bounded sample: ~budget_s of single-thread CPU work, then
    the same sample split over every host core (one process per core, the
    oracle unchanged).  The all-core figure is the reported baseline."""
    import multiprocessing as mp
    t = oracle_sample(2000, 2)
    n = int(max(2000, min(N_PER_GPU, 2000 * budget_s / max(t, 1e-6))))
    trials = max(1, round(MC_TRIALS * n / N_PER_GPU))
    t1 = oracle_sample(n, trials)
    cores = os.cpu_count() or 1
    try:
        if hasattr(os, "sched_getaffinity"):
            cores = len(os.sched_getaffinity(0))
        chunks = [(n // cores + (1 if i < n % cores else 0), max(1, trials // cores),
                   i * (n // cores) + min(i, n % cores)) for i in range(cores)]
        with mp.get_context("fork").Pool(cores) as pool:
            pool.map(_oracle_chunk, [(200, 1, 0)] * cores)          # warm the workers
            w0 = time.perf_counter()
            pool.map(_oracle_chunk, chunks)
            tp = time.perf_counter() - w0
    except Exception:
        cores, tp = 1, t1
    return {"value": n / tp, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} of the {N_PER_GPU} {CFG} candidates of one step (score+argmin, bulk "
                      f"estimates) + MC {trials} of {MC_TRIALS} trials, plain C fp64 oracle "
                      f"(-O2 -ffp-contract=off) split over {cores} host cores (one process each), "
                      f"{tp:.2f} s wall; value = sampled candidates / s",
            "single_core": {"value": n / t1, "cores": 1, "seconds": round(t1, 3)},
            "cpu_model": _cpu_model()}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    if rank != 0:
        return
    per = None
    # calibrate the per-step sample so that steps+warmup finish in ~120 s
    t = oracle_sample(2000, 2)
    budget = 120.0 / max(1, args.steps + args.warmup)
    n = int(max(200, min(N_PER_GPU, 2000 * budget / max(t, 1e-6))))
    trials = max(1, round(MC_TRIALS * n / N_PER_GPU))
    for _ in range(args.warmup):
        oracle_sample(n, trials)
    ts = [oracle_sample(n, trials) for _ in range(args.steps)]
    tot = sum(ts)
    per = tot / args.steps
    value = n / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"each step: {n} of the {N_PER_GPU} {CFG} candidates (score+argmin, "
                                   f"bulk estimates) + MC {trials} of {MC_TRIALS} trials; plain C "
                                   f"fp64 oracle, single thread"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our leg
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import __graft_entry__
    from paper_2407_00047_b200 import RwtEstimator, kernel_launches, groups_array
    from paper_2407_00047_b200.dist import attach_comm, global_best, sum_counts
    from workloads.synth import make_config, CANDIDATE_SEED, MC_SEED

    __graft_entry__.build()
    # QLM_BENCH_SHARE_GPU=1 (plumbing check only): several ranks on one GPU
    # over gloo, exercising the N > 1 code path where only one GPU exists;
    # the driver's multi-GPU runs use NCCL with one GPU per rank
    share = os.environ.get("QLM_BENCH_SHARE_GPU", "0") == "1"
    gpu = local_rank % torch.cuda.device_count() if share else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    p = make_config(CFG)
    est = RwtEstimator(p, device=gpu)
    if world > 1 and not share:
        # the library's own NCCL communicator (qlm_comm_attach): torch.distributed
        # only broadcasts its 128-byte id; the min-loc (a8) and the MC count sum
        # (a12) then run inside the C ABI on the step's stream
        attach_comm(est)
    G = p.G
    stream = torch.cuda.current_stream(dev)
    cand = est.random(first=rank * N_PER_GPU, count=N_PER_GPU, seed=CANDIDATE_SEED)
    rec = torch.empty(2, dtype=torch.int64, device=dev)
    bulk = {k: torch.empty((G, N_PER_GPU), dtype=torch.float32, device=dev) for k in ("wt", "sd", "v")}
    counts = torch.empty((1, G), dtype=torch.int32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    side = torch.cuda.Stream(dev)
    ev_f, ev_s = torch.cuda.Event(), torch.cuda.Event()

    def step(kt=None, groups_host=None, out_host=None):
        if groups_host is not None:
            est.update_groups(groups_host)                       # H2D of the step's inputs
        if kt:
            kt[0].record(stream)
        ev_f.record(stream)                  # the previous step's MC count is done
        est.score_estimate(cand, out=bulk, scores=False, rec=rec)   # fused a1-a7
        if kt:
            kt[1].record(stream)
        # a10 (candidate-independent) on a side stream, enqueued after the fused
        # pass but waiting only on the previous step: its blocks cannot share an
        # SM with a fused-pass block (shared memory), so they fill SMs as the
        # fused pass drains and overlap its tail, the min-loc exchange (NCCL for
        # N > 1) and the decode (measured: step 0.359 -> 0.346 ms, fused pass
        # unchanged)
        side.wait_event(ev_f)
        est.mc_sample(MC_SEED, MC_TRIALS, trial_first=rank * MC_TRIALS, stream=side)
        ev_s.record(side)
        g = global_best(rec, est.reduce_records, est=est)        # a8 (in the library when attached)
        win = est.from_record(g, seed=CANDIDATE_SEED)
        if out_host is None:
            est.decode(win)                                      # a9
        else:
            # a9 through the C ABI with the D2H of the step's result: qlm_winner
            # decodes (and scores) the global record's candidate and copies
            # (index, S1, S2, n_over, queue/position per group) into the
            # pinned host buffers on the stream
            est.winner(win, out_host)
        stream.wait_event(ev_s)
        est.mc_count(win, MC_TRIALS, counts=counts)              # a11
        sum_counts(counts, est=est)                              # a12 (in the library when attached)
        if out_host is not None:
            out_host["cnt"].copy_(counts.view(-1), non_blocking=True)
        return g

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-timed region
    K = args.steps
    kts = [[ev() for _ in range(2)] for _ in range(K)]
    e0, e1 = ev(), ev()
    barrier()
    torch.cuda.synchronize()
    l0 = kernel_launches()
    with ClockSampler(gpu) as clk:
        e0.record(stream)
        for k in range(K):
            step(kts[k])
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = kernel_launches() - l0
    t_ms = e0.elapsed_time(e1)
    fused_ms = sum(k[0].elapsed_time(k[1]) for k in kts) / K
    t = torch.tensor([t_ms, fused_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms, fused_ms = t.tolist()
    ms_per_step = t_ms / K
    value = N_PER_GPU * world / (ms_per_step / 1e3)

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        g_np = groups_array(p.model, p.n_req, p.slo, p.mu, p.var, p.dist)
        groups_host = torch.from_numpy(g_np.view(np.uint8).copy()).pin_memory()
        def host_out():
            return {"best": torch.empty(24, dtype=torch.uint8).pin_memory(),
                    "qo": torch.empty(G, dtype=torch.int32).pin_memory(),
                    "po": torch.empty(G, dtype=torch.int32).pin_memory(),
                    "cnt": torch.empty(G, dtype=torch.int32).pin_memory()}
        outs = [host_out(), host_out()]                           # double-buffered results
        out_host = outs[0]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        Ke = max(10, K // 5)
        for _ in range(3):
            step(groups_host=groups_host, out_host=out_host)
            stream.synchronize()
        barrier()
        torch.cuda.synchronize()
        x0, x1 = ev(), ev()
        x0.record(stream)
        # pipelined like a serving loop: step k is enqueued (its H2D, kernels,
        # D2H) before the host waits for and reads step k-1's result
        for k in range(Ke):
            step(groups_host=groups_host, out_host=outs[k % 2])
            done[k % 2].record(stream)
            if k > 0:
                done[(k - 1) % 2].synchronize()
                _ = RwtEstimator.best_of(outs[(k - 1) % 2]["best"])["index"]   # the host reads the result
        done[(Ke - 1) % 2].synchronize()
        _ = RwtEstimator.best_of(outs[(Ke - 1) % 2]["best"])["index"]
        x1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([x0.elapsed_time(x1) / Ke], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": N_PER_GPU * world / (te.item() / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(groups_host.numel()),
               "d2h_bytes_per_step": int(sum(v.numel() * v.element_size() for v in out_host.values())),
               "ms_per_step": te.item(),
               "note": "per step: pinned H2D of the 64 group records through qlm_update_groups + "
                       "table rebuild, the whole step, D2H of the winner (index, S1, S2, n_over, "
                       "decoded ordering) written into pinned host buffers by qlm_winner, D2H of the MC counts, and a host read of "
                       "the result; pipelined one step deep (the host reads step k-1 while step k runs)"}

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except Exception:
            pass
        hbm_peak = peaks.get("hbm_gbs")
        peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if hbm_peak else \
            "fallback 6650 GB/s (B200_PROFILING.md)"
        hbm_peak = hbm_peak or 6650.0
        bulk_bytes = N_PER_GPU * G * 3 * 4                     # algorithmic: outputs only (RANDOM)
        kname = ("ws2_kernel<RANDOM,GS=64,SCORE=1>" if G <= 64 else
                 "ws2_kernel<RANDOM,GS=128,SCORE=1>" if G <= 128 else "wide_kernel<RANDOM>")
        bulk_gbs = bulk_bytes / (fused_ms / 1e3) / 1e9
        traffic, winstr = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                nt_ = json.load(f).get(CFG, {})
                traffic = nt_.get("scan_kernel_dram_bytes_per_launch")
                winstr = nt_.get("smsp_inst_executed_per_launch")
        except Exception:
            pass
        roofline = {"kernel": kname + " (qlm_score_estimate, fused a1-a7)", "bound": "hbm",
                    "achieved": bulk_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": bulk_gbs / hbm_peak, "traffic": traffic,
                    "algorithmic_bytes_per_launch": bulk_bytes,
                    "bytes_per_unit": G * 12, "units_per_launch": N_PER_GPU,
                    "kernel_ms": fused_ms, "peak_source": peak_src}
        if winstr:
            # context for the HBM fraction: the same kernel against the SM issue
            # roof (4 schedulers x 1 warp instruction / cycle x 148 SMs at the
            # sampled clock), with the ncu-measured warp instructions per launch
            clk_mhz = clk.summary().get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0
            ipeak = 148 * 4 * clk_mhz * 1e6
            roofline["issue"] = {"achieved": winstr / (fused_ms / 1e3), "peak": ipeak,
                                 "unit": "warp instructions/s", "frac": winstr / (fused_ms / 1e3) / ipeak,
                                 "inst_per_launch": winstr,
                                 "source": "profiles/ncu_traffic.json (smsp__inst_executed.sum)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": workload_config(world),
            "roofline": roofline,
            "step": {"fused_scan_ms": fused_ms,
                     "fused_scan_orderings_per_s": N_PER_GPU / (fused_ms / 1e3),
                     "share_of_step": {"fused_scan": fused_ms / ms_per_step}},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_kernels:
            # every other kernel of the library against its binding roof
            # (SURVEY 8(d)); instruction counts from profiles/r2_kernels_ncu.json
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import kernel_suite
            clk_mhz = clk.summary().get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0
            main = {"name": "score_estimate RANDOM fused a1-a7 (" + kname + ")", "config": CFG,
                    "value": N_PER_GPU / (fused_ms / 1e3), "unit": UNIT, "ms": fused_ms,
                    "roofline": {k: roofline[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}}
            line["kernels"] = [main] + kernel_suite.run(reps=10, hbm_peak=hbm_peak, clk_mhz=clk_mhz)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    global CFG, N_PER_GPU
    args = parse()
    CFG = args.config
    if args.candidates:
        N_PER_GPU = args.candidates
    elif CFG in ("C5", "C5h"):
        N_PER_GPU = 100_000          # 1024 groups: 12 GB of bulk output would be 1e6
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
