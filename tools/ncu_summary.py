"""Summarise an ncu --set full report of one kernel: the headline counters and
the stall samples / executed instructions of its hottest SASS ranges.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block",
        "sm__cycles_elapsed.avg.per_second"]


def ncu(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    raw = ncu(rep, "raw")
    d = dict(zip(raw[0], raw[2]))
    for k in KEYS:
        if k in d:
            print(f"{k:80s} {d[k]}")
    stalls = sorted(((float(v), k) for k, v in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")), reverse=True)
    print("stalls per issue:", ", ".join(f"{k[34:-27]}={v:.2f}" for v, k in stalls[:8]))
    rows = ncu(rep, "source", ["--print-source", "sass"])
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    body = [r for r in rows[hi + 1:] if len(r) == len(h)]
    cs, ce = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = int(body[0][0], 16)
    runs, prev = [], None
    for r in body:
        off, e, smp = int(r[0], 16) - base, int(r[ce] or 0), int(r[cs] or 0)
        if prev is None or e != prev[2]:
            prev = [off, off, e, 0, 0]
            runs.append(prev)
        prev[1] = off
        prev[3] += e
        prev[4] += smp
    tot_s = sum(r[4] for r in runs) or 1
    tot_e = sum(r[3] for r in runs) or 1
    print(f"samples {tot_s}, warp instructions {tot_e}")
    for r in sorted(runs, key=lambda r: -r[4])[:top]:
        print(f"  {r[0]:05x}-{r[1]:05x} exec/inst {r[2]:9d} instr {r[3]:10d} ({r[3] / tot_e:5.1%})  samples {r[4]:6d} ({r[4] / tot_s:5.1%})")


if __name__ == "__main__":
    main()
