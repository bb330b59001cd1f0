python tools/c5_split.py 1000000 > gpurun_out/s3_c5_time.txt 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__warps_active.avg.per_cycle_active --csv python tools/c5_split.py 1000000 > gpurun_out/s3_c5_ncu.csv 2>&1
cat gpurun_out/s3_c5_time.txt
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/s3_c5_ncu.csv")) if len(r) > 10]
h = rows[0]; body = rows[1:]
ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in body:
    k = r[ki].split("(")[0][:60]
    try: agg[k][r[mi]] += float(r[vi].replace(",", ""))
    except ValueError: pass
    if r[mi] == "gpu__time_duration.sum": cnt[k] += 1
for k, m in agg.items():
    print(k, cnt[k], {x: round(v / (cnt[k] if 'pct' in x or 'per_cycle' in x else 1), 3) for x, v in m.items()})
PY
