# A/B timing of library variants (build/variants/libqlm_NAME.so), 3 interleaved rounds
out=gpurun_out/s3_ab.txt; : > $out
for rep in 1 2 3; do for v in "$@"; do
  QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/ws_time.py C3 1000000 50 | sed "s/^/$v /" >> $out 2>&1
done; done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for line in open("gpurun_out/s3_ab.txt"):
    n, _, j = line.partition(" ")
    try: d[n].append(json.loads(j)["median_ms"])
    except Exception: print(line.strip())
for n, v in d.items(): print(f"{n:12s} " + " ".join(f"{x:.4f}" for x in v) + f"   min {min(v):.4f}")
PY
