# A/B of library variants on C5 score-only (1e6 candidates)
for rep in 1 2; do for v in "$@"; do
  echo "$v $(QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/c5_split.py 1000000 2>&1 | tail -1)"
done; done | tee gpurun_out/s3_c5ab.txt
