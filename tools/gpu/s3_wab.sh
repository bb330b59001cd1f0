for rep in 1 2; do for v in "$@"; do
  echo "$v $(QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/c5_bulk.py 100000 C5 2>&1 | tail -1)"
done; done | tee gpurun_out/s3_wab.txt
