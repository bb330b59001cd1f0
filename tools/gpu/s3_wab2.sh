for rep in 1 2; do for v in "$@"; do
  echo "$v C5 $(QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/c5_bulk.py 100000 C5 2>&1 | tail -1)"
done; done
QLM_LIB_PATH=build/variants/libqlm_$2.so timeout 900 python -m pytest tests -q -m gpu -x -k "wide or large_G or two_phase or neighbor_bulk or c5" 2>&1 | tail -2
