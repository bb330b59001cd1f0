#!/bin/bash
# Bounds-checked library (device QLM_CHECKs on, -DQLM_BOUNDS) for the GPU tests:
#   tools/build_bounds.sh  ->  build/bounds/libqlm_bounds.so   (QLM_LIB_PATH=... python -m pytest -m gpu)
set -e
cd "$(dirname "$0")/.."
C=paper_2407_00047_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include -DQLM_BOUNDS"
mkdir -p build/bounds
objs=""
for f in qlm_api qlm_kernels qlm_ws qlm_ws2 qlm_wide qlm_req qlm_tier qlm_group qlm_big qlm_comm qlm_large; do
  nvcc $F -c -o build/bounds/$f.o $C/$f.cu &
  objs="$objs build/bounds/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -ldl -o build/bounds/libqlm_bounds.so $objs
echo build/bounds/libqlm_bounds.so
