#!/bin/bash
# Build an experimental libqlm.so with extra -D flags for qlm_ws2.cu only
# (A/B timing through QLM_LIB_PATH; the other objects are cached).
#   tools/build_variant.sh NAME [-DFLAG ...]  ->  build/variants/libqlm_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
C=paper_2407_00047_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include"
mkdir -p build/objs build/variants
for f in qlm_api qlm_kernels qlm_ws qlm_wide qlm_req qlm_tier qlm_group qlm_big qlm_comm; do
  o=build/objs/$f.o
  if [ ! -f $o ] || [ $C/$f.cu -nt $o ] || [ -n "$(find $C -name '*.cuh' -newer $o)" ] || [ $C/qlm_launch.h -nt $o ]; then
    nvcc $F -c -o $o $C/$f.cu &
  fi
done
nvcc $F "$@" -c -o build/objs/ws2_$name.o $C/qlm_ws2.cu &
wait
nvcc $F -shared -ldl -o build/variants/libqlm_$name.so build/objs/qlm_*.o build/objs/ws2_$name.o
echo build/variants/libqlm_$name.so
