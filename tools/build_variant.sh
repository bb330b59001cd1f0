#!/bin/bash
# Build an experimental libqlm.so with extra -D flags for one source (default
# qlm_ws2.cu; VAR_SRC=qlm_large picks another) -- A/B timing through
# QLM_LIB_PATH; the other objects are cached.
#   [VAR_SRC=qlm_large] tools/build_variant.sh NAME [-DFLAG ...]  ->  build/variants/libqlm_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
vs=${VAR_SRC:-qlm_ws2}
C=paper_2407_00047_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include"
mkdir -p build/objs build/variants
objs=""
for f in qlm_api qlm_kernels qlm_ws qlm_ws2 qlm_wide qlm_req qlm_tier qlm_group qlm_big qlm_comm qlm_large; do
  [ $f = $vs ] && continue
  o=build/objs/$f.o
  objs="$objs $o"
  if [ ! -f $o ] || [ $C/$f.cu -nt $o ] || [ -n "$(find $C include -name '*.cuh' -newer $o -o -name '*.h' -newer $o)" ]; then
    nvcc $F -c -o $o $C/$f.cu &
  fi
done
nvcc $F "$@" -c -o build/objs/${vs}_$name.o $C/$vs.cu &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -ldl -o build/variants/libqlm_$name.so $objs build/objs/${vs}_$name.o
echo build/variants/libqlm_$name.so
