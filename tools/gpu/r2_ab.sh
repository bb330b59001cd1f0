# A/B timing of library variants: tools/gpu/r2_ab.sh name1 name2 ...  (old = round-1 kernel control)
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do for v in "$@"; do
  if [ $v = old ]; then QLM_NO_WS2=1 QLM_LIB_PATH=build/variants/libqlm_base.so python tools/ws_time.py C3 1000000 50 | sed "s/^/$v /" >> $out 2>&1
  else QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/ws_time.py C3 1000000 50 | sed "s/^/$v /" >> $out 2>&1; fi
done; done
cat $out
