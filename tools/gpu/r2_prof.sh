# ncu --set full of one library variant's ws2_kernel: tools/gpu/r2_prof.sh variant
v=$1
QLM_LIB_PATH=build/variants/libqlm_$v.so ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/prof_$v python tools/ws_time.py C3 1000000 3 > gpurun_out/ncu_log_$v.txt 2>&1
tail -3 gpurun_out/ncu_log_$v.txt
