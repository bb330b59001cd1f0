# ncu capture of one fused C3 pass (QLM_LIB_PATH variant optional: $1) + per-SASS stall CSV
v=${1:-base}
lib=""; [ "$v" != base ] && lib="QLM_LIB_PATH=build/variants/libqlm_$v.so"
env $lib ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 5 -c 1 -o gpurun_out/s3_$v python tools/ws_time.py C3 1000000 3 > gpurun_out/s3_${v}_log.txt 2>&1
ncu -i gpurun_out/s3_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/s3_${v}_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/s3_$v.ncu-rep 14 > gpurun_out/s3_${v}_sum.txt 2>&1
cat gpurun_out/s3_${v}_sum.txt | head -40
