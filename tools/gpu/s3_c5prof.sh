ncu --set full --clock-control none --import-source on -k regex:"fy_rows_kernel|scan_kernel" -s 2 -c 2 -o gpurun_out/s3_c5 python tools/c5_split.py 262144 > gpurun_out/s3_c5prof_log.txt 2>&1
for k in fy_rows_kernel scan_kernel; do
  ncu -i gpurun_out/s3_c5.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/s3_c5_${k}_src.csv 2>/dev/null
done
ncu -i gpurun_out/s3_c5.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,sm__warps_active.avg.per_cycle_active > gpurun_out/s3_c5_raw.csv 2>&1
cat gpurun_out/s3_c5_raw.csv | cut -c1-300 | head
