python tools/c5_bulk.py 100000 C5 > gpurun_out/s3_wide_time.txt 2>&1
python tools/c5_bulk.py 100000 C5h tiered >> gpurun_out/s3_wide_time.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"wide_kernel" -s 1 -c 1 -o gpurun_out/s3_wide python tools/c5_bulk.py 100000 > /dev/null 2>&1
ncu -i gpurun_out/s3_wide.ncu-rep --page source --csv --print-source sass > gpurun_out/s3_wide_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/s3_wide.ncu-rep 12 > gpurun_out/s3_wide_sum.txt 2>&1
cat gpurun_out/s3_wide_time.txt; head -40 gpurun_out/s3_wide_sum.txt
