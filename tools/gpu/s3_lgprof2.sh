ncu --set full --clock-control none --import-source on -k regex:"large_kernel" -s 1 -c 1 -o gpurun_out/s3_lg2 python tools/c5_split.py 262144 > /dev/null 2>&1
ncu -i gpurun_out/s3_lg2.ncu-rep --page source --csv --print-source sass > gpurun_out/s3_lg2_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/s3_lg2.ncu-rep 8 > gpurun_out/s3_lg2_sum.txt 2>&1
head -24 gpurun_out/s3_lg2_sum.txt
