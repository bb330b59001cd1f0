ncu --set full --clock-control none --import-source on -k regex:"tier_warp_kernel" -s 1 -c 1 -o gpurun_out/s3_tw python tools/c5_bulk.py 100000 C5h tiered > /dev/null 2>&1
ncu -i gpurun_out/s3_tw.ncu-rep --page source --csv --print-source sass > gpurun_out/s3_tw_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/s3_tw.ncu-rep 12 > gpurun_out/s3_tw_sum.txt 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv python tools/c5_bulk.py 100000 C5h tiered 2>/dev/null | grep -E "tier|fy_rows|big" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-150 > gpurun_out/s3_tw_split.txt
head -30 gpurun_out/s3_tw_sum.txt; cat gpurun_out/s3_tw_split.txt | head -20
