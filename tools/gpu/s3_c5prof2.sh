ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none --csv python tools/c5_split.py 262144 > gpurun_out/s3_c5b_ncu.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:"large_kernel" -s 1 -c 1 -o gpurun_out/s3_lg python tools/c5_split.py 262144 > /dev/null 2>&1
ncu -i gpurun_out/s3_lg.ncu-rep --page source --csv --print-source sass > gpurun_out/s3_lg_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/s3_lg.ncu-rep 10 > gpurun_out/s3_lg_sum.txt 2>&1
grep -E "large_kernel|fy_rows" gpurun_out/s3_c5b_ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200 | head -30
head -25 gpurun_out/s3_lg_sum.txt
