python tools/ws_time.py C3 1000000 50 > gpurun_out/t.txt 2>&1
python tools/ws_time.py C3 1000000 50 wt >> gpurun_out/t.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/ws2_full python tools/ws_time.py C3 1000000 3 > gpurun_out/ncu_log.txt 2>&1
cat gpurun_out/t.txt
