for o in wt,sd,v wt wt,sd; do python tools/ws_time.py C3 1000000 50 $o; done > gpurun_out/probe_time.txt 2>&1
python tools/ws_time.py C3 4000000 20 >> gpurun_out/probe_time.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/ws2_full python tools/ws_time.py C3 1000000 3 > gpurun_out/ncu_log.txt 2>&1
cat gpurun_out/probe_time.txt
