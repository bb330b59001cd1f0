set -x
python tools/ws_time.py C3 1000000 50 > gpurun_out/ws2_time.json 2>&1
QLM_NO_WS2=1 python tools/ws_time.py C3 1000000 50 > gpurun_out/ws1_time.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/ws2_gputest.txt
cat gpurun_out/ws2_time.json gpurun_out/ws1_time.json gpurun_out/ws2_gputest.txt
