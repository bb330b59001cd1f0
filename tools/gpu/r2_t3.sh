python tools/ws_time.py C3 1000000 50 > gpurun_out/t.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/gputest.txt
compute-sanitizer --tool memcheck python tools/ws_time.py C3 20000 2 2>&1 | tail -5 > gpurun_out/san.txt
compute-sanitizer --tool racecheck python tools/ws_time.py C3 20000 2 2>&1 | tail -5 >> gpurun_out/san.txt
cat gpurun_out/t.txt gpurun_out/gputest.txt gpurun_out/san.txt
