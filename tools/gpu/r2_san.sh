compute-sanitizer --tool memcheck --show-backtrace no python tools/ws_time.py C3 8192 1 2>&1 | head -40 > gpurun_out/san.txt
cat gpurun_out/san.txt
