# GPU suite against the bounds-checked build (device QLM_CHECKs), then the
# normal build's fused-pass timing (the checks compile to nothing there)
QLM_LIB_PATH=build/bounds/libqlm_bounds.so timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/b_gputest.txt 2>&1
tail -3 gpurun_out/b_gputest.txt; grep -m3 "QLM_CHECK" gpurun_out/b_gputest.txt
QLM_LIB_PATH=build/bounds/libqlm_bounds.so timeout 600 python tools/san_paths.py > gpurun_out/b_paths.txt 2>&1; tail -6 gpurun_out/b_paths.txt
python tools/ws_time.py C3 1000000 50
