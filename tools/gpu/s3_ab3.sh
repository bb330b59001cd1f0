QLM_LOG=1 QLM_LIB_PATH=build/variants/libqlm_w7.so python tools/ws_time.py C3 1000000 3 2>&1 | grep -m2 "ws2_kernel\|median"
bash tools/gpu/s3_ab.sh both w6n w7
