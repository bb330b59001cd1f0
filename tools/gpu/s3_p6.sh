# correctness first (bounded), then timing
QLM_LIB_PATH=build/variants/libqlm_p6on.so timeout 300 python tools/ws_time.py C3 1000000 5 || { echo "P6 HUNG/FAILED"; exit 1; }
QLM_LIB_PATH=build/variants/libqlm_p6on.so timeout 900 python -m pytest tests -q -m gpu -x -k "bulk or ws2 or fifo or fused or bench_step or warp_specialised or tiers_ws or edges or neighbor" 2>&1 | tail -3
bash tools/gpu/s3_ab.sh p6off p6on
