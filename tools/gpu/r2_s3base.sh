# Session-3 baseline on the restored tree: GPU suite, fused-pass timing, bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/s3_gputest.txt
python tools/ws_time.py C3 1000000 50 > gpurun_out/s3_ws.json 2>&1
python bench.py --no-kernels > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
cat gpurun_out/s3_gputest.txt gpurun_out/s3_ws.json; head -c 2500 gpurun_out/s3_bench.json
