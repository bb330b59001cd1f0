set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest0.txt
python tools/ws_time.py C3 1000000 50 > gpurun_out/r2_ws0.json 2>&1
python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
cat gpurun_out/r2_gputest0.txt gpurun_out/r2_ws0.json gpurun_out/r2_bench0.json
