# GPU suite + fused-pass timing + bench line (no kernels list)
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/s3_gputest.txt
python tools/ws_time.py C3 1000000 50 > gpurun_out/s3_ws.json 2>&1
python bench.py --no-kernels --no-cpu-baseline > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
cat gpurun_out/s3_gputest.txt gpurun_out/s3_ws.json; python -c "
import json; d=json.load(open('gpurun_out/s3_bench.json')); r=d['roofline']; print('bench', d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['e2e']['value'])"
