set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -m gpu -k "wide or large or C5 or c5 or two_phase" > gpurun_out/wide_tests.log 2>&1; tail -5 gpurun_out/wide_tests.log
for cfg in C5 C4; do
  QLM_LIB_PATH=build/variants/libqlm_base.so timeout 300 python tools/ws_time.py $cfg 100000 30
  timeout 300 python tools/ws_time.py $cfg 100000 30
done
