set -x
timeout 1200 python -m pytest tests/test_gpu_comm.py tests/test_gpu_parity.py -x -q -m gpu -k "winner or mc_sampler or step" > gpurun_out/win_tests.log 2>&1; tail -3 gpurun_out/win_tests.log
for r in 1 2; do
for lib in build/variants/libqlm_base.so ""; do
  if [ -n "$lib" ]; then export QLM_LIB_PATH=$lib; else unset QLM_LIB_PATH; fi
  timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])"
done
done
