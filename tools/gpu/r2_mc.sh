set -x
timeout 1200 python -m pytest tests -x -q -m gpu -k "mc or MC or step or comm" > gpurun_out/mc_tests.log 2>&1; tail -3 gpurun_out/mc_tests.log
for lib in build/variants/libqlm_base.so ""; do
  if [ -n "$lib" ]; then export QLM_LIB_PATH=$lib; else unset QLM_LIB_PATH; fi
  timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['ms_per_step'], d['step']['fused_scan_ms'], d['e2e']['value'])"
done
unset QLM_LIB_PATH
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:mc_ --csv --log-file gpurun_out/mc_ncu.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-kernels > /dev/null 2>&1
grep -h "mc_sample\|mc_count" gpurun_out/mc_ncu.csv | head -6 | cut -c1-50,200-400
