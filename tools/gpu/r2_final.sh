# Round-2 final evidence: GPU tests, smoke, bench line (+ kernels list),
# ncu launch list, full capture of the fused kernel, kernel-suite ncu metrics,
# reference arm, sanitizers
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_gputest.txt 2>&1; tail -3 gpurun_out/r2_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke.txt 2>&1; tail -1 gpurun_out/r2_smoke.txt
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-kernels > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/r2_ws2_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/r2_ncu_log.txt 2>&1
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/suite.csv python tools/kernel_suite.py --once > gpurun_out/suite_once.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_reference.json 2> gpurun_out/r2_reference.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --show-backtrace no python tools/san_paths.py > gpurun_out/san_$tool.txt 2>&1
  tail -3 gpurun_out/san_$tool.txt
done
tail -2 gpurun_out/r2_bench.err; head -c 1500 gpurun_out/r2_bench.json
