# Session-3 final evidence: GPU suite, smoke, sanitizers, bench (+ kernels), launch list,
# fused-kernel capture, kernel-suite ncu metrics, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_smi.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/f_gputest.txt 2>&1; tail -3 gpurun_out/f_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.txt 2>&1; tail -1 gpurun_out/f_smoke.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --show-backtrace no python tools/san_paths.py > gpurun_out/f_san_$tool.txt 2>&1
  tail -3 gpurun_out/f_san_$tool.txt
done
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f_suite.csv python tools/kernel_suite.py --once > gpurun_out/f_suite_once.txt 2>&1
python tools/kernel_suite.py --ingest gpurun_out/f_suite.csv > gpurun_out/f_ingest.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/f_ws2_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/f_ncu_log.txt 2>&1
ncu -i gpurun_out/f_ws2_full.ncu-rep --page raw --csv > gpurun_out/f_ws2_raw.csv 2>/dev/null
python tools/update_traffic.py gpurun_out/f_ws2_raw.csv "final session-3 capture of the bench step's ws2_kernel" > gpurun_out/f_traffic.txt 2>&1
python tools/ncu_summary.py gpurun_out/f_ws2_full.ncu-rep 14 > gpurun_out/f_ws2_sum.txt 2>&1
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-kernels > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_reference.json 2> gpurun_out/f_reference.err
cp profiles/ncu_traffic.json profiles/r2_kernels_ncu.json gpurun_out/ 2>/dev/null
tail -2 gpurun_out/f_bench.err; head -c 1200 gpurun_out/f_bench.json
