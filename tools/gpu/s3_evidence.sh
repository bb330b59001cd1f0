# Session-3 evidence: GPU tests, smoke, bench line (+ kernels list), ncu launch
# list, full capture of the fused kernel, kernel-suite ncu metrics, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/e_smi.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/e_gputest.txt 2>&1; tail -3 gpurun_out/e_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/e_smoke.txt 2>&1; tail -1 gpurun_out/e_smoke.txt
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/e_suite.csv python tools/kernel_suite.py --once > gpurun_out/e_suite_once.txt 2>&1
python tools/kernel_suite.py --ingest gpurun_out/e_suite.csv > gpurun_out/e_ingest.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/e_ws2_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/e_ncu_log.txt 2>&1
ncu -i gpurun_out/e_ws2_full.ncu-rep --page raw --csv > gpurun_out/e_ws2_raw.csv 2>/dev/null
python tools/update_traffic.py gpurun_out/e_ws2_raw.csv "session-3 capture of the bench step's ws2_kernel" > gpurun_out/e_traffic.txt 2>&1
python tools/ncu_summary.py gpurun_out/e_ws2_full.ncu-rep 14 > gpurun_out/e_ws2_sum.txt 2>&1
timeout 600 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-kernels > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/e_reference.json 2> gpurun_out/e_reference.err
cp profiles/ncu_traffic.json profiles/r2_kernels_ncu.json gpurun_out/ 2>/dev/null
tail -2 gpurun_out/e_bench.err; head -c 1500 gpurun_out/e_bench.json
