# Round-2 evidence: bench line, ncu launch list, one full capture of the fused kernel, reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-kernels > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ws2_kernel -s 3 -c 1 -o gpurun_out/r2_ws2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/r2_ncu_log.txt 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_reference.json 2> gpurun_out/r2_reference.err
tail -2 gpurun_out/r2_bench.err; cat gpurun_out/r2_bench.json | head -c 3000
