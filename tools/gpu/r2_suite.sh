python tools/kernel_suite.py > gpurun_out/suite.json 2> gpurun_out/suite.err
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/suite.csv python tools/kernel_suite.py --once > gpurun_out/suite_once.txt 2>&1
tail -3 gpurun_out/suite.err; cat gpurun_out/suite.json | python -c "import json,sys; [print(x['config'], x['name'][:50], round(x['value']/1e9,4), round(x['ms'],4), (x['roofline'] or {}).get('frac')) for x in json.load(sys.stdin)]"
