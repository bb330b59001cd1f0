timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gputest.txt
QLM_LOG=1 python tools/ws_time.py C2 100000 3 2> gpurun_out/qlm_log.txt > /dev/null
python tools/kernel_suite.py > gpurun_out/suite.json 2> gpurun_out/suite.err
cat gpurun_out/gputest.txt; head -5 gpurun_out/qlm_log.txt; tail -3 gpurun_out/suite.err
python -c "import json; [print(x['config'], x['name'][:60], '%.4g'%x['value'], '%.4f'%x['ms']) for x in json.load(open('gpurun_out/suite.json'))]"
