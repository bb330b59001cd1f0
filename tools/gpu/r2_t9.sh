timeout 900 python -m pytest tests -m gpu -q -x -k "tier" 2>&1 | tail -2 > gpurun_out/gputest.txt
python tools/kernel_suite.py > gpurun_out/suite.json 2> gpurun_out/suite.err
cat gpurun_out/gputest.txt
python -c "import json; [print(x['config'], x['name'][:60], '%.4g'%x['value'], '%.4f'%x['ms']) for x in json.load(open('gpurun_out/suite.json')) if x['config'] in ('C5','C5h')]"
