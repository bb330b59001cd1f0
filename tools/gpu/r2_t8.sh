timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gputest.txt
python tools/kernel_suite.py > gpurun_out/suite.json 2> gpurun_out/suite.err
cat gpurun_out/gputest.txt; grep "Error\|error" gpurun_out/suite.err | tail -3
python -c "import json; [print(x['config'], x['name'][:60], '%.4g'%x['value'], '%.4f'%x['ms']) for x in json.load(open('gpurun_out/suite.json'))]"
