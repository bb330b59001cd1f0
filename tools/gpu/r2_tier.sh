set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tier" > gpurun_out/tier_tests.log 2>&1; tail -5 gpurun_out/tier_tests.log
python tools/kernel_suite.py > gpurun_out/suite.json 2> gpurun_out/suite.err
tail -3 gpurun_out/suite.err; cat gpurun_out/suite.json | python -c "import json,sys; [print(x['config'], x['name'][:60], round(x['value']/1e9,4), round(x['ms'],4), (x['roofline'] or {}).get('frac')) for x in json.load(sys.stdin)]"
