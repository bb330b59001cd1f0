timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/v_gputest.txt 2>&1; tail -2 gpurun_out/v_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python tools/ws_time.py C3 1000000 50
timeout 600 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; python -c "
import json; d=json.load(open('gpurun_out/v_bench.json')); r=d['roofline']; print('bench', d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['e2e']['value'], d['clocks'])"
