timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gputest.txt
python bench.py --steps 200 --warmup 10 --no-kernels --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err
QLM_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-kernels > gpurun_out/b2.json 2> gpurun_out/b2.err
cat gpurun_out/gputest.txt; tail -2 gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['d2h_bytes_per_step'])"
tail -3 gpurun_out/b2.err; head -c 400 gpurun_out/b2.json
