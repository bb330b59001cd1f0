for i in 1 2; do python bench.py --no-kernels --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value', d['value'], 'ms', d['ms_per_step'], 'kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'e2e', d['e2e']['value'], d['gpu_launches'])"; done
git_stash_dummy=1
