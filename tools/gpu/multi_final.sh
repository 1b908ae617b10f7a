bash tools/gpu/torchrun2.sh
timeout 600 python bench.py --gpus 2 --devices 0,0 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('single-process', {k: d.get(k) for k in ('value','n_gpus','ms_per_step','gpu_launches')}); [print(' ', e['workload'], e['scaling'], e['entries_total'], e['value']) for e in d['extra']]
"
