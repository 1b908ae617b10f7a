timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --devices 0,0 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/torchrun2.json 2> gpurun_out/torchrun2.err; echo rc=$?
cat gpurun_out/torchrun2.json | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print({k: d.get(k) for k in ('value','n_gpus','ms_per_step','gpu_launches')}); print(d['config']); print(d['e2e']); [print(e['workload'], e['scaling'], e['entries_total'], e['entries_per_gpu'], e['value']) for e in d['extra']]
"
grep -v "^\s*$" gpurun_out/torchrun2.err | tail -5
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 2>&1 | grep '^{' | cut -c1-200
