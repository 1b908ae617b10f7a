timeout 1500 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_variants.py tests/test_gpu_golden.py tests/test_gpu_runtime.py -m gpu -q -x 2>&1 | tail -3
for n in 10 16; do timeout 60 python tools/quickbench.py one 3 $n f32 262144 10 2>&1 | tail -1; done
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_k3.json 2>gpurun_out/bench_k3.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_k3.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'])
for e in d['extra']: print(e['workload'], e['value'], e['roofline'])"
