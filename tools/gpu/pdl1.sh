# PDL (programmatic dependent launch) A/B: correctness, then configs[0] and headline timings
for e in "X=1" "KB_K3=3" "KB_K2=0" "KB_K2=2"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 1500 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_kron2.py tests/test_gpu_kron3.py tests/test_gpu_shard.py -m gpu -q 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 build/sanitize/kb_sanitize full 2>&1 | tail -3
for r in 1 2; do for d in 0 1; do echo "PDL=$d"; KB_PDL=$d timeout 600 python bench.py --no-cpu --no-e2e --steps 30 --warmup 5 --cooldown 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' headline', d['ms_per_step'], d['roofline']['frac'])
for e in d.get('extra',[]): print(' ', e.get('workload'), e.get('ms_per_step'), e.get('value'), (e.get('roofline') or {}).get('frac'), e.get('cuda_graph'))
"; done; done
for c in "3 8 f64 262144" "3 16 f64 131072" "3 16 f64 32768" "3 14 f32 97827" "3 16 f32 262144" "3 9 f32 368225" "3 6 f32 1242757"; do for d in 0 1; do echo "DYN=$d $c: $(KB_DYN=$d timeout 60 python tools/quickbench.py one $c 10 2>&1 | tail -1)"; done; done
for c in "3 16 f64 131072" "2 10 f32 65536" "3 10 f32 262144"; do for d in 0 1; do echo "PDL=$d $c: $(KB_PDL=$d timeout 60 python tools/quickbench.py one $c 20 2>&1 | tail -1)"; done; done
