for e in "X=1" "KB_K2=2"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 900 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_golden.py tests/test_gpu_runtime.py -m gpu -q 2>&1 | tail -1
timeout 300 python tools/bench_one.py kron2-f32-n10 sleep1 kron2-f32-n16
timeout 300 python - <<'PY'
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_1304_7054_b200 as kb
topo = bench.Topo([0], 1, 0)
print("graph us/launch", min(bench.time_graph(kb, torch, topo, "kron2-f32-n10", 200, 7) for _ in range(3)) * 1e3)
PY
