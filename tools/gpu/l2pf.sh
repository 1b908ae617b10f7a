for e in "X=1" "KB_K2=0" "KB_K2=1"; do echo "$e: $(env $e timeout 600 python tests/variant_check.py | tail -1)"; done
timeout 900 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_golden.py tests/test_gpu_runtime.py tests/test_gpu_sanitizer.py -m gpu -q 2>&1 | tail -1
for pf in 0 1 0 1; do KB_L2PF=$pf timeout 300 python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import torch, bench
import paper_1304_7054_b200 as kb
topo = bench.Topo([0], 1, 0)
g = min(bench.time_graph(kb, torch, topo, "kron2-f32-n10", 200, 7) for _ in range(3)) * 1e3
ms, launch_ms, *_ = bench.time_device(kb, torch, topo, "kron2-f32-n16", 20, 5)
print(f"L2PF={os.environ['KB_L2PF']}: configs[0] graph {g:.2f} us/launch; headline per-launch {launch_ms*1e3:.1f} us", flush=True)
PY
done
