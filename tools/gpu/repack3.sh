timeout 900 python -m pytest tests/test_gpu_kron2.py tests/test_gpu_kron3.py tests/test_gpu_golden.py -m gpu -q 2>&1 | tail -1
timeout 600 python - <<'PY'
import sys
sys.path.insert(0, "tools")
import sweep_configs4 as s
for d3, n in ((False, 4), (False, 7), (False, 10), (False, 16), (True, 4), (True, 7), (True, 10), (True, 16)):
    for dt in ("f32", "f64"):
        batch, t, tf, gbs, path = s.run(d3, n, dt, 1024, 10, 3)
        print(f"{'3d' if d3 else '2d'} {dt} n={n} pad=3: {t*1e3:.3f} ms {tf:.2f} TF/s {gbs:.0f} GB/s {path}", flush=True)
PY
