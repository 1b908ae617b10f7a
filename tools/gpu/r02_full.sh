# Full round check: every -m gpu test, smoke, bench (headline + extras + cpu/parity), reference arm.
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/bench.json", "gpurun_out/bench_ref.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, {k: d.get(k) for k in ("value", "ms_per_step", "n_gpus", "gpu_launches")})
    for k in ("roofline", "e2e", "e2e_pageable", "clocks", "cpu_baseline", "parity"):
        if k in d: print(" ", k, d[k])
    for e in d.get("extra", []): print("  extra", e)
PY
