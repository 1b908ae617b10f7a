"""CPU baseline + full-batch parity for one BASELINE workload (TEST / MEASUREMENT
INFRASTRUCTURE -- the checker, never the product).

Run as its own process (one config per process), launched by
bench.py's cpu_baseline leg and by tests/test_gpu_parity_full.py:

    python -m oracle.cpu_ref --workload kron2-f32-n16 [--batch B] [--reps 10]
                             [--parity] [--max-seconds S]

1. Pins OpenMP before the reference library is loaded (OMP_PROC_BIND=close,
   OMP_PLACES=cores, OMP_WAIT_POLICY=active; all host cores), as BASELINE.md §3
   and the reference's own protocol ask (bench_support.cpp:256-265).
2. Generates the workload with the reference's generator
   (kronbench::generate_batch, seed 1, bench_support.hpp:148-170) at its FULL
   batch (or --batch), alpha 1, beta 0, tight layout.
3. Times the unmodified reference (oracle/_ref/libkronref.so:
   kronbatch::kron2<T> / kron3<T>) -- one warm-up, then the median of --reps
   runs (steady clock, bench_support.cpp:256-265); GFlop/s with the paper's
   flop count (bench_support.cpp:31-35).
4. --parity: runs the PRODUCT (paper_1304_7054_b200, sm_100a) on the same host
   buffers and compares the WHOLE batch: bitwise mismatch count and the
   per-entry rel_err_inf maximum (tests/test_util.hpp:93-113), tolerance
   1e-5 / 1e-12.

Prints one JSON object on stdout. Imports no torch (so the OpenMP runtime is
the reference's own, initialised with the pinning above).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

OMP_ENV = {"OMP_PROC_BIND": "close", "OMP_PLACES": "cores", "OMP_WAIT_POLICY": "active"}

WORKLOADS = {
    # name: (dims3, n, dtype, full batch)  -- BASELINE.json configs[0..3]
    "kron2-f32-n10": (False, 10, "f32", 65536),
    "kron2-f32-n16": (False, 16, "f32", 4194304),
    "kron3-f32-n10": (True, 10, "f32", 262144),
    "kron3-f32-n16": (True, 16, "f32", 262144),
    "kron3-f64-n16": (True, 16, "f64", 131072),
}


def host_info():
    model, numa = platform.processor(), None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("NUMA node(s)"):
                numa = int(ln.split(":")[1])
            if ln.startswith("Model name") and not model:
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model, "numa_nodes": numa}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True, choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="entries (default: the workload's full batch)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--max-seconds", type=float, default=60.0, help="stop timing after this long (>= 3 reps)")
    ap.add_argument("--parity", action="store_true", help="also run the product on the same inputs and compare")
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args(argv)
    # host cores, read before the OpenMP runtime starts (OMP_PROC_BIND pins the
    # initial thread to one core once the reference library is loaded)
    ncores = len(os.sched_getaffinity(0))

    for k, v in OMP_ENV.items():
        os.environ.setdefault(k, v)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import numpy as np

    from oracle.oracle import Oracle, Reference

    dims3, n, dtype, full = WORKLOADS[args.workload]
    batch = args.batch or full
    dt = np.float32 if dtype == "f32" else np.float64
    e = n ** (3 if dims3 else 2)
    ref = Reference()
    assert ref.has_openmp, "reference built without OpenMP"
    # every host core unless told otherwise (a torchrun parent exports OMP_NUM_THREADS=1)
    ref.set_threads(args.threads or ncores)
    t0 = time.perf_counter()
    a, b, c, x, y = ref.generate_batch(dt, 1, n, dims3, batch)
    gen_s = time.perf_counter() - t0
    yref = np.zeros_like(x)
    work = np.empty(n * n * n * batch if dims3 else 0, dt)

    def run_ref():
        if dims3:
            ref.kron3("N", "N", "N", n, n, n, n, n, n, batch, dt(1), a, (n, n), n, b, (n, n), n, c, (n, n), n, x,
                      (n, n, n), n, n * n, e, dt(0), yref, (n, n, n), n, n * n, e, work)
        else:
            ref.kron2("N", "N", "N", n, n, n, n, batch, dt(1), a, (n, n), n, b, (n, n), n, x, (n, n), n, e, dt(0), yref,
                      (n, n), n, e)

    run_ref()  # warm-up: first touch of the workspace, OpenMP team start-up
    times = []
    t_end = time.perf_counter() + args.max_seconds
    while len(times) < args.reps and (len(times) < 3 or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        run_ref()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    flops = (6 * n ** 4 if dims3 else 4 * n ** 3) * batch
    out = {
        "workload": args.workload, "batch": batch, "full_batch": batch == full, "gflops": flops / med / 1e9,
        "median_s": med, "min_s": min(times), "max_s": max(times), "reps": len(times), "cores": ref.max_threads,
        "omp": {k: os.environ.get(k) for k in OMP_ENV}, "host": host_info(), "generate_s": round(gen_s, 2),
        "kind": "reference", "impl": "oracle/_ref/libkronref.so (unmodified kronbatch, g++ -O3 -march=native -fopenmp)",
    }
    if args.parity:
        import paper_1304_7054_b200 as kb  # the product under test (ctypes; no torch)

        ygpu = np.full_like(x, np.nan)
        MV, BV = kb.MatrixView, kb.BatchView
        t0 = time.perf_counter()
        if dims3:
            pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
            kb.kron3(pr, MV(a, n, n, n), MV(b, n, n, n), MV(c, n, n, n),
                     BV(kb.Array3View(x, n, n, n, n, n * n), batch, e), BV(kb.Array3View(ygpu, n, n, n, n, n * n), batch, e),
                     kb.Workspace(None, e * batch))
        else:
            pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
            kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), BV(MV(x, n, n, n), batch, e), BV(MV(ygpu, n, n, n), batch, e))
        gpu_s = time.perf_counter() - t0
        ub = np.uint32 if dt == np.float32 else np.uint64
        mism = int(np.count_nonzero(ygpu.view(ub) != yref.view(ub)))
        # per-entry rel_err_inf = max|g - w| / max(1, max|w|)   (tests/test_util.hpp:93-103)
        worst = 0.0
        step = max(1, (64 << 20) // (e * ygpu.itemsize))
        for p0 in range(0, batch, step):
            g = ygpu[p0 * e:(p0 + step) * e].reshape(-1, e).astype(np.float64)
            w = yref[p0 * e:(p0 + step) * e].reshape(-1, e).astype(np.float64)
            err = np.abs(g - w).max(axis=1) / np.maximum(1.0, np.abs(w).max(axis=1))
            worst = max(worst, float(err.max()))
        tol = 1e-5 if dt == np.float32 else 1e-12
        out["parity"] = {"entries": batch, "full_batch": batch == full, "mismatches": mism,
                         "max_rel_err_inf": worst, "tol": tol, "ok": bool(worst <= tol),
                         "vs": "unmodified reference kronbatch (oracle/_ref), same generate_batch inputs",
                         "product_path": kb.last_path(), "product_call_s": round(gpu_s, 3),
                         "product_buffers": "pageable host (numpy)"}
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
