"""BASELINE.json configs[4]: size sweep n = 2..16 x {2-D, 3-D} x {fp32, fp64}
against the roofline, device-resident, with the batch sized to 1 GiB of X per
size (batch = ceil(2^30 / (n^d * sizeof T)), the reference's memory-scaled
batches, bench_support.cpp:270-297) so every row moves >= 2 GiB of HBM
traffic; plus padded-layout rows (ld = n + 3, entry stride padded too) that
run the generic kernels. Median of CUDA-event-timed reps on one stream.

    python tools/sweep_configs4.py [--reps 10] [--mb 1024] [--gpus-note ...]
"""
import argparse
import json
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1304_7054_b200 as kb  # noqa: E402

FP_PEAK = {"f32": 72.5, "f64": 33.6}  # measured FFMA / DFMA peaks, TFLOP/s (profiles/r01_fma_tput.txt)


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def run(dims3, n, dt, mb, reps, pad=0):
    tdt = torch.float32 if dt == "f32" else torch.float64
    es = 4 if dt == "f32" else 8
    e_tight = n ** (3 if dims3 else 2)
    ld = n + pad
    e_store = (ld * n * n + pad) if dims3 else (ld * n + pad)  # padded entry stride
    batch = math.ceil((mb << 20) / (e_tight * es))
    g = torch.Generator(device="cuda").manual_seed(n)
    X = torch.rand(e_store * batch, dtype=tdt, device="cuda", generator=g)
    Y = torch.zeros(e_store * batch, dtype=tdt, device="cuda")
    A, B, C = (torch.rand(n * n, dtype=tdt) for _ in range(3))
    MV, BV = kb.MatrixView, kb.BatchView
    s = torch.cuda.Stream()
    ex = kb.Exec(stream=s, asynchronous=True)
    if dims3:
        pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        args = (pr, MV(A, n, n, n), MV(B, n, n, n), MV(C, n, n, n),
                BV(kb.Array3View(X, n, n, n, ld, ld * n), batch, e_store),
                BV(kb.Array3View(Y, n, n, n, ld, ld * n), batch, e_store), kb.Workspace(None, e_tight * batch))
        fn = kb.kron3
    else:
        pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
        args = (pr, MV(A, n, n, n), MV(B, n, n, n), BV(MV(X, n, n, ld), batch, e_store),
                BV(MV(Y, n, n, ld), batch, e_store))
        fn = kb.kron2
    for _ in range(3):
        fn(*args, exec_=ex)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(*args, exec_=ex)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t = statistics.median(ts)
    path = kb.last_path()
    del X, Y
    flops = (6 * n ** 4 if dims3 else 4 * n ** 3) * batch
    algo_bytes = 2 * e_tight * es * batch  # X read + Y written (tight payload)
    return batch, t, flops / t / 1e12, algo_bytes / t / 1e9, path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--mb", type=int, default=1024)
    args = ap.parse_args()
    peak = hbm_peak()
    print(f"# configs[4] sweep on {torch.cuda.get_device_name(0)}: X = {args.mb} MiB per size, device-resident, "
          f"median of {args.reps}; roof = min(FP peak, {peak:.0f} GB/s x AI)")
    print("| dims | dtype | n | layout | batch | ms | TFLOP/s | GB/s | roof TF | frac | kernel |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    rows = [(d3, dt, n, 0) for d3 in (False, True) for dt in ("f32", "f64") for n in range(2, 17)]
    rows += [(d3, "f32", n, 3) for d3 in (False, True) for n in (4, 8, 10, 16)]
    for d3, dt, n, pad in rows:
        batch, t, tf, gbs, path = run(d3, n, dt, args.mb, args.reps, pad)
        es = 4 if dt == "f32" else 8
        ai = (6 * n ** 4 if d3 else 4 * n ** 3) / (2 * n ** (3 if d3 else 2) * es)
        roof = min(FP_PEAK[dt], peak * ai / 1e3)
        print(f"| {'3-D' if d3 else '2-D'} | {dt} | {n} | {'ld=n+3' if pad else 'tight'} | {batch} | {t * 1e3:.3f} | "
              f"{tf:.2f} | {gbs:.0f} | {roof:.1f} | {tf / roof:.3f} | {path} |", flush=True)


if __name__ == "__main__":
    main()
