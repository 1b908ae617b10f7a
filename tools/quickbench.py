"""Quick device-resident timing of the fast kernels (development aid, not the bench contract)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1304_7054_b200 as kb  # noqa: E402
from paper_1304_7054_b200 import Array3View, BatchView, KronProblem2D, KronProblem3D, MatrixView, Workspace  # noqa


def bench(dims3, n, batch, dtype, reps=10):
    tdt = torch.float32 if dtype == "f32" else torch.float64
    es = 4 if dtype == "f32" else 8
    e = n ** (3 if dims3 else 2)
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.rand(e * batch, dtype=tdt, device="cuda", generator=g) * 2 - 1
    Y = torch.empty(e * batch, dtype=tdt, device="cuda")
    A, B, C = (torch.rand(n * n, dtype=tdt, device="cuda", generator=g) * 2 - 1 for _ in range(3))
    s = torch.cuda.Stream()
    ex = kb.Exec(stream=s, asynchronous=True)
    if dims3:
        pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        args = (pr, MatrixView(A, n, n, n), MatrixView(B, n, n, n), MatrixView(C, n, n, n),
                BatchView(Array3View(X, n, n, n, n, n * n), batch, e), BatchView(Array3View(Y, n, n, n, n, n * n), batch, e),
                Workspace(None, e * batch))
        fn = kb.kron3
    else:
        pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
        args = (pr, MatrixView(A, n, n, n), MatrixView(B, n, n, n), BatchView(MatrixView(X, n, n, n), batch, e),
                BatchView(MatrixView(Y, n, n, n), batch, e))
        fn = kb.kron2
    for _ in range(3):
        fn(*args, exec_=ex)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        fn(*args, exec_=ex)
        b.record(s)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    ms = ts[len(ts) // 2]
    flops = (6 * n ** 4 if dims3 else 4 * n ** 3) * batch
    byts = 2 * e * es * batch
    print(f"{'3d' if dims3 else '2d'} {dtype} n={n:2d} batch={batch:8d} path={kb.last_path():14s} "
          f"{ms:8.3f} ms  {flops / ms / 1e9:8.1f} TF/s  {byts / ms / 1e6:7.1f} GB/s  (min {ts[0]:.3f})", flush=True)


def bench_gemm_a(n, dtype, opa="N", reps=10):
    """gemm_a C^p = alpha op(A^p) B + beta C^p, square n, 2 GiB of A (device-resident)."""
    tdt = torch.float32 if dtype == "f32" else torch.float64
    es = 4 if dtype == "f32" else 8
    e = n * n
    batch = max(1, int(2 * 1024 ** 3 // (e * es)))
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.rand(e * batch, dtype=tdt, device="cuda", generator=g) * 2 - 1
    Cm = torch.empty(e * batch, dtype=tdt, device="cuda")
    B = torch.rand(e, dtype=tdt, device="cuda", generator=g) * 2 - 1
    s = torch.cuda.Stream()
    ex = kb.Exec(stream=s, asynchronous=True)
    args = (opa, "N", n, n, n, 1.0, BatchView(MatrixView(A, n, n, n), batch, e), MatrixView(B, n, n, n), 0.0,
            BatchView(MatrixView(Cm, n, n, n), batch, e))
    for _ in range(3):
        kb.gemm_a(*args, exec_=ex)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        kb.gemm_a(*args, exec_=ex)
        b.record(s)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    ms = ts[len(ts) // 2]
    print(f"gemm_a op{opa} {dtype} n={n:2d} batch={batch:8d} {ms:8.3f} ms  {2 * n ** 3 * batch / ms / 1e9:8.1f} TF/s  "
          f"{2 * e * es * batch / ms / 1e6:7.1f} GB/s  (min {ts[0]:.3f})", flush=True)


def bench_kron1(n, dtype, reps=10):
    """kron1 y^p = A x^p (shared A), square n, 2 GiB of x (device-resident)."""
    from paper_1304_7054_b200 import VectorView
    tdt = torch.float32 if dtype == "f32" else torch.float64
    es = 4 if dtype == "f32" else 8
    batch = max(1, int(2 * 1024 ** 3 // (n * es)))
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.rand(n * batch, dtype=tdt, device="cuda", generator=g) * 2 - 1
    Y = torch.empty(n * batch, dtype=tdt, device="cuda")
    A = torch.rand(n * n, dtype=tdt, device="cuda", generator=g) * 2 - 1
    s = torch.cuda.Stream()
    ex = kb.Exec(stream=s, asynchronous=True)
    args = ("N", n, n, 1.0, MatrixView(A, n, n, n), BatchView(VectorView(X, n), batch, n), 0.0,
            BatchView(VectorView(Y, n), batch, n))
    for _ in range(3):
        kb.kron1(*args, exec_=ex)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        kb.kron1(*args, exec_=ex)
        b.record(s)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    ms = ts[len(ts) // 2]
    print(f"kron1 {dtype} n={n:2d} batch={batch:9d} {ms:8.3f} ms  {2 * n * n * batch / ms / 1e9:8.1f} TF/s  "
          f"{2 * n * es * batch / ms / 1e6:7.1f} GB/s  (min {ts[0]:.3f})", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "main"
    if which == "main":
        bench(False, 16, 4194304, "f32")
        bench(False, 10, 65536 * 16, "f32")
        bench(True, 16, 262144, "f32")
        bench(True, 10, 262144, "f32")
        bench(True, 16, 131072, "f64")
        bench(False, 16, 2097152, "f64")
    elif which == "one":  # one <2|3> <n> <f32|f64> <batch> [reps]
        reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
        bench(sys.argv[2] == "3", int(sys.argv[3]), int(sys.argv[5]), sys.argv[4], reps=reps)
    elif which == "gemm_a":  # gemm_a [f32|f64]: square n = 1..16, op_a N and T
        for dt in sys.argv[2:] or ["f32", "f64"]:
            for n in range(1, 17):
                for opa in ("N", "T"):
                    bench_gemm_a(n, dt, opa, reps=5)
    elif which == "kron1":  # kron1 [f32|f64]: square n = 1..16
        for dt in sys.argv[2:] or ["f32", "f64"]:
            for n in range(1, 17):
                bench_kron1(n, dt, reps=5)
    elif which == "sweepd":  # sweepd <2|3> <f32|f64>: one rank / dtype of the size sweep
        dims3, dt = sys.argv[2] == "3", sys.argv[3]
        es = 4 if dt == "f32" else 8
        for n in range(1, 17):
            e = n ** (3 if dims3 else 2)
            bench(dims3, n, max(1, int(2 * 1024 ** 3 // (e * es))), dt, reps=5)
    else:
        for dims3 in (False, True):
            for dt in ("f32", "f64"):
                for n in range(1, 17):
                    es = 4 if dt == "f32" else 8
                    e = n ** (3 if dims3 else 2)
                    batch = max(1, int(2 * 1024 ** 3 // (e * es)))
                    bench(dims3, n, batch, dt, reps=5)
