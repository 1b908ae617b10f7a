"""Host-side cost per call for a small batch (BASELINE configs[0]: 2-D fp32 n=10,
batch 65536): wall time per asynchronous call, device time per launch, and the
same launches replayed from a CUDA graph (development aid)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1304_7054_b200 as kb  # noqa: E402
from paper_1304_7054_b200 import BatchView, KronProblem2D, MatrixView  # noqa: E402

n, batch, reps = 10, int(sys.argv[1]) if len(sys.argv) > 1 else 65536, 200
e = n * n
X = torch.rand(e * batch, device="cuda") * 2 - 1
Y = torch.empty(e * batch, device="cuda")
A, B = (torch.rand(n * n) * 2 - 1 for _ in range(2))
s = torch.cuda.Stream()
ex = kb.Exec(stream=s, asynchronous=True)
args = (KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n), MatrixView(A, n, n, n), MatrixView(B, n, n, n),
        BatchView(MatrixView(X, n, n, n), batch, e), BatchView(MatrixView(Y, n, n, n), batch, e))
for _ in range(5):
    kb.kron2(*args, exec_=ex)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    kb.kron2(*args, exec_=ex)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"python api: {1e6 * (t1 - t0) / reps:.1f} us/call host, {1e6 * (t2 - t0) / reps:.1f} us/call incl. drain")
# device time per launch when launches are queued back to back
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(20):
        kb.kron2(*args, exec_=ex)
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
ev0.record(s)
for _ in range(10):
    with torch.cuda.stream(s):
        g.replay()
ev1.record(s)
torch.cuda.synchronize()
us = ev0.elapsed_time(ev1) * 1e3 / 200
print(f"cuda graph: {us:.2f} us/launch -> {4 * n ** 3 * batch / us / 1e6:.1f} GFlop/s, "
      f"{8 * e * batch / us / 1e3:.1f} GB/s")
