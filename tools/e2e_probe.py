"""e2e time of the headline workload (host X/Y staged through the library)
under the current KB_STAGE_* / KB_COPY_THREADS settings (development aid).
  python tools/e2e_probe.py [batch] [pinned|pageable]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1304_7054_b200 as kb  # noqa: E402

n = 16
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 4194304
kind = sys.argv[2] if len(sys.argv) > 2 else "pinned"
e = n * n
if kind == "pinned":
    X = (torch.rand(e * batch) * 2 - 1).pin_memory()
    Y = torch.empty(e * batch).pin_memory()
else:
    X = np.random.default_rng(0).random(e * batch, dtype=np.float32)
    Y = np.zeros(e * batch, np.float32)
A, B = torch.rand(e), torch.rand(e)
args = (kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n), kb.MatrixView(A, n, n, n), kb.MatrixView(B, n, n, n),
        kb.BatchView(kb.MatrixView(X, n, n, n), batch, e), kb.BatchView(kb.MatrixView(Y, n, n, n), batch, e))
kb.kron2(*args)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    kb.kron2(*args)
    ts.append(time.perf_counter() - t0)
t = min(ts)
print(f"{kind:8s} e2e {t * 1e3:7.1f} ms  {2 * 4 * e * batch / t / 1e9:6.1f} GB/s over PCIe (both directions)  "
      f"{4 * n ** 3 * batch / t / 1e9:5.0f} GFlop/s", flush=True)
