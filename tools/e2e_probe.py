"""e2e (pinned host X/Y, PCIe staged) time of the headline workload under the
current KB_STAGE_* settings (development aid)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1304_7054_b200 as kb  # noqa: E402

n, batch = 16, int(sys.argv[1]) if len(sys.argv) > 1 else 4194304
e = n * n
X = (torch.rand(e * batch) * 2 - 1).pin_memory()
Y = torch.empty(e * batch).pin_memory()
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
print(f"e2e {t * 1e3:.1f} ms  {2 * 4 * e * batch / t / 1e9:.1f} GB/s over PCIe (both directions)  "
      f"{4 * n ** 3 * batch / t / 1e9:.0f} GFlop/s")
