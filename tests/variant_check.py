"""Subprocess body for tests/test_gpu_variants.py: every square n = 1..16, 2-D
and 3-D, fp32/fp64, alpha/beta != trivial, ragged batch, bit-exact against the
oracle -- run under whatever KB_* kernel-selection environment the caller set
(the library reads it once per process)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1304_7054_b200 as kb  # noqa: E402
from paper_1304_7054_b200 import (Array3View, BatchView, KronProblem2D, KronProblem3D, MatrixView,  # noqa: E402
                                  Workspace)

from kb_testutil import mismatches, oracle, to_dev, to_host  # noqa: E402


def main():
    o = oracle()
    bad = []
    for dims3 in (False, True):
        for dt in (np.float32, np.float64):
            for n in range(1, 17):
                for beta in (0.0, 1.0, -0.5):
                    batch = 37 + 5 * n
                    a, b, c, x, y = o.generate_batch(dt, 3, n, dims3, batch)
                    e = n ** (3 if dims3 else 2)
                    X, Y = to_dev(x), to_dev(y)
                    want = y.copy()
                    if dims3:
                        pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n, alpha=0.75, beta=beta)
                        kb.kron3(pr, MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n),
                                 MatrixView(to_dev(c), n, n, n), BatchView(Array3View(X, n, n, n, n, n * n), batch, e),
                                 BatchView(Array3View(Y, n, n, n, n, n * n), batch, e), Workspace(None, e * batch))
                        o.kron3("N", "N", "N", n, n, n, n, n, n, batch, dt(0.75), a, n, b, n, c, n, x, n, n * n, e,
                                dt(beta), want, n, n * n, e)
                    else:
                        pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n, alpha=0.75, beta=beta)
                        kb.kron2(pr, MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n),
                                 BatchView(MatrixView(X, n, n, n), batch, e), BatchView(MatrixView(Y, n, n, n), batch, e))
                        o.kron2("N", "N", "N", n, n, n, n, batch, dt(0.75), a, n, b, n, x, n, e, dt(beta), want, n, e)
                    path = kb.last_path()
                    mm = mismatches(to_host(Y), want)
                    if mm or not path.endswith("_fast"):
                        bad.append((dims3, dt.__name__, n, beta, path, mm))
    print("BAD", bad) if bad else print("OK")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
