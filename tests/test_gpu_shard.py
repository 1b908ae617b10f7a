"""Multi-GPU batch sharding through the C ABI on ONE GPU (-m gpu): an exec
with devices [0, 0, 0] makes the runtime split a host-resident batch into
three contiguous slices, one host thread each (its own thread-local streams,
pools and staging), joined before return. The result must be
bit-identical to the unsharded call -- the determinism contract of
README.md:73-75 across worker counts, here across GPUs/threads -- for kron2,
kron3, kron1 and gemm_a, including batches that do not divide evenly."""
import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from kb_testutil import mismatches, oracle, rng, uniform

pytestmark = pytest.mark.gpu
MV, BV = kb.MatrixView, kb.BatchView


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n, batch", [(16, 1001), (10, 777), (7, 5)])
def test_kron2_kron3_sharded_equal_unsharded(dtype, n, batch):
    o = oracle()
    for dims3 in (False, True):
        a, b, c, x, y = o.generate_batch(dtype, 5, n, dims3, batch)
        e = n ** (3 if dims3 else 2)
        outs = []
        for ex in (None, kb.Exec(devices=[0, 0, 0])):
            Y = y.copy()
            if dims3:
                pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n, alpha=0.5, beta=1.5)
                kb.kron3(pr, MV(a, n, n, n), MV(b, n, n, n), MV(c, n, n, n),
                         BV(kb.Array3View(x, n, n, n, n, n * n), batch, e), BV(kb.Array3View(Y, n, n, n, n, n * n), batch, e),
                         kb.Workspace(None, e * batch), exec_=ex)
            else:
                pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n, alpha=0.5, beta=1.5)
                kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), BV(MV(x, n, n, n), batch, e), BV(MV(Y, n, n, n), batch, e),
                         exec_=ex)
            outs.append(Y)
        assert mismatches(outs[0], outs[1]) == 0
        want = y.copy()
        if dims3:
            o.kron3("N", "N", "N", n, n, n, n, n, n, batch, dtype(0.5), a, n, b, n, c, n, x, n, n * n, e, dtype(1.5), want,
                    n, n * n, e)
        else:
            o.kron2("N", "N", "N", n, n, n, n, batch, dtype(0.5), a, n, b, n, x, n, e, dtype(1.5), want, n, e)
        assert mismatches(outs[1], want) == 0


def test_kron1_gemm_a_sharded_equal_unsharded():
    g = rng(11)
    m, n_a, batch = 12, 9, 1003
    A = uniform(g, m * n_a, np.float32)
    X = uniform(g, n_a * batch, np.float32)
    Y0 = uniform(g, m * batch, np.float32)
    outs = []
    for ex in (None, kb.Exec(devices=[0, 0])):
        Y = Y0.copy()
        kb.kron1("N", m, n_a, np.float32(0.75), MV(A, m, n_a, m), BV(kb.VectorView(X, n_a), batch, n_a), np.float32(-1.0),
                 BV(kb.VectorView(Y, m), batch, m), exec_=ex)
        outs.append(Y)
    assert mismatches(outs[0], outs[1]) == 0
    k, n = 7, 5
    A2 = uniform(g, k * m * batch, np.float64)
    B2 = uniform(g, k * n, np.float64)
    C0 = uniform(g, m * n * batch, np.float64)
    outs = []
    for ex in (None, kb.Exec(devices=[0, 0, 0, 0])):
        C = C0.copy()
        kb.gemm_a("T", "N", m, n, k, 1.25, BV(MV(A2, k, m, k), batch, k * m), MV(B2, k, n, k), 0.5,
                  BV(MV(C, m, n, m), batch, m * n), exec_=ex)
        outs.append(C)
    assert mismatches(outs[0], outs[1]) == 0
