"""The tcgen05 3xTF32 tensor-core kron3 kernel (fp32, n = 16; opt-in via
Exec(tf32=True) / KB_EXEC_TF32): parity with the reference within the
1e-5 rel_err_inf contract (tests/test_util.hpp:93-113), every alpha/beta path,
op combinations, ragged batches, padded entry strides, and the BASELINE
config at full size. It is deliberately NOT bit-exact."""
import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from paper_1304_7054_b200 import Array3View, BatchView, Exec, KronProblem3D, MatrixOp, MatrixView, Workspace

from kb_testutil import oracle, rel_err_inf, rng, to_dev, to_host, uniform

pytestmark = pytest.mark.gpu
N_, T_ = MatrixOp.NoTranspose, MatrixOp.Transpose
n = 16
E = n ** 3


def run_tc(pr, a, b, c, x, y, batch, sx=E, sy=E, ldy=n, ldy2=n * n):
    X, Y = to_dev(x), to_dev(y)
    kb.kron3(pr, MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n), MatrixView(to_dev(c), n, n, n),
             BatchView(Array3View(X, n, n, n, n, n * n), batch, sx),
             BatchView(Array3View(Y, n, n, n, ldy, ldy2), batch, sy), Workspace(None, E * batch), Exec(tf32=True))
    return to_host(Y)


def oracle3(pr, a, b, c, x, y, batch):
    out = y.copy()
    oracle().kron3(pr.op_a.value, pr.op_b.value, pr.op_c.value, n, n, n, n, n, n, batch, np.float32(pr.alpha), a, n,
                   b, n, c, n, x, n, n * n, E, np.float32(pr.beta), out, n, n * n, E)
    return out


def check(got, want, batch, tol=1e-5):
    worst = max(rel_err_inf(got[p * E:(p + 1) * E], want[p * E:(p + 1) * E]) for p in range(batch))
    assert worst < tol, worst
    return worst


@pytest.mark.parametrize("batch", [1, 5, 444, 1001])
def test_tc_generated_within_tolerance(batch):
    a, b, c, x, y = oracle().generate_batch(np.float32, 1, n, True, batch)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    got = run_tc(pr, a, b, c, x, y, batch)
    assert kb.last_path() == "kron3_tc"
    w = check(got, oracle3(pr, a, b, c, x, y, batch), batch)
    assert w < 5e-6  # 3xTF32 keeps a 2x margin under the fp32 contract


def test_tc_identity_exact_and_ops_alpha_beta():
    g = rng(5)
    batch = 37
    eye = np.eye(n, dtype=np.float32).ravel(order="F")
    x = uniform(g, E * batch, np.float32)
    y = np.full(E * batch, np.nan, np.float32)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    got = run_tc(pr, eye, eye, eye, x, y, batch)
    assert np.max(np.abs(got - x)) <= 2.0 ** -22 * np.max(np.abs(x)) * 4
    for op_a, op_b, op_c in ((T_, N_, N_), (N_, T_, T_), (T_, T_, T_)):
        for alpha, beta in ((0.75, 1.25), (1.0, 1.0), (-2.0, 0.0)):
            a, b, c = (uniform(g, n * n, np.float32) for _ in range(3))
            y = uniform(g, E * batch, np.float32)
            pr = KronProblem3D(op_a, op_b, op_c, n, n, n, n, n, n, alpha, beta)
            check(run_tc(pr, a, b, c, x, y, batch), oracle3(pr, a, b, c, x, y, batch), batch)


def test_tc_padded_strides_and_untouched_padding():
    g = rng(9)
    batch = 23
    a, b, c = (uniform(g, n * n, np.float32) for _ in range(3))
    x = uniform(g, E * batch, np.float32)
    y0 = uniform(g, E * batch, np.float32)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n, alpha=0.5, beta=2.0)
    want = oracle3(pr, a, b, c, x, y0, batch)
    sx, ldy, ldy2 = E + 64, n + 3, (n + 3) * n + 5
    sy = ldy2 * n + 7
    xp = np.full(sx * batch, np.nan, np.float32)
    yp = np.full(sy * batch, 321.0, np.float32)
    for p in range(batch):
        xp[p * sx:p * sx + E] = x[p * E:(p + 1) * E]
        for k in range(n):
            for j in range(n):
                o = p * sy + k * ldy2 + j * ldy
                yp[o:o + n] = y0[p * E + k * n * n + j * n:p * E + k * n * n + (j + 1) * n]
    got = run_tc(pr, a, b, c, xp, yp, batch, sx=sx, sy=sy, ldy=ldy, ldy2=ldy2)
    assert kb.last_path() == "kron3_tc"
    mask = np.ones_like(got, bool)
    for p in range(batch):
        blk = np.empty(E, np.float32)
        for k in range(n):
            for j in range(n):
                o = p * sy + k * ldy2 + j * ldy
                blk[k * n * n + j * n:k * n * n + (j + 1) * n] = got[o:o + n]
                mask[o:o + n] = False
        assert rel_err_inf(blk, want[p * E:(p + 1) * E]) < 1e-5
    assert np.all(got[mask] == 321.0)


def test_tc_baseline_config_sampled_oracle():
    """BASELINE config 3 (3-D fp32 n=16, batch 262,144): run_one's sampled
    entries vs the double O(m^6) oracle within 1e-5."""
    import torch

    o = oracle()
    batch = 262144
    a, b, c, x, y = o.generate_batch(np.float32, 1, n, True, batch)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    X, Y = to_dev(x), torch.empty(E * batch, dtype=torch.float32, device="cuda")
    kb.kron3(pr, MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n), MatrixView(to_dev(c), n, n, n),
             BatchView(Array3View(X, n, n, n, n, n * n), batch, E), BatchView(Array3View(Y, n, n, n, n, n * n), batch, E),
             Workspace(None, E * batch), Exec(tf32=True))
    assert kb.last_path() == "kron3_tc"
    got = to_host(Y)
    A, B, Cm = (v.reshape(n, n).T.astype(np.float64) for v in (a, b, c))
    for p in sorted(set(rng(3).integers(0, batch, 8).tolist()) | {0, batch - 1}):
        s = slice(p * E, (p + 1) * E)
        X64 = x[s].reshape(n, n, n).transpose(2, 1, 0).astype(np.float64)
        assert rel_err_inf(got[s], o.ref_kron3_apply(A, B, Cm, X64).ravel(order="F")) < 1e-5
