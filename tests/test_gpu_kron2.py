"""GPU parity tests for kron2 through the C ABI (-m gpu).

Mirrors the properties the reference pins in proj/tests/test_kron2.cpp and
acceptance.cpp (C1/C2/C5), re-expressed as sm_100a-vs-oracle checks:
  * bit-exact equality with the oracle's FMA-chain restatement (the
    Appendix-A contraction order), every size / op / alpha / beta;
  * the reference itself (oracle/_ref) within 1e-5 / 1e-12 rel_err_inf, and
    bit-exact at the sizes where its g++ codegen is an FMA chain;
  * KATs, NaN safety, padding untouched, transpose consistency, host-buffer
    staging, determinism across batch splits.
"""
import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from paper_1304_7054_b200 import BatchView, KronProblem2D, MatrixOp, MatrixView

from kb_testutil import (TOL, bits, fused_sizes, ints, mismatches, oracle, reference, rel_err_inf, rng, to_dev,
                         to_host, uniform)

pytestmark = pytest.mark.gpu
N_, T_ = MatrixOp.NoTranspose, MatrixOp.Transpose


def stored(op, r, c):
    return (c, r) if op != N_ else (r, c)


def run(pr, a, a_shape, lda, b, b_shape, ldb, x, x_shape, ldx, sx, y, ldy, sy, batch, host=False, exec_=None):
    """Run kb.kron2 on copies of the numpy buffers; returns the new Y (numpy)."""
    if host:
        A, B, X, Y = a.copy(), b.copy(), x.copy(), y.copy()
    else:
        A, B, X, Y = to_dev(a), to_dev(b), to_dev(x), to_dev(y)
    kb.kron2(pr, MatrixView(A, *a_shape, lda), MatrixView(B, *b_shape, ldb),
             BatchView(MatrixView(X, *x_shape, ldx), batch, sx), BatchView(MatrixView(Y, pr.m_a, pr.m_b, ldy), batch, sy),
             exec_)
    return Y if host else to_host(Y)


def run_oracle(pr, a, lda, b, ldb, x, ldx, sx, y, ldy, sy, batch, fused=True):
    o = oracle()
    o.set_fused(fused)
    out = y.copy()
    o.kron2(pr.op_a.value, pr.op_b.value, pr.op_x.value, pr.m_a, pr.n_a, pr.m_b, pr.n_b, batch, y.dtype.type(pr.alpha),
            a, lda, b, ldb, x, ldx, sx, y.dtype.type(pr.beta), out, ldy, sy)
    o.set_fused(True)
    return out


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", list(range(1, 17)))
def test_square_generated_bitwise(dtype, n):
    """generate_batch inputs (bench_support.hpp:148-170), alpha 1 beta 0, every
    n <= 16: GPU fast path == oracle bit for bit; == reference within tol."""
    batch = 1000 + n  # ragged last group
    a, b, _, x, y = oracle().generate_batch(dtype, 1, n, False, batch)
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    got = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
    assert kb.last_path() == "kron2_fast"
    want = run_oracle(pr, a, n, b, n, x, n, n * n, y, n, n * n, batch)
    assert mismatches(got, want) == 0
    ref = reference()
    if ref is not None:
        yr = y.copy()
        ref.kron2("N", "N", "N", n, n, n, n, batch, dtype(1), a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n,
                  dtype(0), yr, (n, n), n, n * n)
        for p in range(0, batch, 97):
            s = slice(p * n * n, (p + 1) * n * n)
            assert rel_err_inf(got[s], yr[s]) < TOL[np.dtype(dtype)]
        if n in fused_sizes(dtype):
            assert mismatches(got, yr) == 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [4, 7, 10, 16])
def test_square_ops_alpha_beta_bitwise(dtype, n):
    """All 8 op combinations at square n with alpha .75 / beta 1.25 (fast path,
    op_x both ways) and beta -> 0 / 1 special cases."""
    g = rng(100 + n)
    batch = 257
    for op_a in (N_, T_):
        for op_b in (N_, T_):
            for op_x in (N_, T_):
                for alpha, beta in ((0.75, 1.25), (1.0, 1.0), (-2.0, 0.0)):
                    a, b = uniform(g, n * n, dtype), uniform(g, n * n, dtype)
                    x, y = uniform(g, n * n * batch, dtype), uniform(g, n * n * batch, dtype)
                    pr = KronProblem2D(op_a, op_b, op_x, n, n, n, n, alpha, beta)
                    got = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
                    assert kb.last_path() == "kron2_fast"
                    want = run_oracle(pr, a, n, b, n, x, n, n * n, y, n, n * n, batch)
                    assert mismatches(got, want) == 0, (op_a, op_b, op_x, alpha, beta)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_rectangular_op_combinations(dtype):
    """test_kron2.cpp:96-140: m_a=3, n_a=5, m_b=4, n_b=2, batch 16, alpha .75,
    beta 1.25, all op combos, vs the double oracle (ref_kron2_apply) and bitwise
    vs the restated CPU path (generic kernel)."""
    o = oracle()
    g = rng(227)
    m_a, n_a, m_b, n_b, batch = 3, 5, 4, 2, 16
    for op_a in (N_, T_):
        for op_b in (N_, T_):
            for op_x in (N_, T_):
                ar, ac = stored(op_a, m_a, n_a)
                br, bc = stored(op_b, m_b, n_b)
                xr, xc = stored(op_x, n_a, n_b)
                a, b = uniform(g, ar * ac, dtype), uniform(g, br * bc, dtype)
                x, y0 = uniform(g, xr * xc * batch, dtype), uniform(g, m_a * m_b * batch, dtype)
                pr = KronProblem2D(op_a, op_b, op_x, m_a, n_a, m_b, n_b, 0.75, 1.25)
                got = run(pr, a, (ar, ac), ar, b, (br, bc), br, x, (xr, xc), xr, xr * xc, y0, m_a, m_a * m_b, batch)
                want = run_oracle(pr, a, ar, b, br, x, xr, xr * xc, y0, m_a, m_a * m_b, batch)
                assert mismatches(got, want) == 0
                A = a.reshape(ac, ar).T.astype(np.float64)
                B = b.reshape(bc, br).T.astype(np.float64)
                A = A.T if op_a != N_ else A
                B = B.T if op_b != N_ else B
                for p in range(batch):
                    X = x[p * xr * xc:(p + 1) * xr * xc].reshape(xc, xr).T.astype(np.float64)
                    X = X.T if op_x != N_ else X
                    w = o.ref_kron2_apply(A, B, X).ravel(order="F")
                    w = 0.75 * w + 1.25 * y0[p * m_a * m_b:(p + 1) * m_a * m_b]
                    assert rel_err_inf(got[p * m_a * m_b:(p + 1) * m_a * m_b], w) < TOL[np.dtype(dtype)]


def test_identity_passthrough():
    """test_kron2.cpp:43-57."""
    for dtype in (np.float32, np.float64):
        g = rng(211)
        m, batch = 3, 5
        eye = np.eye(m, dtype=dtype).ravel(order="F")
        x = uniform(g, m * m * batch, dtype)
        y = np.full(m * m * batch, -1, dtype)
        pr = KronProblem2D(m_a=m, n_a=m, m_b=m, n_b=m)
        got = run(pr, eye, (m, m), m, eye, (m, m), m, x, (m, m), m, m * m, y, m, m * m, batch)
        assert np.array_equal(got, x)


def test_all_ones_grand_sum():
    """test_kron2.cpp:59-67: 1x2 all-ones A, B on X=[[1,2],[3,4]] -> 10."""
    ones = np.ones(2)
    x = np.array([1.0, 3.0, 2.0, 4.0])
    y = np.array([-1.0])
    pr = KronProblem2D(m_a=1, n_a=2, m_b=1, n_b=2)
    got = run(pr, ones, (1, 2), 1, ones, (1, 2), 1, x, (2, 2), 2, 4, y, 1, 1, 1)
    assert got[0] == 10.0


@pytest.mark.parametrize("n", [2, 3, 16])
def test_integer_case_exact(n):
    """test_kron2.cpp:69-94: integer operands in [-3, 3] are exact in double."""
    o = oracle()
    g = rng(223)
    batch = 6
    a, b = ints(g, n * n, np.float64), ints(g, n * n, np.float64)
    x = ints(g, n * n * batch, np.float64)
    y = np.full(n * n * batch, np.nan)
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    got = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
    A, B = a.reshape(n, n).T, b.reshape(n, n).T
    for p in range(batch):
        X = x[p * n * n:(p + 1) * n * n].reshape(n, n).T
        assert np.array_equal(got[p * n * n:(p + 1) * n * n], o.ref_kron2_apply(A, B, X).ravel(order="F"))


def test_beta_zero_ignores_nan_y():
    """test_kron2.cpp:196-210."""
    for n in (5, 16):
        g = rng(229)
        batch = 33
        a, b = uniform(g, n * n, np.float32), uniform(g, n * n, np.float32)
        x = uniform(g, n * n * batch, np.float32)
        y = np.full(n * n * batch, np.nan, np.float32)
        pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
        got = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
        assert not np.isnan(got).any()


def test_alpha_zero_and_empty_sums_never_read_operands():
    """test_kron2.cpp:353-408: alpha == 0 or n_a == 0 / n_b == 0 -> Y <- beta*Y,
    NaN in A/B/X never read; batch 0 / m == 0 are no-ops."""
    n, batch = 4, 9
    nan = np.full(n * n * batch, np.nan)
    y0 = uniform(rng(1), n * n * batch, np.float64)
    for beta in (0.0, 1.0, 2.5):
        pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n, alpha=0.0, beta=beta)
        got = run(pr, nan[:n * n], (n, n), n, nan[:n * n], (n, n), n, nan, (n, n), n, n * n, y0, n, n * n, batch)
        want = np.zeros_like(y0) if beta == 0 else y0 * beta
        assert np.array_equal(got, want)
    # n_a == 0: X and A are empty
    pr = KronProblem2D(m_a=n, n_a=0, m_b=n, n_b=n, alpha=1.0, beta=0.5)
    got = run(pr, np.zeros(0), (n, 0), n, nan[:n * n], (n, n), n, np.zeros(n * batch), (0, n), 1, n, y0, n, n * n,
              batch)
    assert np.array_equal(got, y0 * 0.5)
    # batch 0 and m_a == 0 are no-ops
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    y = y0.copy()
    got = run(pr, y0[:n * n], (n, n), n, y0[:n * n], (n, n), n, np.zeros(0), (n, n), n, n * n, y, n, n * n, 0)
    assert np.array_equal(got, y0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [3, 10, 16])
def test_padding_bit_identity_and_untouched(dtype, n):
    """test_kron2.cpp:212-257: padded ld / batch strides give bit-identical
    results to tight ones and never write Y padding."""
    g = rng(233 + n)
    batch = 41
    a, b = uniform(g, n * n, dtype), uniform(g, n * n, dtype)
    x, y0 = uniform(g, n * n * batch, dtype), uniform(g, n * n * batch, dtype)
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n, alpha=0.5, beta=-1.5)
    tight = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y0, n, n * n, batch)
    lda, ldb, ldx, ldy = n + 3, n + 5, n + 7, n + 3
    sx, sy = ldx * n + 5, ldy * n + 7
    ap = np.full(lda * n, np.nan, dtype)
    bp = np.full(ldb * n, np.nan, dtype)
    xp = np.full(sx * batch, np.nan, dtype)
    yp = np.full(sy * batch, 12345.0, dtype)
    for j in range(n):
        ap[j * lda:j * lda + n] = a[j * n:(j + 1) * n]
        bp[j * ldb:j * ldb + n] = b[j * n:(j + 1) * n]
    for p in range(batch):
        for j in range(n):
            xp[p * sx + j * ldx:p * sx + j * ldx + n] = x[p * n * n + j * n:p * n * n + (j + 1) * n]
            yp[p * sy + j * ldy:p * sy + j * ldy + n] = y0[p * n * n + j * n:p * n * n + (j + 1) * n]
    for host in (False, True):
        got = run(pr, ap, (n, n), lda, bp, (n, n), ldb, xp, (n, n), ldx, sx, yp, ldy, sy, batch, host=host)
        mask = np.ones_like(got, bool)
        for p in range(batch):
            for j in range(n):
                s = p * sy + j * ldy
                assert mismatches(got[s:s + n], tight[p * n * n + j * n:p * n * n + (j + 1) * n]) == 0
                mask[s:s + n] = False
        assert np.all(got[mask] == 12345.0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_transpose_consistency_bit_identical(dtype):
    """test_kron2.cpp:259-313: storing X^T with op_x = T (and A^T/B^T with
    op T) gives results bit-identical to the untransposed call."""
    n, batch = 16, 77
    g = rng(239)
    a, b = uniform(g, n * n, dtype), uniform(g, n * n, dtype)
    x = uniform(g, n * n * batch, dtype)
    y = np.zeros(n * n * batch, dtype)
    tr = lambda m: m.reshape(-1, n, n).transpose(0, 2, 1).ravel()
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    base = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
    prt = KronProblem2D(T_, T_, T_, n, n, n, n)
    alt = run(prt, tr(a), (n, n), n, tr(b), (n, n), n, tr(x), (n, n), n, n * n, y, n, n * n, batch)
    assert mismatches(base, alt) == 0


def test_host_buffers_staged_equal_device():
    """Pageable numpy and pinned torch host buffers go through the staged
    pipeline (several chunks) and give the same bits as device buffers."""
    import torch

    n, batch = 16, 70000  # > one 64 MiB staging chunk
    a, b, _, x, y = oracle().generate_batch(np.float32, 3, n, False, batch)
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    dev = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
    host = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch, host=True)
    assert mismatches(dev, host) == 0
    X = torch.from_numpy(x).pin_memory()
    Y = torch.zeros(n * n * batch, dtype=torch.float32).pin_memory()
    kb.kron2(pr, MatrixView(torch.from_numpy(a), n, n, n), MatrixView(torch.from_numpy(b), n, n, n),
             BatchView(MatrixView(X, n, n, n), batch, n * n), BatchView(MatrixView(Y, n, n, n), batch, n * n))
    assert mismatches(dev, Y.numpy()) == 0


def test_batch_split_determinism():
    """Worker-count determinism analogue (test_kron2.cpp:462-491): every entry's
    bits are independent of how the batch is split across launches / grids."""
    n, batch = 16, 5000
    a, b, _, x, y = oracle().generate_batch(np.float32, 5, n, False, batch)
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    full = run(pr, a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n, y, n, n * n, batch)
    for lo, hi in ((0, 1), (1, 9), (9, 1234), (1234, 5000)):
        part = run(pr, a, (n, n), n, b, (n, n), n, x[lo * 256:hi * 256], (n, n), n, n * n, y[lo * 256:hi * 256], n,
                   n * n, hi - lo)
        assert mismatches(part, full[lo * 256:hi * 256]) == 0


def test_baseline_config_sampled_oracle():
    """BASELINE config 2 (2-D fp32 n=16, batch 4,194,304) at full size: the
    run_one protocol (bench_support.cpp:219-241) -- 16 sampled entries vs the
    double oracle within 1e-5 -- plus bitwise equality with the restated CPU
    path on those entries."""
    import torch

    o = oracle()
    n, batch = 16, 4194304
    a, b, _, x, y = o.generate_batch(np.float32, 1, n, False, batch)
    pr = KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    X, Y = to_dev(x), torch.empty(n * n * batch, dtype=torch.float32, device="cuda")
    kb.kron2(pr, MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n),
             BatchView(MatrixView(X, n, n, n), batch, n * n), BatchView(MatrixView(Y, n, n, n), batch, n * n))
    got = to_host(Y)
    A, B = a.reshape(n, n).T.astype(np.float64), b.reshape(n, n).T.astype(np.float64)
    picks = sorted(set(rng(7).integers(0, batch, 16).tolist()) | {0, batch - 1})
    for p in picks:
        s = slice(p * 256, (p + 1) * 256)
        X64 = x[s].reshape(n, n).T.astype(np.float64)
        assert rel_err_inf(got[s], o.ref_kron2_apply(A, B, X64).ravel(order="F")) < 1e-5
        yo = np.zeros(256, np.float32)
        o.kron2("N", "N", "N", n, n, n, n, 1, np.float32(1), a, n, b, n, x[s], n, 256, np.float32(0), yo, n, 256)
        assert mismatches(got[s], yo) == 0
