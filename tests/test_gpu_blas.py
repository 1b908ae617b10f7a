"""GPU parity for kron1 / gemm_a through the C ABI (-m gpu): the properties of
proj/tests/test_kron1.cpp and test_gemm_a.cpp re-expressed as sm_100a vs
oracle checks -- bit-exact against the FMA-chain restatement, the reference
within 1e-5 / 1e-12, op combinations, alpha/beta paths, NaN with beta = 0,
alpha = 0 never reading A / X / B, zero dims, padded strides (padding
untouched), host-staged buffers, batch independence."""
import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from kb_testutil import TOL, mismatches, oracle, reference, rel_err_inf, rng, to_dev, to_host, uniform

pytestmark = pytest.mark.gpu
MV, BV, VV = kb.MatrixView, kb.BatchView, kb.VectorView


def run_kron1(opa, m, n_a, alpha, A, lda, X, sx, batch, beta, Y, sy, host=False):
    Ad, Xd, Yd = (A.copy(), X.copy(), Y.copy()) if host else (to_dev(A), to_dev(X), to_dev(Y))
    ash = (m, n_a) if opa == "N" else (n_a, m)
    kb.kron1(opa, m, n_a, alpha, MV(Ad, ash[0], ash[1], lda), BV(VV(Xd, n_a), batch, sx), beta,
             BV(VV(Yd, m), batch, sy))
    return Yd if host else to_host(Yd)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m, n_a", [(1, 1), (3, 5), (10, 10), (16, 16), (17, 9), (64, 48)])
@pytest.mark.parametrize("opa", ["N", "T"])
@pytest.mark.parametrize("alpha, beta", [(1.0, 0.0), (0.75, 1.25), (-1.5, 1.0)])
def test_kron1_bitwise_vs_oracle(dtype, m, n_a, opa, alpha, beta):
    g = rng(7 * m + n_a)
    batch = 301
    ash = (m, n_a) if opa == "N" else (n_a, m)
    A = uniform(g, ash[0] * ash[1], dtype)
    X = uniform(g, n_a * batch, dtype)
    Y = uniform(g, m * batch, dtype)
    got = run_kron1(opa, m, n_a, dtype(alpha), A, ash[0], X, n_a, batch, dtype(beta), Y, m)
    want = Y.copy()
    oracle().kron1(opa, m, n_a, batch, dtype(alpha), A, ash[0], X, n_a, dtype(beta), want, m)
    assert kb.last_path() == "kron1"
    assert mismatches(got, want) == 0
    ref = reference()
    if ref is not None:
        yr = Y.copy()
        ref.kron1(opa, m, n_a, dtype(alpha), A, ash, ash[0], X, n_a, n_a, batch, dtype(beta), yr, m, m)
        assert rel_err_inf(got, yr) < TOL[np.dtype(dtype)]


def test_kron1_identity_padding_nan_alpha0_host():
    g = rng(3)
    m, batch, sx, sy = 6, 50, 9, 8
    A = np.eye(m)
    X = uniform(g, sx * batch, np.float64)
    Y = np.full(sy * batch, np.nan)
    got = run_kron1("N", m, m, 1.0, A.ravel(order="F"), m, X, sx, batch, 0.0, Y, sy)
    for p in range(batch):
        assert np.array_equal(got[p * sy:p * sy + m], X[p * sx:p * sx + m])  # identity, NaN prior ignored
        assert np.isnan(got[p * sy + m:(p + 1) * sy]).all()  # padding untouched
    # alpha = 0: Y <- beta*Y, A / X never read (NaN there)
    Y2 = uniform(g, m * batch, np.float64)
    got2 = run_kron1("N", m, m, 0.0, np.full(m * m, np.nan), m, np.full(m * batch, np.nan), m, batch, 2.0, Y2, m)
    assert np.array_equal(got2, 2.0 * Y2)
    # host-staged buffers: same bits as device-resident
    X3, Y3 = uniform(g, m * batch, np.float32), uniform(g, m * batch, np.float32)
    A3 = uniform(g, m * m, np.float32)
    a = run_kron1("T", m, m, np.float32(0.5), A3, m, X3, m, batch, np.float32(-1.0), Y3, m)
    b = run_kron1("T", m, m, np.float32(0.5), A3, m, X3, m, batch, np.float32(-1.0), Y3, m, host=True)
    assert mismatches(a, b) == 0


def run_gemm_a(opa, opb, m, n, k, alpha, A, lda, sa, batch, B, ldb, beta, Cm, ldc, sc, host=False):
    Ad, Bd, Cd = (A.copy(), B.copy(), Cm.copy()) if host else (to_dev(A), to_dev(B), to_dev(Cm))
    ash = (m, k) if opa == "N" else (k, m)
    bsh = (k, n) if opb == "N" else (n, k)
    kb.gemm_a(opa, opb, m, n, k, alpha, BV(MV(Ad, ash[0], ash[1], lda), batch, sa), MV(Bd, bsh[0], bsh[1], ldb), beta,
              BV(MV(Cd, m, n, ldc), batch, sc))
    return Cd if host else to_host(Cd)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m, n, k", [(1, 1, 1), (4, 3, 5), (5, 5, 5), (10, 10, 10), (13, 13, 13), (16, 16, 16), (9, 20, 7),
                                     (33, 2, 19)])
@pytest.mark.parametrize("opa, opb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("alpha, beta", [(1.0, 0.0), (0.75, 1.25)])
def test_gemm_a_vs_oracle(dtype, m, n, k, opa, opb, alpha, beta):
    g = rng(m * 131 + n * 17 + k)
    batch = 77
    ash = (m, k) if opa == "N" else (k, m)
    bsh = (k, n) if opb == "N" else (n, k)
    A = uniform(g, ash[0] * ash[1] * batch, dtype)
    B = uniform(g, bsh[0] * bsh[1], dtype)
    Cm = uniform(g, m * n * batch, dtype)
    got = run_gemm_a(opa, opb, m, n, k, dtype(alpha), A, ash[0], ash[0] * ash[1], batch, B, bsh[0], dtype(beta), Cm, m,
                     m * n)
    want = Cm.copy()
    oracle().gemm_a(opa, opb, m, n, k, batch, dtype(alpha), A, ash[0], ash[0] * ash[1], B, bsh[0], dtype(beta), want, m,
                    m * n)
    assert kb.last_path() == "gemm_a"
    assert mismatches(got, want) == 0  # identical arithmetic to the restatement
    ref = reference()
    if ref is not None:
        cr = Cm.copy()
        ref.gemm_a(opa, opb, m, n, k, dtype(alpha), A, ash, ash[0], ash[0] * ash[1], batch, B, bsh, bsh[0],
                   dtype(beta), cr, (m, n), m, m * n)
        e = m * n
        for p in range(0, batch, 7):
            assert rel_err_inf(got[p * e:(p + 1) * e], cr[p * e:(p + 1) * e]) < TOL[np.dtype(dtype)]


def test_gemm_a_padding_nan_alpha0_zero_dims_host():
    g = rng(5)
    m, n, k, batch = 5, 4, 3, 40
    lda, sa, ldc, sc = 7, 7 * k + 2, 6, 6 * n + 3
    A = uniform(g, sa * batch, np.float64)
    B = uniform(g, k * n, np.float64)
    C = np.full(sc * batch, np.nan)
    got = run_gemm_a("N", "N", m, n, k, 1.0, A, lda, sa, batch, B, k, 0.0, C, ldc, sc)
    tight = run_gemm_a("N", "N", m, n, k, 1.0,
                       np.concatenate([A[p * sa:p * sa + lda * k].reshape(k, lda)[:, :m].ravel() for p in range(batch)]),
                       m, m * k, batch, B, k, 0.0, np.zeros(m * n * batch), m, m * n)
    for p in range(batch):
        blk = got[p * sc:p * sc + ldc * n].reshape(n, ldc)
        assert np.array_equal(blk[:, :m].ravel(), tight[p * m * n:(p + 1) * m * n])  # padded == tight, bit for bit
        assert np.isnan(blk[:, m:]).all() and np.isnan(got[p * sc + ldc * n:(p + 1) * sc]).all()
    C2 = uniform(g, m * n * batch, np.float64)
    got2 = run_gemm_a("N", "N", m, n, k, 0.0, np.full(m * k * batch, np.nan), m, m * k, batch, np.full(k * n, np.nan), k,
                      -1.0, C2, m, m * n)
    assert np.array_equal(got2, -C2)
    got3 = run_gemm_a("N", "N", m, n, 0, 2.0, np.zeros(1), m, 0, batch, np.full(n, np.nan), 1, 0.5, C2, m, m * n)
    assert np.array_equal(got3, 0.5 * C2)  # k = 0: empty sum
    # host-staged buffers: same bits as device-resident
    A4, B4, C4 = uniform(g, k * m * batch, np.float32), uniform(g, k * n, np.float32), uniform(g, m * n * batch, np.float32)
    a = run_gemm_a("T", "N", m, n, k, np.float32(1.5), A4, k, k * m, batch, B4, k, np.float32(0.5), C4, m, m * n)
    b = run_gemm_a("T", "N", m, n, k, np.float32(1.5), A4, k, k * m, batch, B4, k, np.float32(0.5), C4, m, m * n,
                   host=True)
    assert mismatches(a, b) == 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [2, 7, 16])
@pytest.mark.parametrize("opa", ["N", "T"])
def test_gemm_a_square_many_tiles(dtype, n, opa):
    """The square n <= 16 kernel over many CTA tiles (grid-stride loop, ragged last tile)."""
    g = rng(n * 7 + (opa == "T"))
    batch = 60_001
    A = uniform(g, n * n * batch, dtype)
    B = uniform(g, n * n, dtype)
    Cm = uniform(g, n * n * batch, dtype)
    got = run_gemm_a(opa, "T", n, n, n, dtype(-0.625), A, n, n * n, batch, B, n, dtype(0.5), Cm, n, n * n)
    want = Cm.copy()
    oracle().gemm_a(opa, "T", n, n, n, batch, dtype(-0.625), A, n, n * n, B, n, dtype(0.5), want, n, n * n)
    assert mismatches(got, want) == 0
