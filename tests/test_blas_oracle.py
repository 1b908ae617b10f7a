"""kron1 / gemm_a oracle (oracle/kron_oracle.c) pinned against the compiled
reference (oracle/_ref: proj/include/kronbatch/kron1.hpp, gemm_a.hpp), and the
Python API's validation messages against the reference's -- CPU only.

Contraction pattern of the reference build (g++ -O3 -march=native), probed
here: kron1 and gemm_a(op_a = N) are strict FMA chains for m >= 9 (fp32) /
m >= 8 (fp64) -- the generic m > 16 loop included -- and unfused or mixed at
some smaller m; gemm_a(op_a = T) (gemm_dot) matches neither chain exactly
(the compiler re-forms the final alpha*acc + beta*C), so it is pinned to the
1e-5 / 1e-12 tolerance everywhere."""
import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from kb_testutil import TOL, mismatches, oracle, reference, rel_err_inf, rng, uniform

REF = reference()
needs_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built (needs /root/reference)")


def fused_rows(dtype, m):
    return m >= (9 if np.dtype(dtype) == np.float32 else 8)


@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m, n_a", [(1, 3), (4, 4), (9, 12), (16, 16), (17, 5), (33, 40)])
@pytest.mark.parametrize("opa", ["N", "T"])
@pytest.mark.parametrize("alpha, beta", [(1.0, 0.0), (0.75, 1.25), (-2.0, 1.0)])
def test_kron1_oracle_vs_reference(dtype, m, n_a, opa, alpha, beta):
    g = rng(m * 100 + n_a)
    batch = 13
    ash = (m, n_a) if opa == "N" else (n_a, m)
    A = uniform(g, ash[0] * ash[1], dtype)
    X = uniform(g, n_a * batch, dtype)
    Y0 = uniform(g, m * batch, dtype)
    yo, yr = Y0.copy(), Y0.copy()
    oracle().kron1(opa, m, n_a, batch, dtype(alpha), A, ash[0], X, n_a, dtype(beta), yo, m)
    REF.kron1(opa, m, n_a, dtype(alpha), A, ash, ash[0], X, n_a, n_a, batch, dtype(beta), yr, m, m)
    for p in range(batch):
        assert rel_err_inf(yo[p * m:(p + 1) * m], yr[p * m:(p + 1) * m]) < TOL[np.dtype(dtype)]
    if fused_rows(dtype, m):
        assert mismatches(yo, yr) == 0


@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m, n, k", [(1, 1, 1), (3, 5, 4), (9, 4, 7), (16, 16, 16), (20, 3, 11)])
@pytest.mark.parametrize("opa, opb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_gemm_a_oracle_vs_reference(dtype, m, n, k, opa, opb):
    g = rng(m * 1000 + n * 10 + k)
    batch = 9
    ash = (m, k) if opa == "N" else (k, m)
    bsh = (k, n) if opb == "N" else (n, k)
    A = uniform(g, ash[0] * ash[1] * batch, dtype)
    B = uniform(g, bsh[0] * bsh[1], dtype)
    C0 = uniform(g, m * n * batch, dtype)
    co, cr = C0.copy(), C0.copy()
    oracle().gemm_a(opa, opb, m, n, k, batch, dtype(0.75), A, ash[0], ash[0] * ash[1], B, bsh[0], dtype(1.25), co, m,
                    m * n)
    REF.gemm_a(opa, opb, m, n, k, dtype(0.75), A, ash, ash[0], ash[0] * ash[1], batch, B, bsh, bsh[0], dtype(1.25), cr,
               (m, n), m, m * n)
    e = m * n
    for p in range(batch):
        assert rel_err_inf(co[p * e:(p + 1) * e], cr[p * e:(p + 1) * e]) < TOL[np.dtype(dtype)]
    if opa == "N" and fused_rows(dtype, m):
        assert mismatches(co, cr) == 0


@needs_ref
def test_kron1_known_answers():
    """test_kron1.cpp:49-63: identity passthrough and a direct 2x2 matvec."""
    for opa in "NT":
        A = np.array([1.0, 3.0, 2.0, 4.0])  # [[1, 2], [3, 4]] column-major
        X = np.array([1.0, 1.0])
        Y = np.zeros(2)
        REF.kron1(opa, 2, 2, 1.0, A, (2, 2), 2, X, 2, 2, 1, 0.0, Y, 2, 2)
        Yo = np.zeros(2)
        oracle().kron1(opa, 2, 2, 1, 1.0, A, 2, X, 2, 0.0, Yo, 2)
        assert list(Yo) == list(Y) == ([3.0, 7.0] if opa == "N" else [4.0, 6.0])


def _ref_error(fn):
    try:
        fn()
    except ValueError as e:
        return str(e)
    return None


@needs_ref
def test_kron1_validation_messages_match_reference():
    d = np.zeros(64)
    cases = [  # (python call, reference call)
        (lambda: kb.kron1("N", 2, 2, 1.0, kb.MatrixView(d, 2, 2, 1), kb.BatchView(kb.VectorView(d, 2), 1, 2), 0.0,
                          kb.BatchView(kb.VectorView(d, 2), 1, 2)),
         lambda: REF.kron1("N", 2, 2, 1.0, d, (2, 2), 1, d, 2, 2, 1, 0.0, d, 2, 2)),
        (lambda: kb.kron1("N", 2, 3, 1.0, kb.MatrixView(d, 2, 2, 2), kb.BatchView(kb.VectorView(d, 3), 1, 3), 0.0,
                          kb.BatchView(kb.VectorView(d, 2), 1, 2)),
         lambda: REF.kron1("N", 2, 3, 1.0, d, (2, 2), 2, d, 3, 3, 1, 0.0, d, 2, 2)),
        (lambda: kb.kron1("N", 2, 2, 1.0, kb.MatrixView(d, 2, 2, 2), kb.BatchView(kb.VectorView(d, 3), 1, 3), 0.0,
                          kb.BatchView(kb.VectorView(d, 2), 1, 2)),
         lambda: REF.kron1("N", 2, 2, 1.0, d, (2, 2), 2, d, 3, 3, 1, 0.0, d, 2, 2)),
        (lambda: kb.kron1("N", 2, 2, 1.0, kb.MatrixView(d, 2, 2, 2), kb.BatchView(kb.VectorView(d, 2), 2, 2), 0.0,
                          kb.BatchView(kb.VectorView(d, 2), 3, 2)),
         lambda: REF.kron1("N", 2, 2, 1.0, d, (2, 2), 2, d, 2, 2, 2, 0.0, d, 2, 2, lens=None)),
        (lambda: kb.kron1("N", 2, 2, 1.0, kb.MatrixView(d, 2, 2, 2), kb.BatchView(kb.VectorView(d, 2), 2, 1), 0.0,
                          kb.BatchView(kb.VectorView(d, 2), 2, 2)),
         lambda: REF.kron1("N", 2, 2, 1.0, d, (2, 2), 2, d, 2, 1, 2, 0.0, d, 2, 2)),
    ]
    for py, ref in cases[:3] + cases[4:]:
        want = _ref_error(ref)
        assert want is not None
        with pytest.raises(ValueError) as ei:
            py()
        assert str(ei.value) == want


@needs_ref
def test_gemm_a_validation_messages_match_reference():
    d = np.zeros(256)
    MV, BV = kb.MatrixView, kb.BatchView
    cases = [
        (lambda: kb.gemm_a("N", "N", 2, 2, 2, 1.0, BV(MV(d, 2, 2, 1), 1, 4), MV(d, 2, 2, 2), 0.0, BV(MV(d, 2, 2, 2), 1, 4)),
         lambda: REF.gemm_a("N", "N", 2, 2, 2, 1.0, d, (2, 2), 1, 4, 1, d, (2, 2), 2, 0.0, d, (2, 2), 2, 4)),
        (lambda: kb.gemm_a("N", "N", 2, 3, 2, 1.0, BV(MV(d, 2, 2, 2), 1, 4), MV(d, 2, 2, 2), 0.0, BV(MV(d, 2, 3, 2), 1, 6)),
         lambda: REF.gemm_a("N", "N", 2, 3, 2, 1.0, d, (2, 2), 2, 4, 1, d, (2, 2), 2, 0.0, d, (2, 3), 2, 6)),
        (lambda: kb.gemm_a("T", "N", 3, 2, 2, 1.0, BV(MV(d, 3, 2, 3), 1, 6), MV(d, 2, 2, 2), 0.0, BV(MV(d, 3, 2, 3), 1, 6)),
         lambda: REF.gemm_a("T", "N", 3, 2, 2, 1.0, d, (3, 2), 3, 6, 1, d, (2, 2), 2, 0.0, d, (3, 2), 3, 6)),
        (lambda: kb.gemm_a("N", "N", 2, 2, 2, 1.0, BV(MV(d, 2, 2, 2), 2, 3), MV(d, 2, 2, 2), 0.0, BV(MV(d, 2, 2, 2), 2, 4)),
         lambda: REF.gemm_a("N", "N", 2, 2, 2, 1.0, d, (2, 2), 2, 3, 2, d, (2, 2), 2, 0.0, d, (2, 2), 2, 4)),
    ]
    for py, ref in cases:
        want = _ref_error(ref)
        assert want is not None
        with pytest.raises(ValueError) as ei:
            py()
        assert str(ei.value) == want
