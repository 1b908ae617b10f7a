"""Pins the C oracle (oracle/kron_oracle.c) against the reference (CPU only).

1. Against the committed golden fixtures tests/golden/kron_golden.npz, which
   were produced by the reference itself (tests/golden/make_golden.py):
   generator bit-exactness, reference KATs, and the kron2/kron3 outputs --
   bit-exact under the contraction rule the reference's g++ codegen uses at
   each size (FMA chain, or mul+add at n in {2,4,8}), within 1e-5 / 1e-12
   everywhere.
2. Against the live reference build (oracle/_ref) when present.
"""
import os

import numpy as np
import pytest

from kb_testutil import TOL, fused_sizes, mismatches, oracle, reference, rel_err_inf

GOLD = os.path.join(os.path.dirname(__file__), "golden", "kron_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_kats(gold):
    o = oracle()
    assert np.array_equal(gold["kat_kron_matrix"], [[1, 0, 2, 0], [0, 1, 0, 2], [3, 0, 4, 0], [0, 3, 0, 4]])
    assert np.array_equal(o.kron_matrix(np.array([[1.0, 2.0], [3.0, 4.0]]), np.eye(2)), gold["kat_kron_matrix"])
    assert gold["kat_all_ones"][0] == 10.0
    y = np.array([-1.0])
    o.kron2("N", "N", "N", 1, 2, 1, 2, 1, 1.0, np.ones(2), 1, np.ones(2), 1, np.array([1.0, 3.0, 2.0, 4.0]), 2, 4, 0.0,
            y, 1, 1)
    assert y[0] == 10.0
    assert list(gold["kat_flops"]) == [4000, 393216, 4, 6]
    assert [o.flops_kron(10, False), o.flops_kron(16, True), o.flops_kron(1, False), o.flops_kron(1, True)] == \
        list(gold["kat_flops"])
    assert int(gold["kat_problem_bytes"][0]) == 3 * 1638400000 + 3072 == o.problem_bytes(16, True, False, 100000)
    assert list(gold["kat_workspace"]) == [640, 0, 0, 409600000]
    assert [o.kron3_workspace_size(4, 8, 20, 1), o.kron3_workspace_size(0, 8, 20, 5),
            o.kron3_workspace_size(4, 8, 20, 0), o.kron3_workspace_size(100, 64, 64, 1000)] == [640, 0, 0, 409600000]
    with pytest.raises(OverflowError):
        o.kron3_workspace_size(1 << 31, 1 << 31, 4, 1)


@pytest.mark.parametrize("dtype,tag", [(np.float32, "f32"), (np.float64, "f64")])
@pytest.mark.parametrize("dims3", [False, True])
def test_generator_and_square_outputs(gold, dtype, tag, dims3):
    o = oracle()
    for n in range(1, 17):
        key = f"gen_{tag}_{'3d' if dims3 else '2d'}_{n}"
        a, b, c, x, y0 = o.generate_batch(dtype, 1, n, dims3, 3)
        assert mismatches(a, gold[key + "_a"]) == 0 and mismatches(b, gold[key + "_b"]) == 0
        assert mismatches(x, gold[key + "_x"]) == 0 and mismatches(y0, gold[key + "_y0"]) == 0
        if dims3:
            assert mismatches(c, gold[key + "_c"]) == 0
        want = gold[key + "_y"]
        for fused in (True, False):
            o.set_fused(fused)
            y = y0.copy()
            if dims3:
                o.kron3("N", "N", "N", n, n, n, n, n, n, 3, dtype(1), a, n, b, n, c, n, x, n, n * n, n ** 3, dtype(0), y,
                        n, n * n, n ** 3)
            else:
                o.kron2("N", "N", "N", n, n, n, n, 3, dtype(1), a, n, b, n, x, n, n * n, dtype(0), y, n, n * n)
            o.set_fused(True)
            e = n ** (3 if dims3 else 2)
            for p in range(3):
                assert rel_err_inf(y[p * e:(p + 1) * e], want[p * e:(p + 1) * e]) < TOL[np.dtype(dtype)]
            expect_bitwise = (n in fused_sizes(dtype)) if fused else (n in ({2, 4, 8} if dtype == np.float32 else {2, 4}))
            if expect_bitwise:
                assert mismatches(y, want) == 0, (n, fused)


@pytest.mark.parametrize("dtype,tag", [(np.float32, "f32"), (np.float64, "f64")])
def test_rectangular_padded_op_combos(gold, dtype, tag):
    """Rectangular shapes with padded ld / strides, every op, alpha .75 beta 1.25:
    the oracle reproduces the reference within tolerance, and never writes padding."""
    o = oracle()
    for oa in "NT":
        for ob in "NT":
            for ox in "NT":
                key = f"rect2_{tag}_{oa}{ob}{ox}"
                m_a, n_a, m_b, n_b, batch, lda, ldb, ldx, sx, ldy, sy = (int(v) for v in gold[key + "_dims"])
                y = gold[key + "_y0"].copy()
                o.kron2(oa, ob, ox, m_a, n_a, m_b, n_b, batch, dtype(0.75), gold[key + "_a"], lda, gold[key + "_b"],
                        ldb, gold[key + "_x"], ldx, sx, dtype(1.25), y, ldy, sy)
                want = gold[key + "_y"]
                assert rel_err_inf(y, want) < TOL[np.dtype(dtype)]
                untouched = gold[key + "_y0"] == want
                assert np.array_equal(y[untouched], want[untouched])
                key = f"rect3_{tag}_{oa}{ob}{ox}"
                m_a, n_a, m_b, n_b, m_c, n_c, batch, ldx, ldx2, sx, ldy, ldy2, sy = (int(v) for v in gold[key + "_dims"])
                ar = n_a if oa == "T" else m_a
                br = n_b if ob == "T" else m_b
                cr = n_c if ox == "T" else m_c
                y = gold[key + "_y0"].copy()
                o.kron3(oa, ob, ox, m_a, n_a, m_b, n_b, m_c, n_c, batch, dtype(0.75), gold[key + "_a"], ar,
                        gold[key + "_b"], br, gold[key + "_c"], cr, gold[key + "_x"], ldx, ldx2, sx, dtype(1.25), y,
                        ldy, ldy2, sy)
                assert rel_err_inf(y, gold[key + "_y"]) < TOL[np.dtype(dtype)]


def test_brute_force_oracle_identities():
    """test_reference.cpp:160-232: the literal sums equal the explicit Kronecker
    matrix applied to vec(X)."""
    o = oracle()
    g = np.random.default_rng(5)
    A, B, X = g.random((3, 4)), g.random((2, 5)), g.random((4, 5))
    Y = o.ref_kron2_apply(A, B, X)
    K = o.kron_matrix(B, A)
    assert np.allclose(Y.ravel(order="F"), K @ X.ravel(order="F"), rtol=0, atol=1e-12)
    Cm, X3 = g.random((3, 2)), g.random((4, 5, 2))
    Y3 = o.ref_kron3_apply(A, B, Cm, X3)
    K3 = o.kron_matrix(Cm, o.kron_matrix(B, A))
    assert np.allclose(Y3.ravel(order="F"), K3 @ X3.ravel(order="F"), rtol=0, atol=1e-12)


def test_live_reference_matches_oracle():
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    o = oracle()
    for n in (3, 9, 16):
        a, b, _, x, y = ref.generate_batch(np.float32, 42, n, False, 50)
        yr, yo = y.copy(), y.copy()
        ref.kron2("T", "N", "T", n, n, n, n, 50, np.float32(-0.5), a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n,
                  np.float32(2.0), yr, (n, n), n, n * n)
        o.kron2("T", "N", "T", n, n, n, n, 50, np.float32(-0.5), a, n, b, n, x, n, n * n, np.float32(2.0), yo, n, n * n)
        assert rel_err_inf(yo, yr) < 1e-5
        if n in fused_sizes(np.float32):
            assert mismatches(yo, yr) == 0
