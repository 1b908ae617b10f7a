"""The sm_100a path against golden vectors produced by the REFERENCE itself
(tests/golden/kron_golden.npz, made by tests/golden/make_golden.py from the
unmodified reference build) -- no oracle in the loop (-m gpu).

* square n = 1..16, fp32/fp64, 2-D and 3-D, generate_batch seed 1 (3 entries):
  within 1e-5 / 1e-12 everywhere, and BIT-identical wherever the reference's
  g++ code is an FMA chain (fp32 n in {1, 5-7, 9-16}, fp64
  n in {1, 5-16});
* rectangular shapes with padded ld / batch strides, all 8 op combinations,
  alpha .75 beta 1.25: within tolerance, and Y padding untouched
  (test_kron2.cpp:249-256, test_kron3.cpp:316-324);
* the KATs: all-ones -> 10 (test_kron2.cpp:59-67).
"""
import os

import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from kb_testutil import TOL, fused_sizes, mismatches, rel_err_inf, to_dev, to_host

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "kron_golden.npz")
MV, BV, A3 = kb.MatrixView, kb.BatchView, kb.Array3View


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("dtype,tag", [(np.float32, "f32"), (np.float64, "f64")])
@pytest.mark.parametrize("dims3", [False, True])
def test_square_generated_vs_reference_outputs(gold, dtype, tag, dims3):
    for n in range(1, 17):
        key = f"gen_{tag}_{'3d' if dims3 else '2d'}_{n}"
        a, b, x, y0, want = (gold[key + s] for s in ("_a", "_b", "_x", "_y0", "_y"))
        e = n ** (3 if dims3 else 2)
        Y = to_dev(y0)
        if dims3:
            pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
            kb.kron3(pr, MV(to_dev(a), n, n, n), MV(to_dev(b), n, n, n), MV(to_dev(gold[key + "_c"]), n, n, n),
                     BV(A3(to_dev(x), n, n, n, n, n * n), 3, e), BV(A3(Y, n, n, n, n, n * n), 3, e),
                     kb.Workspace(None, e * 3))
        else:
            pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
            kb.kron2(pr, MV(to_dev(a), n, n, n), MV(to_dev(b), n, n, n), BV(MV(to_dev(x), n, n, n), 3, e),
                     BV(MV(Y, n, n, n), 3, e))
        got = to_host(Y)
        for p in range(3):
            assert rel_err_inf(got[p * e:(p + 1) * e], want[p * e:(p + 1) * e]) < TOL[np.dtype(dtype)], (n, p)
        if n in fused_sizes(dtype):
            assert mismatches(got, want) == 0, n


@pytest.mark.parametrize("dtype,tag", [(np.float32, "f32"), (np.float64, "f64")])
def test_rectangular_padded_op_combos_vs_reference(gold, dtype, tag):
    for oa in "NT":
        for ob in "NT":
            for ox in "NT":
                key = f"rect2_{tag}_{oa}{ob}{ox}"
                m_a, n_a, m_b, n_b, batch, lda, ldb, ldx, sx, ldy, sy = (int(v) for v in gold[key + "_dims"])
                y0, want = gold[key + "_y0"], gold[key + "_y"]
                ar, ac = (n_a, m_a) if oa == "T" else (m_a, n_a)
                br, bc = (n_b, m_b) if ob == "T" else (m_b, n_b)
                xr, xc = (n_b, n_a) if ox == "T" else (n_a, n_b)
                Y = to_dev(y0)
                pr = kb.KronProblem2D(op_a=oa, op_b=ob, op_x=ox, m_a=m_a, n_a=n_a, m_b=m_b, n_b=n_b, alpha=0.75,
                                      beta=1.25)
                kb.kron2(pr, MV(to_dev(gold[key + "_a"]), ar, ac, lda), MV(to_dev(gold[key + "_b"]), br, bc, ldb),
                         BV(MV(to_dev(gold[key + "_x"]), xr, xc, ldx), batch, sx), BV(MV(Y, m_a, m_b, ldy), batch, sy))
                got = to_host(Y)
                assert rel_err_inf(got, want) < TOL[np.dtype(dtype)], key
                untouched = y0 == want  # padding (and any unchanged entries) keep their bits
                assert np.array_equal(got[untouched], want[untouched]), key

                key = f"rect3_{tag}_{oa}{ob}{ox}"
                m_a, n_a, m_b, n_b, m_c, n_c, batch, ldx, ldx2, sx, ldy, ldy2, sy = (int(v) for v in gold[key + "_dims"])
                y0, want = gold[key + "_y0"], gold[key + "_y"]
                ar, ac = (n_a, m_a) if oa == "T" else (m_a, n_a)
                br, bc = (n_b, m_b) if ob == "T" else (m_b, n_b)
                cr, cc = (n_c, m_c) if ox == "T" else (m_c, n_c)
                Y = to_dev(y0)
                pr = kb.KronProblem3D(op_a=oa, op_b=ob, op_c=ox, m_a=m_a, n_a=n_a, m_b=m_b, n_b=n_b, m_c=m_c, n_c=n_c,
                                      alpha=0.75, beta=1.25)
                kb.kron3(pr, MV(to_dev(gold[key + "_a"]), ar, ac, ar), MV(to_dev(gold[key + "_b"]), br, bc, br),
                         MV(to_dev(gold[key + "_c"]), cr, cc, cr),
                         BV(A3(to_dev(gold[key + "_x"]), n_a, n_b, n_c, ldx, ldx2), batch, sx),
                         BV(A3(Y, m_a, m_b, m_c, ldy, ldy2), batch, sy), kb.Workspace(None, m_a * m_b * n_c * batch))
                got = to_host(Y)
                assert rel_err_inf(got, want) < TOL[np.dtype(dtype)], key
                untouched = y0 == want
                assert np.array_equal(got[untouched], want[untouched]), key


def test_all_ones_kat():
    """kron2 with 1x2 all-ones operators on X = [[1,2],[3,4]] -> 10 (test_kron2.cpp:59-67)."""
    Y = to_dev(np.array([-1.0]))
    pr = kb.KronProblem2D(m_a=1, n_a=2, m_b=1, n_b=2)
    kb.kron2(pr, MV(np.ones(2), 1, 2, 1), MV(np.ones(2), 1, 2, 1), BV(MV(to_dev(np.array([1.0, 3.0, 2.0, 4.0])), 2, 2, 2), 1, 4),
             BV(MV(Y, 1, 1, 1), 1, 1))
    assert to_host(Y)[0] == 10.0
