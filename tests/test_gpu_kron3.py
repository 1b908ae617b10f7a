"""GPU parity tests for kron3 through the C ABI (-m gpu).

Properties of proj/tests/test_kron3.cpp and acceptance.cpp C1-C3/C5,
re-expressed as sm_100a-vs-oracle checks (bit-exact vs the FMA-chain
restatement; reference within 1e-5 / 1e-12; KATs; NaN; padding; workspace
contract; determinism).
"""
import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from paper_1304_7054_b200 import Array3View, BatchView, KronProblem3D, MatrixOp, MatrixView, Workspace

from kb_testutil import (TOL, fused_sizes, ints, mismatches, oracle, reference, rel_err_inf, rng, to_dev, to_host,
                         uniform)

pytestmark = pytest.mark.gpu
N_, T_ = MatrixOp.NoTranspose, MatrixOp.Transpose


def stored(op, r, c):
    return (c, r) if op != N_ else (r, c)


def run(pr, a, a_shape, lda, b, b_shape, ldb, c, c_shape, ldc, x, ldx, ldx2, sx, y, ldy, ldy2, sy, batch, host=False,
        work_cap=None):
    if host:
        A, B, Cm, X, Y = a.copy(), b.copy(), c.copy(), x.copy(), y.copy()
    else:
        A, B, Cm, X, Y = to_dev(a), to_dev(b), to_dev(c), to_dev(x), to_dev(y)
    cap = kb.kron3_workspace_size(pr, batch) if work_cap is None else work_cap
    kb.kron3(pr, MatrixView(A, *a_shape, lda), MatrixView(B, *b_shape, ldb), MatrixView(Cm, *c_shape, ldc),
             BatchView(Array3View(X, pr.n_a, pr.n_b, pr.n_c, ldx, ldx2), batch, sx),
             BatchView(Array3View(Y, pr.m_a, pr.m_b, pr.m_c, ldy, ldy2), batch, sy), Workspace(None, cap))
    return Y if host else to_host(Y)


def run_oracle(pr, a, lda, b, ldb, c, ldc, x, ldx, ldx2, sx, y, ldy, ldy2, sy, batch):
    out = y.copy()
    oracle().kron3(pr.op_a.value, pr.op_b.value, pr.op_c.value, pr.m_a, pr.n_a, pr.m_b, pr.n_b, pr.m_c, pr.n_c, batch,
                   y.dtype.type(pr.alpha), a, lda, b, ldb, c, ldc, x, ldx, ldx2, sx, y.dtype.type(pr.beta), out, ldy,
                   ldy2, sy)
    return out


def tight(pr, a, b, c, x, y, batch, **kw):
    n_a, n_b, n_c, m_a, m_b, m_c = pr.n_a, pr.n_b, pr.n_c, pr.m_a, pr.m_b, pr.m_c
    ash, bsh, csh = stored(pr.op_a, m_a, n_a), stored(pr.op_b, m_b, n_b), stored(pr.op_c, m_c, n_c)
    args = (a, ash, max(ash[0], 1), b, bsh, max(bsh[0], 1), c, csh, max(csh[0], 1), x, max(n_a, 1), max(n_a, 1) * n_b,
            n_a * n_b * n_c, y, max(m_a, 1), max(m_a, 1) * m_b, m_a * m_b * m_c, batch)
    return run(pr, *args, **kw), run_oracle(pr, args[0], args[2], args[3], args[5], args[6], args[8], *args[9:])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", list(range(1, 17)))
def test_square_generated_bitwise(dtype, n):
    batch = 67 + n
    a, b, c, x, y = oracle().generate_batch(dtype, 1, n, True, batch)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    got, want = tight(pr, a, b, c, x, y, batch)
    assert kb.last_path() == "kron3_fast"
    assert mismatches(got, want) == 0
    ref = reference()
    if ref is not None:
        yr = y.copy()
        work = np.empty(n ** 3 * batch, dtype)
        ref.kron3("N", "N", "N", n, n, n, n, n, n, batch, dtype(1), a, (n, n), n, b, (n, n), n, c, (n, n), n, x,
                  (n, n, n), n, n * n, n ** 3, dtype(0), yr, (n, n, n), n, n * n, n ** 3, work)
        e = n ** 3
        for p in range(0, batch, 13):
            assert rel_err_inf(got[p * e:(p + 1) * e], yr[p * e:(p + 1) * e]) < TOL[np.dtype(dtype)]
        if n in fused_sizes(dtype):
            assert mismatches(got, yr) == 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(3, 5, 4, 2, 2, 6), (2, 3, 4, 5, 6, 7), (16, 16, 16, 16, 16, 16), (7, 7, 7, 7, 7, 7),
                                   (1, 4, 9, 2, 3, 1)])
def test_op_combinations_alpha_beta(dtype, shape):
    """test_kron3.cpp:136-183 / 185-223: all 8 ops, alpha .75 beta 1.25,
    rectangular (generic kernel) and square (fast kernel)."""
    m_a, n_a, m_b, n_b, m_c, n_c = shape
    g = rng(241)
    batch = 19
    for op_a in (N_, T_):
        for op_b in (N_, T_):
            for op_c in (N_, T_):
                pr = KronProblem3D(op_a, op_b, op_c, m_a, n_a, m_b, n_b, m_c, n_c, 0.75, 1.25)
                a, b, c = uniform(g, m_a * n_a, dtype), uniform(g, m_b * n_b, dtype), uniform(g, m_c * n_c, dtype)
                x = uniform(g, n_a * n_b * n_c * batch, dtype)
                y = uniform(g, m_a * m_b * m_c * batch, dtype)
                got, want = tight(pr, a, b, c, x, y, batch)
                assert mismatches(got, want) == 0, (op_a, op_b, op_c)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_vs_double_oracle(dtype):
    """ref_kron3_apply (O(m^6)) within tolerance, alpha/beta affine contract."""
    o = oracle()
    m_a, n_a, m_b, n_b, m_c, n_c = 4, 3, 5, 2, 3, 6
    g = rng(251)
    batch = 7
    a, b, c = uniform(g, m_a * n_a, dtype), uniform(g, m_b * n_b, dtype), uniform(g, m_c * n_c, dtype)
    x, y = uniform(g, n_a * n_b * n_c * batch, dtype), uniform(g, m_a * m_b * m_c * batch, dtype)
    pr = KronProblem3D(N_, N_, N_, m_a, n_a, m_b, n_b, m_c, n_c, -0.5, 2.0)
    got, _ = tight(pr, a, b, c, x, y, batch)
    A = a.reshape(n_a, m_a).T.astype(np.float64)
    B = b.reshape(n_b, m_b).T.astype(np.float64)
    Cm = c.reshape(n_c, m_c).T.astype(np.float64)
    ex, ey = n_a * n_b * n_c, m_a * m_b * m_c
    for p in range(batch):
        X = x[p * ex:(p + 1) * ex].reshape(n_c, n_b, n_a).transpose(2, 1, 0).astype(np.float64)
        w = o.ref_kron3_apply(A, B, Cm, X).ravel(order="F") * -0.5 + 2.0 * y[p * ey:(p + 1) * ey]
        assert rel_err_inf(got[p * ey:(p + 1) * ey], w) < TOL[np.dtype(dtype)]


def test_identity_and_integer_exact():
    """test_kron3.cpp:88-134."""
    o = oracle()
    for n in (3, 16):
        batch = 4
        eye = np.eye(n).ravel(order="F")
        g = rng(257)
        x = uniform(g, n ** 3 * batch, np.float64)
        y = np.full(n ** 3 * batch, -1.0)
        pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        got, _ = tight(pr, eye, eye, eye, x, y, batch)
        assert np.array_equal(got, x)
        a, b, c = ints(g, n * n, np.float64), ints(g, n * n, np.float64), ints(g, n * n, np.float64)
        xi = ints(g, n ** 3 * batch, np.float64)
        got, _ = tight(pr, a, b, c, xi, np.full(n ** 3 * batch, np.nan), batch)
        A, B, Cm = (v.reshape(n, n).T for v in (a, b, c))
        for p in range(batch):
            X = xi[p * n ** 3:(p + 1) * n ** 3].reshape(n, n, n).transpose(2, 1, 0)
            assert np.array_equal(got[p * n ** 3:(p + 1) * n ** 3], o.ref_kron3_apply(A, B, Cm, X).ravel(order="F"))


def test_nan_y_beta_zero_and_alpha_zero():
    """test_kron3.cpp:225-245 and the alpha == 0 path (kron3.hpp:113-128)."""
    n, batch = 6, 11
    g = rng(263)
    a, b, c = uniform(g, n * n, np.float32), uniform(g, n * n, np.float32), uniform(g, n * n, np.float32)
    x = uniform(g, n ** 3 * batch, np.float32)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    got, _ = tight(pr, a, b, c, x, np.full(n ** 3 * batch, np.nan, np.float32), batch)
    assert not np.isnan(got).any()
    nanm = np.full(n * n, np.nan, np.float32)
    y0 = uniform(g, n ** 3 * batch, np.float32)
    pr0 = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n, alpha=0.0, beta=3.0)
    got, _ = tight(pr0, nanm, nanm, nanm, np.full(n ** 3 * batch, np.nan, np.float32), y0, batch)
    assert np.array_equal(got, y0 * np.float32(3.0))


def test_workspace_contract():
    """test_kron3.cpp:67-86 / 247-264: workspace_size values, overflow, and the
    too-small error (message names "workspace", needed and given counts) raised
    before any exit -- also with batch 0 irrelevant here (needed = 0 then)."""
    pr = KronProblem3D(m_a=2, n_a=2, m_b=3, n_b=3, m_c=2, n_c=4)
    assert kb.kron3_workspace_size(pr, 1) == 24
    n, batch = 2, 1
    a = np.ones(4)
    x = np.ones(2 * 3 * 4)
    with pytest.raises(ValueError) as e:
        run(pr, a, (2, 2), 2, np.ones(9), (3, 3), 3, np.ones(8), (2, 4), 2, x, 2, 6, 24, np.zeros(12), 2, 6, 12, batch,
            work_cap=23)
    assert "workspace" in str(e.value) and "24" in str(e.value) and "23" in str(e.value)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [3, 16])
def test_padding_bit_identity(dtype, n):
    """test_kron3.cpp:266-325: padded ld/ld2/strides == tight bits; Y padding untouched."""
    g = rng(269 + n)
    batch = 9
    a, b, c = uniform(g, n * n, dtype), uniform(g, n * n, dtype), uniform(g, n * n, dtype)
    x, y0 = uniform(g, n ** 3 * batch, dtype), uniform(g, n ** 3 * batch, dtype)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n, alpha=1.5, beta=0.25)
    tight_y, _ = tight(pr, a, b, c, x, y0, batch)
    ld, ld2 = n + 3, (n + 3) * n + 5
    s = ld2 * n + 7
    xp = np.full(s * batch, np.nan, dtype)
    yp = np.full(s * batch, 777.0, dtype)
    for p in range(batch):
        for k in range(n):
            for j in range(n):
                o = p * s + k * ld2 + j * ld
                t = p * n ** 3 + k * n * n + j * n
                xp[o:o + n] = x[t:t + n]
                yp[o:o + n] = y0[t:t + n]
    for host in (False, True):
        got = run(pr, a, (n, n), n, b, (n, n), n, c, (n, n), n, xp, ld, ld2, s, yp, ld, ld2, s, batch, host=host)
        mask = np.ones_like(got, bool)
        for p in range(batch):
            for k in range(n):
                for j in range(n):
                    o = p * s + k * ld2 + j * ld
                    t = p * n ** 3 + k * n * n + j * n
                    assert mismatches(got[o:o + n], tight_y[t:t + n]) == 0
                    mask[o:o + n] = False
        assert np.all(got[mask] == 777.0)


def test_composition_via_kron2_and_gemm():
    """test_kron3.cpp:327-383 (Algorithm 1): kron3 == per-plane kron2 followed
    by the mode-3 contraction -- checked bit-exactly through the oracle's
    staged restatement, and kron2 planes through the GPU kron2."""
    n, batch = 5, 3
    g = rng(271)
    a, b, c = uniform(g, n * n, np.float64), uniform(g, n * n, np.float64), uniform(g, n * n, np.float64)
    x = uniform(g, n ** 3 * batch, np.float64)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    got, want = tight(pr, a, b, c, x, np.zeros(n ** 3 * batch), batch)
    assert mismatches(got, want) == 0
    # stage 1 as a batched kron2 over the n*batch planes (alpha 1, beta 0)
    from paper_1304_7054_b200 import KronProblem2D

    X, T = to_dev(x), to_dev(np.zeros(n ** 3 * batch))
    kb.kron2(KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n), MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n),
             BatchView(MatrixView(X, n, n, n), n * batch, n * n), BatchView(MatrixView(T, n, n, n), n * batch, n * n))
    t2 = to_host(T)
    # stage 2: Y(i,j,k) = sum_N T2(i,j,N) C(k,N) in ascending N with fma
    Cm = c.reshape(n, n).T
    for p in range(batch):
        T2 = t2[p * n ** 3:(p + 1) * n ** 3].reshape(n, n, n).transpose(2, 1, 0)
        Y = np.zeros((n, n, n))
        for k in range(n):
            acc = np.zeros((n, n))
            for N in range(n):
                acc = acc + T2[:, :, N] * Cm[k, N]  # close to fma order; tolerance check
            Y[:, :, k] = acc
        assert rel_err_inf(got[p * n ** 3:(p + 1) * n ** 3], Y.ravel(order="F")) < 1e-12


def test_batch_split_determinism_and_host_staging():
    n, batch = 16, 600
    a, b, c, x, y = oracle().generate_batch(np.float32, 9, n, True, batch)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    full, _ = tight(pr, a, b, c, x, y, batch)
    e = n ** 3
    for lo, hi in ((0, 1), (1, 5), (5, 333), (333, 600)):
        part, _ = tight(pr, a, b, c, x[lo * e:hi * e], y[lo * e:hi * e], hi - lo)
        assert mismatches(part, full[lo * e:hi * e]) == 0
    host, _ = tight(pr, a, b, c, x, y, batch, host=True)
    assert mismatches(host, full) == 0


@pytest.mark.parametrize("dtype,batch", [(np.float32, 262144), (np.float64, 131072)])
def test_baseline_configs_sampled_oracle(dtype, batch):
    """BASELINE configs 3/4 at full size (3-D n=16, fp32 262,144 / fp64
    131,072): run_one's 16 sampled entries vs the double O(m^6) oracle, and
    bit-exact vs the restated CPU path on those entries."""
    import torch

    o = oracle()
    n = 16
    a, b, c, x, y = o.generate_batch(dtype, 1, n, True, batch)
    pr = KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    X, Y = to_dev(x), torch.empty(n ** 3 * batch, dtype=tdt, device="cuda")
    kb.kron3(pr, MatrixView(to_dev(a), n, n, n), MatrixView(to_dev(b), n, n, n), MatrixView(to_dev(c), n, n, n),
             BatchView(Array3View(X, n, n, n, n, n * n), batch, n ** 3),
             BatchView(Array3View(Y, n, n, n, n, n * n), batch, n ** 3), Workspace(None, n ** 3 * batch))
    got = to_host(Y)
    A, B, Cm = (v.reshape(n, n).T.astype(np.float64) for v in (a, b, c))
    e = n ** 3
    for p in sorted(set(rng(11).integers(0, batch, 6).tolist()) | {batch - 1}):
        s = slice(p * e, (p + 1) * e)
        X64 = x[s].reshape(n, n, n).transpose(2, 1, 0).astype(np.float64)
        assert rel_err_inf(got[s], o.ref_kron3_apply(A, B, Cm, X64).ravel(order="F")) < TOL[np.dtype(dtype)]
        yo = np.zeros(e, dtype)
        o.kron3("N", "N", "N", n, n, n, n, n, n, 1, dtype(1), a, n, b, n, c, n, x[s], n, n * n, e, dtype(0), yo, n,
                n * n, e)
        assert mismatches(got[s], yo) == 0


_SMEM_ORDER = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_1304_7054_b200 as kb
from kb_testutil import mismatches, oracle, to_dev, to_host
o = oracle()
n, batch = 13, 41
e = n ** 3
for dt in (np.float32, np.float64):
    for pad in (5, 0):  # padded Y entry stride first (no Y image), then tight (Y image: more smem)
        a, b, c, x, y = o.generate_batch(dt, 1, n, True, batch)
        sy = e + pad
        y0 = np.zeros(sy * batch, dt)
        want = y0.copy()
        X, Y = to_dev(x), to_dev(y0)
        pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        kb.kron3(pr, kb.MatrixView(to_dev(a), n, n, n), kb.MatrixView(to_dev(b), n, n, n), kb.MatrixView(to_dev(c), n, n, n),
                 kb.BatchView(kb.Array3View(X, n, n, n, n, n * n), batch, e),
                 kb.BatchView(kb.Array3View(Y, n, n, n, n, n * n), batch, sy), kb.Workspace(None, e * batch))
        o.kron3("N", "N", "N", n, n, n, n, n, n, batch, dt(1), a, n, b, n, c, n, x, n, n * n, e, dt(0), want, n, n * n, sy)
        assert mismatches(to_host(Y), want) == 0, (dt, pad)
print("OK")
"""


def test_same_kernel_two_smem_sizes_fresh_process():
    """One kernel, two dynamic shared-memory sizes in one process: the odd-n
    column-wise kernel reserves its Y image only for a tight Y, so a padded-Y
    call followed by a tight one needs the opt-in smem limit raised (a cache
    keyed by kernel alone launched the second with 'invalid argument')."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SMEM_ORDER, root], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
