"""CPU-side checks of the C ABI boundary (no GPU needed).

* libkronbatch_b200.so loads and exports every symbol include/kronbatch_b200.h
  declares;
* the ABI's host-side contract -- validation order and message text, the
  workspace contract, early exits that launch nothing -- matches the
  reference (messages pinned by tests/golden/kron_golden.npz, produced by the
  reference itself);
* the Python mirror raises the same errors before touching the device.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1304_7054_b200 as kb
from paper_1304_7054_b200 import (Array3View, BatchView, KronProblem2D, KronProblem3D, MatrixOp, MatrixView,
                                  Workspace, _lib)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "kron_golden.npz")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kronbatch_b200.h")).read()
    return sorted(set(re.findall(r"\b(kb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert set(syms) >= {"kb_skron2", "kb_dkron2", "kb_skron3", "kb_dkron3", "kb_kron3_workspace_size"}
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(_lib.ABI_SYMBOLS) == set(syms)
    assert "sm_100a" in kb.version()


def abi_kron2(**over):
    """Call kb_dkron2 directly with a valid 3x3 batch-3 layout, then overrides."""
    a = np.zeros(9)
    x = np.zeros(27)
    y = np.zeros(27)
    kw = dict(ta=b"N", tb=b"N", tx=b"N", m_a=3, n_a=3, m_b=3, n_b=3, batch=3, alpha=1.0, lda=3, lena=9, ldb=3, lenb=9,
              ldx=3, sx=9, lenx=27, beta=0.0, ldy=3, sy=9, leny=27)
    kw.update(over)
    err = C.create_string_buffer(512)
    p = lambda v: v.ctypes.data_as(C.c_void_p)
    rc = _lib.lib.kb_dkron2(kw["ta"], kw["tb"], kw["tx"], kw["m_a"], kw["n_a"], kw["m_b"], kw["n_b"], kw["batch"],
                            kw["alpha"], p(a), kw["lda"], kw["lena"], p(a), kw["ldb"], kw["lenb"], p(x), kw["ldx"],
                            kw["sx"], kw["lenx"], kw["beta"], p(y), kw["ldy"], kw["sy"], kw["leny"], None, err, 512)
    return rc, err.value.decode()


def test_abi_validation_messages_match_reference():
    gold = np.load(GOLD)
    cases = [dict(ldx=2), dict(sx=8), dict(lenx=20), dict(ldy=1), dict(lena=5), dict(batch=-1)]
    assert [repr(c) for c in cases] == list(gold["msg_kron2_cases"])
    for case, want in zip(cases, gold["msg_kron2"]):
        rc, msg = abi_kron2(**case)
        assert rc == _lib.KB_EINVAL
        assert msg == want


def test_abi_early_exits_do_not_touch_device():
    # batch 0, m_a 0 and alpha 0 with beta 1 return before any CUDA call
    assert abi_kron2(batch=0, lenx=0, leny=0) == (0, "")
    assert abi_kron2(m_a=0, lda=1, lena=3, ldy=1, sy=3, leny=9)[0] == 0
    assert abi_kron2(alpha=0.0, beta=1.0)[0] == 0
    assert abi_kron2(ta=b"Q")[0] == _lib.KB_EINVAL


def test_workspace_size_contract():
    gold = np.load(GOLD)
    pr = lambda a, b, c: KronProblem3D(m_a=a, m_b=b, n_c=c)
    got = [kb.kron3_workspace_size(pr(4, 8, 20), 1), kb.kron3_workspace_size(pr(0, 8, 20), 5),
           kb.kron3_workspace_size(pr(4, 8, 20), 0), kb.kron3_workspace_size(pr(100, 64, 64), 1000)]
    assert got == list(gold["kat_workspace"])
    with pytest.raises(OverflowError):
        kb.kron3_workspace_size(pr(1 << 32, 1 << 32, 4), 1)
    with pytest.raises(ValueError):
        kb.kron3_workspace_size(pr(-1, 1, 1), 1)


def test_workspace_too_small_message_before_any_exit():
    """kron3 checks capacity before the batch==0 / alpha==0 exits
    (kron3.hpp:104-111); message pinned against the reference."""
    gold = np.load(GOLD)
    pr = KronProblem3D(m_a=2, n_a=2, m_b=3, n_b=3, m_c=2, n_c=4)
    with pytest.raises(ValueError) as e:
        kb.kron3(pr, MatrixView(np.ones(4), 2, 2, 2), MatrixView(np.ones(9), 3, 3, 3), MatrixView(np.ones(8), 2, 4, 2),
                 BatchView(Array3View(np.ones(24), 2, 3, 4, 2, 6), 1, 24),
                 BatchView(Array3View(np.zeros(12), 2, 3, 2, 2, 6), 1, 12), Workspace(None, 23))
    assert str(e.value) == gold["msg_workspace"][0]


def test_python_mirror_validation():
    """test_layout.cpp / test_kron2.cpp:410-460 shapes of errors."""
    a, x, y = np.zeros(9), np.zeros(27), np.zeros(27)
    A = MatrixView(a, 3, 3, 3)
    ok_x = BatchView(MatrixView(x, 3, 3, 3), 3, 9)
    ok_y = BatchView(MatrixView(y, 3, 3, 3), 3, 9)
    with pytest.raises(ValueError, match=r"^kron2: A: op\(A\) is 3 x 3, expected 4 x 3$"):
        kb.kron2(KronProblem2D(m_a=4, n_a=3, m_b=3, n_b=3), A, A, ok_x, ok_y)
    with pytest.raises(ValueError, match="^kron2: X and Y batch_count differ$"):
        kb.kron2(KronProblem2D(m_a=3, n_a=3, m_b=3, n_b=3), A, A, ok_x, BatchView(MatrixView(y, 3, 3, 3), 2, 9))
    with pytest.raises(ValueError, match=r"^kron2: X: ld2|^kron2: X: ld \(2\) < \(3\)$"):
        kb.kron2(KronProblem2D(m_a=3, n_a=3, m_b=3, n_b=3), A, A, BatchView(MatrixView(x, 3, 3, 2), 3, 9), ok_y)
    with pytest.raises(ValueError, match=r"ld2 \(5\) < \(6\)"):
        kb.validate(Array3View(np.zeros(100), 2, 3, 4, 2, 5), "kron3: X")
    with pytest.raises(ValueError, match=r"^kron3: X: entry dims do not match n_a x n_b x n_c$"):
        kb.kron3(KronProblem3D(m_a=2, n_a=2, m_b=2, n_b=2, m_c=2, n_c=2), MatrixView(np.ones(4), 2, 2, 2),
                 MatrixView(np.ones(4), 2, 2, 2), MatrixView(np.ones(4), 2, 2, 2),
                 BatchView(Array3View(np.ones(27), 3, 3, 3, 3, 9), 1, 27),
                 BatchView(Array3View(np.ones(8), 2, 2, 2, 2, 4), 1, 8), Workspace(None, 100))
    with pytest.raises(TypeError):  # one element type per call
        kb.kron2(KronProblem2D(m_a=3, n_a=3, m_b=3, n_b=3), MatrixView(np.zeros(9, np.float32), 3, 3, 3), A, ok_x, ok_y)
    assert kb.op_dims(MatrixOp.Transpose, 3, 5) == (5, 3) and kb.op_dims(MatrixOp.NoTranspose, 3, 5) == (3, 5)
    assert kb.footprint(MatrixView(np.zeros(20), 4, 0, 4)) == 0
    assert kb.footprint(Array3View(np.zeros(40), 2, 3, 4, 2, 7)) == 28
