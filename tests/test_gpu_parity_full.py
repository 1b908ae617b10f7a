"""Full-batch parity at every BASELINE config (-m gpu): the GPU output over
the WHOLE batch vs the unmodified reference (oracle/_ref, OpenMP) on the same
generate_batch inputs (seed 1, alpha 1, beta 0, tight layout) -- SURVEY.md
§8c protocol (1) (the gate: per-entry rel_err_inf <= 1e-5 / 1e-12,
/root/reference/proj/tests/test_util.hpp:93-113) and (2) (bitwise: at n = 10
and n = 16 the reference's g++ code is an FMA chain in the Appendix-A order,
so the expected mismatch count is 0).

Entries past 2^31 elements (the 2-D n = 16 config holds 1.07e9 elements per
buffer, the 3-D n = 16 ones 1.07e9 too) are covered whole, not sampled.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_1304_7054_b200 as kb
from kb_testutil import TOL, reference

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CONFIGS = [  # BASELINE.json configs[0..3]
    ("kron2-f32-n10", False, 10, np.float32, 65536),
    ("kron2-f32-n16", False, 16, np.float32, 4194304),
    ("kron3-f32-n10", True, 10, np.float32, 262144),
    ("kron3-f32-n16", True, 16, np.float32, 262144),
    ("kron3-f64-n16", True, 16, np.float64, 131072),
]


def _rel_err_inf_per_entry(got, want, e):
    worst = 0.0
    step = max(1, (64 << 20) // (e * got.itemsize))
    for p0 in range(0, got.size // e, step):
        g = got[p0 * e:(p0 + step) * e].reshape(-1, e).astype(np.float64)
        w = want[p0 * e:(p0 + step) * e].reshape(-1, e).astype(np.float64)
        worst = max(worst, float((np.abs(g - w).max(axis=1) / np.maximum(1.0, np.abs(w).max(axis=1))).max()))
    return worst


@pytest.mark.parametrize("name, dims3, n, dtype, batch", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_full_batch_parity_device_resident(name, dims3, n, dtype, batch):
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    e = n ** (3 if dims3 else 2)
    a, b, c, x, _ = ref.generate_batch(dtype, 1, n, dims3, batch)
    want = np.zeros_like(x)
    if dims3:
        ref.kron3("N", "N", "N", n, n, n, n, n, n, batch, dtype(1), a, (n, n), n, b, (n, n), n, c, (n, n), n, x,
                  (n, n, n), n, n * n, e, dtype(0), want, (n, n, n), n, n * n, e, np.empty(e * batch, dtype))
    else:
        ref.kron2("N", "N", "N", n, n, n, n, batch, dtype(1), a, (n, n), n, b, (n, n), n, x, (n, n), n, e, dtype(0),
                  want, (n, n), n, e)
    X = torch.from_numpy(x).cuda()
    del x
    Y = torch.full_like(X, float("nan"))
    MV, BV = kb.MatrixView, kb.BatchView
    if dims3:
        pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        kb.kron3(pr, MV(a, n, n, n), MV(b, n, n, n), MV(c, n, n, n), BV(kb.Array3View(X, n, n, n, n, n * n), batch, e),
                 BV(kb.Array3View(Y, n, n, n, n, n * n), batch, e), kb.Workspace(None, e * batch))
        assert kb.last_path() == "kron3_fast"
    else:
        pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
        kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), BV(MV(X, n, n, n), batch, e), BV(MV(Y, n, n, n), batch, e))
        assert kb.last_path() == "kron2_fast"
    del X
    got = Y.cpu().numpy()
    del Y
    ub = np.uint32 if dtype == np.float32 else np.uint64
    mism = int(np.count_nonzero(got.view(ub) != want.view(ub)))
    err = _rel_err_inf_per_entry(got, want, e)
    print(f"{name}: {batch} entries, mismatches {mism}, max rel_err_inf {err:.3g}")
    assert err <= TOL[np.dtype(dtype)]
    assert mism == 0  # bitwise: FMA-chain sizes


def test_cpu_ref_tool_parity_through_pageable_host_path():
    """oracle/cpu_ref.py (the bench's cpu_baseline + parity leg) on the 3-D
    fp64 config: the product called with the reference's own pageable host
    buffers (the staged pipeline with pinned bounce buffers) over the full
    batch, bit-identical; the CPU timing is the full config with pinned
    OpenMP."""
    if reference() is None:
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "-m", "oracle.cpu_ref", "--workload", "kron3-f64-n16", "--reps", "3",
                        "--parity"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["full_batch"] and out["batch"] == 131072
    assert out["omp"]["OMP_PROC_BIND"] == "close"
    p = out["parity"]
    assert p["ok"] and p["mismatches"] == 0 and p["entries"] == 131072
    assert p["product_path"] == "kron3_fast"
