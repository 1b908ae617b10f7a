"""Generate tests/golden/kron_golden.npz from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libkronref.so, compiled by
oracle/Makefile from /root/reference/proj sources) on small, fixed cases and
stores inputs + outputs. The fixtures travel with the repo (the reference does
not exist on the GPU box) and pin both the C oracle (tests/test_oracle.py) and
the sm_100a path (tests/test_gpu_golden.py).

    python tests/golden/make_golden.py        # needs /root/reference + make -C oracle
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402

OPS = ("N", "T")


def stored(op, r, c):
    return (c, r) if op != "N" else (r, c)


def main(out=os.path.join(HERE, "kron_golden.npz")):
    ref = Reference()
    assert ref.has_openmp, "reference built without OpenMP"
    g = np.random.default_rng(20131304)
    d = {}

    # -- KATs of the reference's own tests
    # test_reference.cpp:41-51 kron_matrix([[1,2],[3,4]], I2)
    d["kat_kron_matrix"] = ref.kron_matrix(np.array([[1.0, 2.0], [3.0, 4.0]]), np.eye(2))
    # test_kron2.cpp:59-67 all-ones -> 10
    y = np.array([-1.0])
    ref.kron2("N", "N", "N", 1, 2, 1, 2, 1, 1.0, np.ones(2), (1, 2), 1, np.ones(2), (1, 2), 1,
              np.array([1.0, 3.0, 2.0, 4.0]), (2, 2), 2, 4, 0.0, y, (1, 1), 1, 1)
    d["kat_all_ones"] = y
    # test_bench.cpp:34-40, 57-65; test_kron3.cpp:67-86
    d["kat_flops"] = np.array([ref.flops_kron(10, False), ref.flops_kron(16, True), ref.flops_kron(1, False),
                               ref.flops_kron(1, True)], np.int64)
    d["kat_problem_bytes"] = np.array([ref.problem_bytes(16, True, False, 100000)], np.uint64)
    d["kat_workspace"] = np.array([ref.kron3_workspace_size(4, 8, 20, 1), ref.kron3_workspace_size(0, 8, 20, 5),
                                   ref.kron3_workspace_size(4, 8, 20, 0),
                                   ref.kron3_workspace_size(100, 64, 64, 1000)], np.int64)

    # -- generate_batch + reference kron2/kron3 at every n (alpha 1, beta 0)
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        for n in range(1, 17):
            for dims3 in (False, True):
                batch = 3
                a, b, c, x, y = ref.generate_batch(dt, 1, n, dims3, batch)
                key = f"gen_{tag}_{'3d' if dims3 else '2d'}_{n}"
                d[key + "_a"], d[key + "_b"], d[key + "_x"], d[key + "_y0"] = a, b, x, y
                yo = y.copy()
                if dims3:
                    d[key + "_c"] = c
                    work = np.empty(n ** 3 * batch, dt)
                    ref.kron3("N", "N", "N", n, n, n, n, n, n, batch, dt(1), a, (n, n), n, b, (n, n), n, c, (n, n), n,
                              x, (n, n, n), n, n * n, n ** 3, dt(0), yo, (n, n, n), n, n * n, n ** 3, work)
                else:
                    ref.kron2("N", "N", "N", n, n, n, n, batch, dt(1), a, (n, n), n, b, (n, n), n, x, (n, n), n, n * n,
                              dt(0), yo, (n, n), n, n * n)
                d[key + "_y"] = yo

    # -- rectangular op combinations, alpha .75 beta 1.25 (test_kron2.cpp:96-140,
    #    test_kron3.cpp:136-183), padded layouts included
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        m_a, n_a, m_b, n_b, batch = 3, 5, 4, 2, 4
        for oa in OPS:
            for ob in OPS:
                for ox in OPS:
                    ar, ac = stored(oa, m_a, n_a)
                    br, bc = stored(ob, m_b, n_b)
                    xr, xc = stored(ox, n_a, n_b)
                    lda, ldb, ldx, ldy = ar + 1, br + 2, xr + 3, m_a + 1
                    sx, sy = ldx * xc + 2, ldy * m_b + 3
                    a = (g.random(lda * ac) * 2 - 1).astype(dt)
                    b = (g.random(ldb * bc) * 2 - 1).astype(dt)
                    x = (g.random(sx * batch) * 2 - 1).astype(dt)
                    y0 = (g.random(sy * batch) * 2 - 1).astype(dt)
                    y = y0.copy()
                    ref.kron2(oa, ob, ox, m_a, n_a, m_b, n_b, batch, dt(0.75), a, (ar, ac), lda, b, (br, bc), ldb, x,
                              (xr, xc), ldx, sx, dt(1.25), y, (m_a, m_b), ldy, sy)
                    key = f"rect2_{tag}_{oa}{ob}{ox}"
                    for k, v in (("a", a), ("b", b), ("x", x), ("y0", y0), ("y", y)):
                        d[f"{key}_{k}"] = v
                    d[f"{key}_dims"] = np.array([m_a, n_a, m_b, n_b, batch, lda, ldb, ldx, sx, ldy, sy], np.int64)
        m_a, n_a, m_b, n_b, m_c, n_c, batch = 3, 5, 4, 2, 2, 6, 3
        for oa in OPS:
            for ob in OPS:
                for oc in OPS:
                    ar, ac = stored(oa, m_a, n_a)
                    br, bc = stored(ob, m_b, n_b)
                    cr, cc = stored(oc, m_c, n_c)
                    ldx, ldx2 = n_a + 1, (n_a + 1) * n_b + 2
                    ldy, ldy2 = m_a + 2, (m_a + 2) * m_b + 1
                    sx, sy = ldx2 * n_c + 3, ldy2 * m_c + 1
                    a = (g.random(ar * ac) * 2 - 1).astype(dt)
                    b = (g.random(br * bc) * 2 - 1).astype(dt)
                    c = (g.random(cr * cc) * 2 - 1).astype(dt)
                    x = (g.random(sx * batch) * 2 - 1).astype(dt)
                    y0 = (g.random(sy * batch) * 2 - 1).astype(dt)
                    y = y0.copy()
                    work = np.empty(m_a * m_b * n_c * batch, dt)
                    ref.kron3(oa, ob, oc, m_a, n_a, m_b, n_b, m_c, n_c, batch, dt(0.75), a, (ar, ac), ar, b, (br, bc),
                              br, c, (cr, cc), cr, x, (n_a, n_b, n_c), ldx, ldx2, sx, dt(1.25), y, (m_a, m_b, m_c),
                              ldy, ldy2, sy, work)
                    key = f"rect3_{tag}_{oa}{ob}{oc}"
                    for k, v in (("a", a), ("b", b), ("c", c), ("x", x), ("y0", y0), ("y", y)):
                        d[f"{key}_{k}"] = v
                    d[f"{key}_dims"] = np.array([m_a, n_a, m_b, n_b, m_c, n_c, batch, ldx, ldx2, sx, ldy, ldy2, sy],
                                                np.int64)

    # -- reference validation messages (what the product must reproduce)
    msgs = []
    cases = [
        # (kron2 args tweaks): stored X 3x3 with ld 2
        dict(ldx=2), dict(sx=8), dict(lenx=20), dict(ldy=1), dict(lena=5), dict(batch=-1),
    ]
    for cse in cases:
        n, batch = 3, 3
        a = np.zeros(9)
        x = np.zeros(27)
        y = np.zeros(27)
        kw = dict(ldx=3, sx=9, lenx=27, ldy=3, lena=9, batch=batch)
        kw.update(cse)
        try:
            ref.kron2("N", "N", "N", n, n, n, n, kw["batch"], 1.0, a, (n, n), 3, a, (n, n), 3, x, (n, n), kw["ldx"],
                      kw["sx"], 0.0, y, (n, n), kw["ldy"], 9, lens=(kw["lena"], 9, kw["lenx"], 27))
            msgs.append("")
        except ValueError as e:
            msgs.append(str(e))
    d["msg_kron2"] = np.array(msgs)
    d["msg_kron2_cases"] = np.array([repr(c) for c in cases])
    try:
        pr_args = ("N", "N", "N", 2, 2, 3, 3, 2, 4, 1, 1.0, np.ones(4), (2, 2), 2, np.ones(9), (3, 3), 3, np.ones(8),
                   (2, 4), 2, np.ones(24), (2, 3, 4), 2, 6, 24, 0.0, np.zeros(12), (2, 3, 2), 2, 6, 12, None, 23)
        ref.kron3(*pr_args)
        d["msg_workspace"] = np.array([""])
    except ValueError as e:
        d["msg_workspace"] = np.array([str(e)])
    np.savez_compressed(out, **d)
    print(f"wrote {out}: {len(d)} arrays")


if __name__ == "__main__":
    main()
