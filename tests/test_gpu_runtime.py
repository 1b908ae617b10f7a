"""The runtime around the kernels (-m gpu): the device-buffer manager (lane
pool), multi-device sharding, the parts API for batches already split over
GPUs, stream ordering, and the staged host-buffer pipeline (pinned and
pageable).

Reference analogues: detail::run_chunked's worker-count invariance
(/root/reference/proj/include/kronbatch/detail.hpp:156-180,
tests/test_kron2.cpp:462-491 -- here across GPU slices / parts / host
threads), "no per-call cudaMalloc", and the synchronous,
thread-safe call contract.
"""
import threading

import numpy as np
import pytest
import torch

import paper_1304_7054_b200 as kb
from kb_testutil import mismatches, oracle, rng, to_dev, uniform

pytestmark = pytest.mark.gpu
MV, BV, A3 = kb.MatrixView, kb.BatchView, kb.Array3View


def _kron2_args(n, x, y, batch, alpha=1.0, beta=0.0):
    pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n, alpha=alpha, beta=beta)
    return pr, BV(MV(x, n, n, n), batch, n * n), BV(MV(y, n, n, n), batch, n * n)


def _ref2(o, dtype, n, batch, a, b, x, y, alpha=1.0, beta=0.0):
    want = y.copy()
    o.kron2("N", "N", "N", n, n, n, n, batch, dtype(alpha), a, n, b, n, x, n, n * n, dtype(beta), want, n, n * n)
    return want


def _free_bytes():
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


# ------------------------------------------------------------ lane pool ----

def test_sharded_calls_do_not_grow_device_memory():
    """500 sharded calls (devices [0, 0]: two slices, two pool workers) of a
    host-resident batch: streams and staging buffers are allocated once, so
    free device memory and the pool size stay flat (the old
    per-call thread-local resources leaked ~hundreds of MiB per call)."""
    o = oracle()
    n, batch = 16, 3001
    a, b, _, x, y = o.generate_batch(np.float32, 2, n, False, batch)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.zeros(y.size, dtype=torch.float32).pin_memory()
    ypg = np.zeros_like(y)  # pageable Y: the bounce-buffer path too
    ex = kb.Exec(devices=[0, 0])
    pr, xb, yb = _kron2_args(n, xp, yp, batch)
    _, xb2, yb2 = _kron2_args(n, x, ypg, batch)
    for _ in range(10):
        kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb, yb, exec_=ex)
        kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb2, yb2, exec_=ex)
    free0, pool0 = _free_bytes(), kb.pooled_bytes(0)
    for _ in range(250):
        kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb, yb, exec_=ex)
        kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb2, yb2, exec_=ex)
    free1, pool1 = _free_bytes(), kb.pooled_bytes(0)
    assert pool1 == pool0
    assert free0 - free1 < (4 << 20), (free0, free1)
    want = _ref2(o, np.float32, n, batch, a, b, x, y)
    assert mismatches(yp.numpy(), want) == 0
    assert mismatches(ypg, want) == 0


def test_release_buffers_returns_pooled_memory():
    o = oracle()
    n, batch = 16, 50000
    a, b, _, x, y = o.generate_batch(np.float32, 3, n, False, batch)
    yh = np.zeros_like(y)
    pr, xb, yb = _kron2_args(n, x, yh, batch)
    kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb, yb)
    assert kb.pooled_bytes(0) >= x.nbytes  # staging buffers held for reuse
    free0 = _free_bytes()
    kb.release_buffers()
    assert kb.pooled_bytes(-1) == 0
    assert _free_bytes() - free0 >= x.nbytes // 2
    kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb, yb)  # the pool refills on demand
    assert mismatches(yh, _ref2(o, np.float32, n, batch, a, b, x, y)) == 0


def test_concurrent_callers_from_many_threads():
    """Concurrent calls on disjoint buffers from 6 host threads:
    each gets its own lane; results are bit-exact."""
    o = oracle()
    n, batch = 12, 2000
    a, b, _, x, y = o.generate_batch(np.float64, 4, n, False, batch)
    want = _ref2(o, np.float64, n, batch, a, b, x, y, 0.5, 1.5)
    outs, errs = [], []

    def work(i):
        try:
            for _ in range(20):
                Y = y.copy() if i % 2 else to_dev(y)
                X = x if i % 3 else to_dev(x)
                pr, xb, yb = _kron2_args(n, X, Y, batch, 0.5, 1.5)
                kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb, yb)
            outs.append(Y if isinstance(Y, np.ndarray) else Y.cpu().numpy())
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert len(outs) == 6
    for got in outs:
        assert mismatches(got, want) == 0


# ------------------------------------------------------------- ordering ----

def _busy(ms_target=200):
    """Queue ~ms_target of work on the current (legacy default) stream."""
    m = torch.randn(4096, 4096, device="cuda")
    for _ in range(max(1, ms_target // 2)):
        m = torch.tanh(m @ m * 1e-3)
    return m


def test_call_is_ordered_after_default_stream_producers():
    """X and Y (beta != 0) are written by torch on the legacy default stream
    behind ~200 ms of queued work, and the library is called with no
    synchronisation in between: the (blocking) library stream must wait for
    them (a non-blocking library stream could read stale X)."""
    o = oracle()
    n, batch = 16, 20000
    a, b, _, x, y = o.generate_batch(np.float32, 6, n, False, batch)
    Xsrc, Ysrc = to_dev(x), to_dev(y)
    torch.cuda.synchronize()
    X = torch.full_like(Xsrc, float("nan"))
    Y = torch.full_like(Ysrc, float("nan"))
    torch.cuda.synchronize()
    _busy()
    X.copy_(Xsrc)  # the producers, queued last on stream 0
    Y.copy_(Ysrc)
    pr, xb, yb = _kron2_args(n, X, Y, batch, 0.5, 2.0)
    kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), xb, yb)
    assert mismatches(Y.cpu().numpy(), _ref2(o, np.float32, n, batch, a, b, x, y, 0.5, 2.0)) == 0


def test_async_calls_on_two_streams_do_not_share_pooled_buffers():
    """Two asynchronous generic-path calls (rectangular: the constants are
    uploaded into pooled device memory) on two streams, the first one queued
    behind long work: the second call must not overwrite the constants the
    first kernel has yet to read (KB_EXEC_ASYNC)."""
    o = oracle()
    g = rng(21)
    m_a, n_a, m_b, n_b, batch = 5, 7, 6, 3, 3000
    outs, wants = [], []
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    calls = []
    for s in (s1, s2):
        A = uniform(g, m_a * n_a, np.float32)
        B = uniform(g, m_b * n_b, np.float32)
        x = uniform(g, n_a * n_b * batch, np.float32)
        X = to_dev(x)
        Y = torch.zeros(m_a * m_b * batch, dtype=torch.float32, device="cuda")
        want = np.zeros(m_a * m_b * batch, np.float32)
        o.kron2("N", "N", "N", m_a, n_a, m_b, n_b, batch, np.float32(1), A, m_a, B, m_b, x, n_a, n_a * n_b,
                np.float32(0), want, m_a, m_a * m_b)
        calls.append((s, A, B, X, Y))
        wants.append(want)
    torch.cuda.synchronize()
    for i, (s, A, B, X, Y) in enumerate(calls):
        if i == 0:
            with torch.cuda.stream(s):
                _busy()
        pr = kb.KronProblem2D(m_a=m_a, n_a=n_a, m_b=m_b, n_b=n_b)
        kb.kron2(pr, MV(A, m_a, n_a, m_a), MV(B, m_b, n_b, m_b), BV(MV(X, n_a, n_b, n_a), batch, n_a * n_b),
                 BV(MV(Y, m_a, m_b, m_a), batch, m_a * m_b), exec_=kb.Exec(stream=s, asynchronous=True))
        assert kb.last_path() == "kron2_generic"
    torch.cuda.synchronize()
    for (_, _, _, _, Y), want in zip(calls, wants):
        assert mismatches(Y.cpu().numpy(), want) == 0


# ---------------------------------------------------------------- parts ----

@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("dims3", [False, True])
def test_parts_api_bit_identical_to_one_call(dtype, dims3):
    """A device-resident batch split into 3 ragged parts (devices [0, 0, 0],
    one stream each) through kb_?kron{2,3}_parts == one call over the whole
    batch, sync and async."""
    o = oracle()
    n, batch = 16 if dtype == np.float32 else 10, 1001
    a, b, c, x, y = o.generate_batch(dtype, 8, n, dims3, batch)
    e = n ** (3 if dims3 else 2)
    X = to_dev(x)
    cuts = [0, 400, 401, batch]
    for asynchronous in (False, True):
        Y = torch.zeros(e * batch, dtype=X.dtype, device="cuda")
        streams = [torch.cuda.Stream() for _ in range(3)]
        parts = []
        for i in range(3):
            p0, p1 = cuts[i], cuts[i + 1]
            if dims3:
                xv = BV(A3(X[p0 * e:p1 * e], n, n, n, n, n * n), p1 - p0, e)
                yv = BV(A3(Y[p0 * e:p1 * e], n, n, n, n, n * n), p1 - p0, e)
            else:
                xv = BV(MV(X[p0 * e:p1 * e], n, n, n), p1 - p0, e)
                yv = BV(MV(Y[p0 * e:p1 * e], n, n, n), p1 - p0, e)
            parts.append(kb.Part(0, xv, yv, streams[i] if asynchronous else None))
        if dims3:
            pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n, alpha=0.75)
            kb.kron3_parts(pr, MV(a, n, n, n), MV(b, n, n, n), MV(c, n, n, n), parts, asynchronous=asynchronous)
            want = np.zeros_like(y)
            o.kron3("N", "N", "N", n, n, n, n, n, n, batch, dtype(0.75), a, n, b, n, c, n, x, n, n * n, e, dtype(0),
                    want, n, n * n, e)
        else:
            pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n, alpha=0.75)
            kb.kron2_parts(pr, MV(a, n, n, n), MV(b, n, n, n), parts, asynchronous=asynchronous)
            want = np.zeros_like(y)
            o.kron2("N", "N", "N", n, n, n, n, batch, dtype(0.75), a, n, b, n, x, n, e, dtype(0), want, n, e)
        torch.cuda.synchronize()
        assert mismatches(Y.cpu().numpy(), want) == 0


def test_parts_api_validates_every_part_before_running():
    o = oracle()
    n, batch = 8, 100
    a, b, _, x, y = o.generate_batch(np.float32, 9, n, False, batch)
    X = to_dev(x)
    Y = torch.full((n * n * batch,), 7.0, device="cuda")
    good = kb.Part(0, BV(MV(X, n, n, n), 50, n * n), BV(MV(Y, n, n, n), 50, n * n))
    short = kb.Part(0, BV(MV(X[:n * n * 10], n, n, n), 50, n * n), BV(MV(Y[n * n * 50:], n, n, n), 50, n * n))
    pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    with pytest.raises(ValueError, match=r"part 1: kron2: X: buffer length"):
        kb.kron2_parts(pr, MV(a, n, n, n), MV(b, n, n, n), [good, short])
    assert bool((Y == 7.0).all())  # nothing ran


# -------------------------------------------------------------- staging ----

@pytest.mark.parametrize("beta", [0.0, 1.5])
def test_pageable_staging_multi_chunk_equals_pinned_and_device(beta):
    """A host batch larger than one staging chunk (128 MiB of X+Y: 65,536
    entries at n = 16 fp32), ragged last chunk: pageable (bounce buffers +
    copy pool), pinned (direct DMA) and device-resident runs are
    bit-identical, with beta != 0 exercising the Y upload through the bounce
    buffers."""
    o = oracle()
    n, batch = 16, 200003
    a, b, _, x, y = o.generate_batch(np.float32, 10, n, False, batch)
    pr, _, _ = _kron2_args(n, x, y, batch, 1.0, beta)
    outs = []
    for kind in ("pageable", "pinned", "device", "pageable-sharded"):
        if kind.startswith("pageable"):
            X, Y = x, y.copy()
        elif kind == "pinned":
            X, Y = torch.from_numpy(x).pin_memory(), torch.from_numpy(y.copy()).pin_memory()
        else:
            X, Y = to_dev(x), to_dev(y)
        ex = kb.Exec(devices=[0, 0, 0]) if kind.endswith("sharded") else None
        kb.kron2(pr, MV(a, n, n, n), MV(b, n, n, n), BV(MV(X, n, n, n), batch, n * n), BV(MV(Y, n, n, n), batch, n * n),
                 exec_=ex)
        outs.append(Y if isinstance(Y, np.ndarray) else Y.cpu().numpy())
    want = _ref2(o, np.float32, n, batch, a, b, x, y, 1.0, beta)
    for got in outs:
        assert mismatches(got, want) == 0


def test_pageable_padded_y_padding_untouched_kron3():
    """Padded pageable Y (ld = m+1, entry stride + 5): staged through the
    bounce buffers with its padding round-tripped untouched
    (test_kron3.cpp:316-324)."""
    o = oracle()
    g = rng(33)
    n, batch = 9, 70001
    ld, ld2 = n + 1, (n + 1) * n
    sy = ld2 * n + 5
    a, b, c = (uniform(g, n * n, np.float64) for _ in range(3))
    x = uniform(g, n ** 3 * batch, np.float64)
    y = np.full(sy * batch, -3.25)
    pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    kb.kron3(pr, MV(a, n, n, n), MV(b, n, n, n), MV(c, n, n, n), BV(A3(x, n, n, n, n, n * n), batch, n ** 3),
             BV(A3(y, n, n, n, ld, ld2), batch, sy), kb.Workspace(None, n ** 3 * batch))
    want = np.full(sy * batch, -3.25)
    o.kron3("N", "N", "N", n, n, n, n, n, n, batch, 1.0, a, n, b, n, c, n, x, n, n * n, n ** 3, 0.0, want, ld, ld2, sy)
    assert mismatches(y, want) == 0


# ------------------------------------------------------ CUDA-graph capture ----

@pytest.mark.parametrize("dims3,n,dtype", [(False, 10, np.float32), (False, 13, np.float64), (True, 16, np.float32),
                                           (True, 9, np.float32), (True, 16, np.float64)])
def test_graph_capture_replays_bit_exact(dims3, n, dtype):
    """Calls captured into a CUDA graph on the exec stream (as bench.py's
    configs[0] leg does) replay bit-exactly with NEW X contents: the captured
    kernels (PDL launches, dynamic-tile counters, Y bulk stores) read the
    buffers at replay time; host-resident constants are baked in."""
    o = oracle()
    batch = 301
    a, b, c, x, y = o.generate_batch(dtype, 5, n, dims3, batch)
    e = n ** (3 if dims3 else 2)
    X, Y = to_dev(x), to_dev(np.zeros_like(y))
    s = torch.cuda.Stream()
    ex = kb.Exec(stream=s, asynchronous=True)
    if dims3:
        pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
        args = (pr, MV(a, n, n, n), MV(b, n, n, n), MV(c, n, n, n), BV(A3(X, n, n, n, n, n * n), batch, e),
                BV(A3(Y, n, n, n, n, n * n), batch, e), kb.Workspace(None, e * batch))
        fn = kb.kron3
    else:
        pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
        args = (pr, MV(a, n, n, n), MV(b, n, n, n), BV(MV(X, n, n, n), batch, e), BV(MV(Y, n, n, n), batch, e))
        fn = kb.kron2
    fn(*args, exec_=ex)  # warm-up outside the capture (lane, counters)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(*args, exec_=ex)
        fn(*args, exec_=ex)  # two captured launches back to back (PDL edge inside the graph)
    x2 = uniform(rng(977), x.size, dtype)
    X.copy_(torch.from_numpy(x2))
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    want = np.zeros_like(y)
    if dims3:
        o.kron3("N", "N", "N", n, n, n, n, n, n, batch, dtype(1), a, n, b, n, c, n, x2, n, n * n, e, dtype(0), want, n,
                n * n, e)
    else:
        o.kron2("N", "N", "N", n, n, n, n, batch, dtype(1), a, n, b, n, x2, n, n * n, dtype(0), want, n, n * n)
    assert mismatches(Y.cpu().numpy(), want) == 0


def test_graph_capture_with_device_constants_fails_clearly():
    """Device-resident A/B must be read back (synchronously) to be folded into
    the kernel parameters -- impossible during capture: a clear error instead
    of an invalidated capture deep inside the driver."""
    n, batch = 8, 16
    X = torch.rand(n * n * batch, device="cuda")
    Y = torch.empty_like(X)
    A, B = torch.rand(n * n, device="cuda"), torch.rand(n * n, device="cuda")
    pr, xv, yv = _kron2_args(n, X, Y, batch)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(Exception) as ei:
        with torch.cuda.graph(g, stream=s):
            kb.kron2(pr, MV(A, n, n, n), MV(B, n, n, n), xv, yv, exec_=kb.Exec(stream=s, asynchronous=True))
    assert "capture" in str(ei.value)
    torch.cuda.synchronize()
    # the library (and the device) stay usable afterwards
    kb.kron2(pr, MV(A, n, n, n), MV(B, n, n, n), xv, yv)
    torch.cuda.synchronize()
