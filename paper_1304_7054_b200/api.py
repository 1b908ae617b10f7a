"""Python mirror of the reference ``kronbatch`` operator API, on the sm_100a path.

Same names, argument meaning and error behaviour as the reference C++ API
(``/root/reference/proj/include/kronbatch``), so host code and parity tests read
like the reference's own:

==========================  ==================================================
this module                 reference
==========================  ==================================================
``MatrixOp``, ``op_dims``,  types.hpp:30-45
``is_transposed``
``MatrixView``,             views.hpp:51-170 (non-owning strided column-major
``Array3View``,             views over a flat buffer; ``len`` = addressable
``BatchView``, ``footprint`` elements, default: the buffer's length)
``validate``,               views.hpp:189-240 -- first violated invariant,
``validate_batch``          same message text; ``std::invalid_argument`` ->
                            ``ValueError``
``KronProblem2D/3D``,       kron2.hpp:12-21, kron3.hpp:14-39
``Workspace``
``kron3_workspace_size``    kron3.hpp:43-53 (``std::overflow_error`` ->
                            ``OverflowError``)
``kron2``                   kron2.hpp:37-110
``kron3``                   kron3.hpp:72-166
``kron1``, ``VectorView``   kron1.hpp:17-62, views.hpp:22-46
``gemm_a``                  gemm_a.hpp:18-76
==========================  ==================================================

Buffers are 1-D ``torch.Tensor`` (CUDA or CPU, pinned or pageable) or numpy
arrays of float32/float64. Every call goes through the C ABI of
``libkronbatch_b200.so`` (``include/kronbatch_b200.h``); CPU-resident buffers
are staged through device memory by the library -- the arithmetic always runs
on the GPU. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Any, Optional, Sequence

import numpy as np

from . import _lib

index_t = int


class MatrixOp(str, enum.Enum):
    """BLAS-style op selector; ConjTranspose == Transpose for real types."""

    NoTranspose = "N"
    Transpose = "T"
    ConjTranspose = "C"


def op_dims(op: MatrixOp, stored_rows: int, stored_cols: int):
    return (stored_rows, stored_cols) if MatrixOp(op) == MatrixOp.NoTranspose else (stored_cols, stored_rows)


def is_transposed(op: MatrixOp) -> bool:
    return MatrixOp(op) != MatrixOp.NoTranspose


# ----------------------------------------------------------------- buffers --

_TORCH = None


def _torch():
    """torch, imported once (False when absent); the per-call path must not re-import."""
    global _TORCH
    if _TORCH is None:
        try:
            import torch

            _TORCH = torch
        except ImportError:  # pragma: no cover
            _TORCH = False
    return _TORCH


def _buf_info(data):
    """(address, numel, dtype-name) of a flat buffer; None -> (0, 0, None)."""
    if data is None:
        return 0, 0, None
    torch = _torch()
    if torch and isinstance(data, torch.Tensor):
        dt = data.dtype
        if dt is torch.float32:
            name = "float32"
        elif dt is torch.float64:
            name = "float64"
        else:
            raise TypeError(f"unsupported element type {data.dtype}: float32 or float64 only")
        if not data.is_contiguous():
            raise TypeError("buffer tensors must be contiguous (describe strides with ld / batch_stride)")
        return data.data_ptr(), data.numel(), name
    if isinstance(data, np.ndarray):
        if data.dtype not in (np.float32, np.float64):
            raise TypeError(f"unsupported element type {data.dtype}: float32 or float64 only")
        if not (data.flags.c_contiguous or data.flags.f_contiguous):
            raise TypeError("buffer arrays must be contiguous")
        return data.ctypes.data, data.size, data.dtype.name
    raise TypeError(f"unsupported buffer type {type(data)!r}")


@dataclass
class VectorView:
    """Contiguous vector of ``size`` elements (a kron1 batch entry; views.hpp:22-46)."""

    data: Any
    size: int
    len: Optional[int] = None
    offset: int = 0

    def __post_init__(self):
        if self.len is None:
            self.len = _buf_info(self.data)[1] - self.offset

    def shifted(self, off: int) -> "VectorView":
        return VectorView(self.data, self.size, self.len - off, self.offset + off)


@dataclass
class MatrixView:
    """Column-major matrix: element (i, j) at flat index i + j*ld (views.hpp:51-83)."""

    data: Any
    rows: int
    cols: int
    ld: int
    len: Optional[int] = None
    offset: int = 0  # element offset of (0, 0) into ``data``

    def __post_init__(self):
        if self.len is None:
            self.len = _buf_info(self.data)[1] - self.offset

    def shifted(self, off: int) -> "MatrixView":
        return MatrixView(self.data, self.rows, self.cols, self.ld, self.len - off, self.offset + off)


@dataclass
class Array3View:
    """Column-major 3-D array: (i, j, k) at i + j*ld + k*ld2 (views.hpp:88-126)."""

    data: Any
    dim1: int
    dim2: int
    dim3: int
    ld: int
    ld2: int
    len: Optional[int] = None
    offset: int = 0

    def __post_init__(self):
        if self.len is None:
            self.len = _buf_info(self.data)[1] - self.offset

    def shifted(self, off: int) -> "Array3View":
        return Array3View(self.data, self.dim1, self.dim2, self.dim3, self.ld, self.ld2, self.len - off,
                          self.offset + off)


@dataclass
class BatchView:
    """Uniform-stride batch: entry p starts p*batch_stride after entry 0 (views.hpp:154-170)."""

    base: Any
    batch_count: int = 0
    batch_stride: int = 0

    def entry(self, p: int):
        return self.base.shifted(p * self.batch_stride)


def footprint(v) -> int:
    """Elements an entry occupies (views.hpp:137-148)."""
    if isinstance(v, VectorView):
        return v.size
    if isinstance(v, MatrixView):
        return 0 if v.cols == 0 else v.ld * v.cols
    if isinstance(v, Array3View):
        return 0 if v.dim3 == 0 else v.ld2 * v.dim3
    raise TypeError(type(v))


def _nums(a: int, b: int) -> str:
    return f"({a}) < ({b})"


def _layout_error(context: str, what: str):
    raise ValueError(what if not context else f"{context}: {what}")


def validate(v, context: str = "") -> None:
    """views.hpp:190-223: raises ValueError describing the first violated invariant."""
    if isinstance(v, VectorView):
        if v.size < 0:
            _layout_error(context, "size " + _nums(v.size, 0))
        if v.len < v.size:
            _layout_error(context, "buffer length " + _nums(v.len, v.size))
    elif isinstance(v, MatrixView):
        if v.rows < 0 or v.cols < 0:
            _layout_error(context, "negative rows/cols")
        if v.ld < max(v.rows, 1):
            _layout_error(context, "ld " + _nums(v.ld, max(v.rows, 1)))
        if v.len < footprint(v):
            _layout_error(context, "buffer length " + _nums(v.len, footprint(v)))
    elif isinstance(v, Array3View):
        if v.dim1 < 0 or v.dim2 < 0 or v.dim3 < 0:
            _layout_error(context, "negative dims")
        if v.ld < max(v.dim1, 1):
            _layout_error(context, "ld " + _nums(v.ld, max(v.dim1, 1)))
        if v.ld2 < v.ld * v.dim2:
            _layout_error(context, "ld2 " + _nums(v.ld2, v.ld * v.dim2))
        if v.len < footprint(v):
            _layout_error(context, "buffer length " + _nums(v.len, footprint(v)))
    else:
        raise TypeError(type(v))


def validate_batch(b: BatchView, context: str = "") -> None:
    """views.hpp:225-240."""
    if b.batch_count < 0:
        _layout_error(context, "negative batch_count")
    if b.batch_count == 0:
        return
    validate(b.base, context)
    fp = footprint(b.base)
    if b.batch_stride < fp:
        _layout_error(context, "batch_stride " + _nums(b.batch_stride, fp) + ", batch_stride < entry footprint")
    needed = (b.batch_count - 1) * b.batch_stride + fp
    if b.base.len < needed:
        _layout_error(context, "buffer length " + _nums(b.base.len, needed) + f" for {b.batch_count} entries")


def _require(ok: bool, context: str, what: str):
    if not ok:
        _layout_error(context, what)


def _dim2s(a: int, b: int) -> str:
    return f"{a} x {b}"


# ---------------------------------------------------------------- problems --

@dataclass
class KronProblem2D:
    op_a: MatrixOp = MatrixOp.NoTranspose
    op_b: MatrixOp = MatrixOp.NoTranspose
    op_x: MatrixOp = MatrixOp.NoTranspose
    m_a: int = 0
    n_a: int = 0
    m_b: int = 0
    n_b: int = 0
    alpha: float = 1.0
    beta: float = 0.0


@dataclass
class KronProblem3D:
    op_a: MatrixOp = MatrixOp.NoTranspose
    op_b: MatrixOp = MatrixOp.NoTranspose
    op_c: MatrixOp = MatrixOp.NoTranspose
    m_a: int = 0
    n_a: int = 0
    m_b: int = 0
    n_b: int = 0
    m_c: int = 0
    n_c: int = 0
    alpha: float = 1.0
    beta: float = 0.0


@dataclass
class Workspace:
    """Caller scratch for kron3 (kron3.hpp:29-39): only its capacity is part of
    the contract on the sm_100a path (the intermediate stays on chip)."""

    data: Any = None
    capacity: int = 0

    @classmethod
    def over(cls, buf) -> "Workspace":
        return cls(buf, _buf_info(buf)[1])


def kron3_workspace_size(pr: KronProblem3D, batch_count: int) -> int:
    """m_a*m_b*n_c*batch_count; OverflowError past int64 (kron3.hpp:43-53)."""
    out = C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = _lib.lib.kb_kron3_workspace_size(pr.m_a, pr.m_b, pr.n_c, batch_count, C.byref(out), err, 512)
    _lib.raise_for(rc, err)
    return out.value


# --------------------------------------------------------------- execution --

@dataclass
class Exec:
    """Execution options (kb_exec): devices to shard host-resident batches over,
    a CUDA stream for device-resident calls, async flag."""

    devices: Sequence[int] = field(default_factory=tuple)
    stream: Any = None
    asynchronous: bool = False
    tf32: bool = False  # allow the tcgen05 3xTF32 kernel (fp32 kron3, n = 16): 1e-5 parity, not bit-exact

    def to_c(self):
        """(kb_exec struct, keep-alive) -- cached while the fields are unchanged."""
        key = (tuple(self.devices), self.stream, self.asynchronous, self.tf32)
        cached = self.__dict__.get("_c_cache")
        if cached is not None and cached[0] == key:
            return cached[1], cached[2]
        ex, arr = self._build_c()
        self.__dict__["_c_cache"] = (key, ex, arr)
        return ex, arr

    def _build_c(self):
        arr = (C.c_int32 * max(1, len(self.devices)))(*self.devices) if self.devices else None
        s = self.stream
        if s is not None and hasattr(s, "cuda_stream"):
            s = s.cuda_stream
        ex = _lib.KbExec(len(self.devices), C.cast(arr, C.POINTER(C.c_int32)) if arr is not None else None,
                         C.c_void_p(s) if s else None,
                         (_lib.KB_EXEC_ASYNC if self.asynchronous else 0) | (_lib.KB_EXEC_TF32 if self.tf32 else 0))
        return ex, arr


def _ptr_of(view):
    addr, _, dt = _buf_info(view.data)
    esz = 4 if dt == "float32" else 8
    return (addr + view.offset * esz) if addr else 0, dt


def _ptrs_and_dtype(*views):
    """Element-0 addresses of the views' buffers (0 for none) and their common
    element type -- one _buf_info per buffer."""
    ptrs, dts = [], set()
    for v in views:
        addr, _, dt = _buf_info(v.data)
        if dt is not None:
            dts.add(dt)
        ptrs.append((addr + v.offset * (4 if dt == "float32" else 8)) if addr else 0)
    if len(dts) > 1:
        raise TypeError("all buffers in a kernel call share one element type (float32 or float64)")
    return ptrs, (dts.pop() if dts else "float64")


def _common_dtype(*views):
    return _ptrs_and_dtype(*[v for v in views if v is not None])[1]


_OPCODE = {MatrixOp.NoTranspose: b"N", MatrixOp.Transpose: b"T", MatrixOp.ConjTranspose: b"C"}
_ERR = threading.local()


def _opc(op) -> bytes:
    code = _OPCODE.get(op)
    return code if code is not None else _OPCODE[MatrixOp(op)]


def _call(fn, *args, exec_: Optional[Exec] = None):
    err = getattr(_ERR, "buf", None)
    if err is None:
        err = _ERR.buf = C.create_string_buffer(1024)
    ex_ptr = None
    keep = None
    if exec_ is not None:
        ex, keep = exec_.to_c()
        ex_ptr = C.byref(ex)
    rc = fn(*args, ex_ptr, err, 1024)
    del keep
    if rc:
        _lib.raise_for(rc, err)


def kron2(pr: KronProblem2D, a: MatrixView, b: MatrixView, x: BatchView, y: BatchView,
          exec_: Optional[Exec] = None) -> None:
    """Y^p <- alpha * op(A) * op(X^p) * op(B)^T + beta * Y^p (kron2.hpp:23-110)."""
    validate(a, "kron2: A")
    validate(b, "kron2: B")
    validate_batch(x, "kron2: X")
    validate_batch(y, "kron2: Y")
    ra, ca = op_dims(pr.op_a, a.rows, a.cols)
    rb, cb = op_dims(pr.op_b, b.rows, b.cols)
    if not (ra == pr.m_a and ca == pr.n_a):
        _layout_error("kron2: A", f"op(A) is {_dim2s(ra, ca)}, expected {_dim2s(pr.m_a, pr.n_a)}")
    if not (rb == pr.m_b and cb == pr.n_b):
        _layout_error("kron2: B", f"op(B) is {_dim2s(rb, cb)}, expected {_dim2s(pr.m_b, pr.n_b)}")
    _require(x.batch_count == y.batch_count, "kron2", "X and Y batch_count differ")
    rx, cx = op_dims(pr.op_x, x.base.rows, x.base.cols)
    if not (rx == pr.n_a and cx == pr.n_b):
        _layout_error("kron2: X", f"op(X) is {_dim2s(rx, cx)}, expected {_dim2s(pr.n_a, pr.n_b)}")
    if not (y.base.rows == pr.m_a and y.base.cols == pr.m_b):
        _layout_error("kron2: Y", f"entry is {_dim2s(y.base.rows, y.base.cols)}, expected {_dim2s(pr.m_a, pr.m_b)}")
    (pa, pb, px, py), dt = _ptrs_and_dtype(a, b, x.base, y.base)
    fn = _lib.lib.kb_skron2 if dt == "float32" else _lib.lib.kb_dkron2
    _call(fn, _opc(pr.op_a), _opc(pr.op_b), _opc(pr.op_x),
          pr.m_a, pr.n_a, pr.m_b, pr.n_b, x.batch_count, pr.alpha, pa or None, a.ld, a.len, pb or None, b.ld, b.len,
          px or None, x.base.ld, x.batch_stride, x.base.len, pr.beta, py or None, y.base.ld, y.batch_stride,
          y.base.len, exec_=exec_)


def kron3(pr: KronProblem3D, a: MatrixView, b: MatrixView, c: MatrixView, x: BatchView, y: BatchView,
          work: Workspace, exec_: Optional[Exec] = None) -> None:
    """vec(Y^p) <- alpha * (op(C) (x) op(B) (x) op(A)) vec(X^p) + beta vec(Y^p) (kron3.hpp:55-166)."""
    validate(a, "kron3: A")
    validate(b, "kron3: B")
    validate(c, "kron3: C")
    validate_batch(x, "kron3: X")
    validate_batch(y, "kron3: Y")
    ra, ca = op_dims(pr.op_a, a.rows, a.cols)
    rb, cb = op_dims(pr.op_b, b.rows, b.cols)
    rc, cc = op_dims(pr.op_c, c.rows, c.cols)
    if not (ra == pr.m_a and ca == pr.n_a):
        _layout_error("kron3: A", f"op(A) is {_dim2s(ra, ca)}, expected {_dim2s(pr.m_a, pr.n_a)}")
    if not (rb == pr.m_b and cb == pr.n_b):
        _layout_error("kron3: B", f"op(B) is {_dim2s(rb, cb)}, expected {_dim2s(pr.m_b, pr.n_b)}")
    if not (rc == pr.m_c and cc == pr.n_c):
        _layout_error("kron3: C", f"op(C) is {_dim2s(rc, cc)}, expected {_dim2s(pr.m_c, pr.n_c)}")
    _require(x.batch_count == y.batch_count, "kron3", "X and Y batch_count differ")
    _require(x.base.dim1 == pr.n_a and x.base.dim2 == pr.n_b and x.base.dim3 == pr.n_c, "kron3: X",
             "entry dims do not match n_a x n_b x n_c")
    _require(y.base.dim1 == pr.m_a and y.base.dim2 == pr.m_b and y.base.dim3 == pr.m_c, "kron3: Y",
             "entry dims do not match m_a x m_b x m_c")
    (pa, pb, pc, px, py), dt = _ptrs_and_dtype(a, b, c, x.base, y.base)
    fn = _lib.lib.kb_skron3 if dt == "float32" else _lib.lib.kb_dkron3
    wp = _buf_info(work.data)[0] if work.data is not None else 0
    _call(fn, _opc(pr.op_a), _opc(pr.op_b), _opc(pr.op_c),
          pr.m_a, pr.n_a, pr.m_b, pr.n_b, pr.m_c, pr.n_c, x.batch_count, pr.alpha, pa or None, a.ld, a.len,
          pb or None, b.ld, b.len, pc or None, c.ld, c.len, px or None, x.base.ld, x.base.ld2, x.batch_stride,
          x.base.len, pr.beta, py or None, y.base.ld, y.base.ld2, y.batch_stride, y.base.len, wp or None,
          work.capacity, exec_=exec_)


def kron1(op_a, m_a: int, n_a: int, alpha, a: MatrixView, x: BatchView, beta, y: BatchView,
          exec_: Optional[Exec] = None) -> None:
    """y^p <- alpha * op(A) * x^p + beta * y^p (kron1.hpp:9-62): a batched GEMV
    with A shared across the batch; x, y are batches of VectorView."""
    validate(a, "kron1: A")
    validate_batch(x, "kron1: X")
    validate_batch(y, "kron1: Y")
    ra, ca = op_dims(op_a, a.rows, a.cols)
    if not (ra == m_a and ca == n_a):
        _layout_error("kron1: A", f"op(A) is {_dim2s(ra, ca)}, expected {_dim2s(m_a, n_a)}")
    _require(x.batch_count == y.batch_count, "kron1", "X and Y batch_count differ")
    if x.base.size != n_a:
        _layout_error("kron1: X", f"entry length {x.base.size}, expected {n_a}")
    if y.base.size != m_a:
        _layout_error("kron1: Y", f"entry length {y.base.size}, expected {m_a}")
    (pa, px, py), dt = _ptrs_and_dtype(a, x.base, y.base)
    fn = _lib.lib.kb_skron1 if dt == "float32" else _lib.lib.kb_dkron1
    _call(fn, _opc(op_a), m_a, n_a, x.batch_count, alpha, pa or None, a.ld, a.len, px or None, x.batch_stride,
          x.base.len, beta, py or None, y.batch_stride, y.base.len, exec_=exec_)


def gemm_a(op_a, op_b, m: int, n: int, k: int, alpha, a: BatchView, b: MatrixView, beta, c: BatchView,
           parallel_hint: int = 0, exec_: Optional[Exec] = None) -> None:
    """C^p <- alpha * op(A^p) * op(B) + beta * C^p (gemm_a.hpp:9-76): a batched
    GEMM with the left matrix varying and B shared. ``parallel_hint`` (a CPU
    worker-chunk hint in the reference) does not change results and is ignored."""
    validate_batch(a, "gemm_a: A")
    validate(b, "gemm_a: B")
    validate_batch(c, "gemm_a: C")
    ram, rak = op_dims(op_a, a.base.rows, a.base.cols)
    rbk, rbn = op_dims(op_b, b.rows, b.cols)
    _require(a.batch_count == c.batch_count, "gemm_a", "A and C batch_count differ")
    if not (ram == m and rak == k):
        _layout_error("gemm_a: A", f"op(A) is {_dim2s(ram, rak)}, expected {_dim2s(m, k)}")
    if not (rbk == k and rbn == n):
        _layout_error("gemm_a: B", f"op(B) is {_dim2s(rbk, rbn)}, expected {_dim2s(k, n)}")
    if not (c.base.rows == m and c.base.cols == n):
        _layout_error("gemm_a: C", f"entry is {_dim2s(c.base.rows, c.base.cols)}, expected {_dim2s(m, n)}")
    (pa, pb, pc), dt = _ptrs_and_dtype(a.base, b, c.base)
    fn = _lib.lib.kb_sgemm_a if dt == "float32" else _lib.lib.kb_dgemm_a
    _call(fn, _opc(op_a), _opc(op_b), m, n, k, a.batch_count, alpha, pa or None, a.base.ld, a.batch_stride,
          a.base.len, pb or None, b.ld, b.len, beta, pc or None, c.base.ld, c.batch_stride, c.base.len, exec_=exec_)


# -------------------------------------------------- multi-device parts ----

@dataclass
class Part:
    """One part of a batch split over GPUs (kb_part): the part's X / Y batch
    views (same entry layout in every part), the GPU that runs it (where its
    device buffers live) and an optional CUDA stream on that GPU."""

    device: int
    x: BatchView
    y: BatchView
    stream: Any = None


def _parts_c(parts: Sequence[Part], ctx: str):
    if not parts:
        return (_lib.KbPart * 1)(), 0, []
    x0, y0 = parts[0].x, parts[0].y
    arr = (_lib.KbPart * len(parts))()
    ptrs = []
    for i, p in enumerate(parts):
        for v, v0, nm in ((p.x, x0, "X"), (p.y, y0, "Y")):
            same = (type(v.base) is type(v0.base) and v.batch_stride == v0.batch_stride and
                    getattr(v.base, "ld", None) == getattr(v0.base, "ld", None) and
                    getattr(v.base, "ld2", None) == getattr(v0.base, "ld2", None))
            if not same:
                _layout_error(ctx, f"part {i}: {nm} entry layout differs from part 0")
        _require(p.x.batch_count == p.y.batch_count, ctx, f"part {i}: X and Y batch_count differ")
        (px, py), dt = _ptrs_and_dtype(p.x.base, p.y.base)
        ptrs.append(dt)
        s = p.stream
        if s is not None and hasattr(s, "cuda_stream"):
            s = s.cuda_stream
        arr[i] = _lib.KbPart(int(p.device), int(p.x.batch_count), px or None, int(p.x.base.len), py or None,
                             int(p.y.base.len), C.c_void_p(s) if s else None)
    if len(set(ptrs)) > 1:
        raise TypeError("all parts share one element type")
    return arr, len(parts), ptrs


def _parts_call(fn, *args, nparts, arr, asynchronous):
    err = getattr(_ERR, "buf", None)
    if err is None:
        err = _ERR.buf = C.create_string_buffer(1024)
    rc = fn(*args, nparts, arr, _lib.KB_EXEC_ASYNC if asynchronous else 0, err, 1024)
    if rc:
        _lib.raise_for(rc, err)


def kron2_parts(pr: KronProblem2D, a: MatrixView, b: MatrixView, parts: Sequence[Part],
                asynchronous: bool = False) -> None:
    """kron2 over a batch already split across GPUs (kb_?kron2_parts): every part
    validated first, then all parts run concurrently, one per device, with no
    collective; returns when all are done (or all are queued, asynchronous)."""
    arr, n, dts = _parts_c(parts, "kron2")
    if n == 0:
        return
    x0, y0 = parts[0].x, parts[0].y
    kron2(pr, a, b, BatchView(x0.base, 0, x0.batch_stride), BatchView(y0.base, 0, y0.batch_stride))  # shape checks
    (pa, pb), _ = _ptrs_and_dtype(a, b)
    fn = _lib.lib.kb_skron2_parts if dts[0] == "float32" else _lib.lib.kb_dkron2_parts
    _parts_call(fn, _opc(pr.op_a), _opc(pr.op_b), _opc(pr.op_x), pr.m_a, pr.n_a, pr.m_b, pr.n_b, pr.alpha,
                pa or None, a.ld, a.len, pb or None, b.ld, b.len, x0.base.ld, x0.batch_stride, pr.beta, y0.base.ld,
                y0.batch_stride, nparts=n, arr=arr, asynchronous=asynchronous)


def kron3_parts(pr: KronProblem3D, a: MatrixView, b: MatrixView, c: MatrixView, parts: Sequence[Part],
                asynchronous: bool = False) -> None:
    """kron3 over a batch already split across GPUs (kb_?kron3_parts); no
    workspace (the sm_100a path never uses one)."""
    arr, n, dts = _parts_c(parts, "kron3")
    if n == 0:
        return
    x0, y0 = parts[0].x, parts[0].y
    kron3(pr, a, b, c, BatchView(x0.base, 0, x0.batch_stride), BatchView(y0.base, 0, y0.batch_stride),
          Workspace(None, 0))  # shape checks (batch 0: nothing runs)
    (pa, pb, pc), _ = _ptrs_and_dtype(a, b, c)
    fn = _lib.lib.kb_skron3_parts if dts[0] == "float32" else _lib.lib.kb_dkron3_parts
    _parts_call(fn, _opc(pr.op_a), _opc(pr.op_b), _opc(pr.op_c), pr.m_a, pr.n_a, pr.m_b, pr.n_b, pr.m_c, pr.n_c,
                pr.alpha, pa or None, a.ld, a.len, pb or None, b.ld, b.len, pc or None, c.ld, c.len, x0.base.ld,
                x0.base.ld2, x0.batch_stride, pr.beta, y0.base.ld, y0.base.ld2, y0.batch_stride, nparts=n, arr=arr,
                asynchronous=asynchronous)


def pooled_bytes(device: int = -1) -> int:
    """Device bytes held by the library's buffer pool (idle lanes) on `device` (-1: all)."""
    return int(_lib.lib.kb_pooled_bytes(device))


def launch_count() -> int:
    """Kernels this process has launched through libkronbatch_b200 (all devices)."""
    return int(_lib.lib.kb_launch_count())


def last_path() -> str:
    """Kernel family the calling thread's last call used (kron2_fast, kron3_generic, ...)."""
    return _lib.lib.kb_last_path().decode()


def version() -> str:
    return _lib.lib.kb_version().decode()


def release_buffers() -> None:
    _lib.lib.kb_release_buffers()
