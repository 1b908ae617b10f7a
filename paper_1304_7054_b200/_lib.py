"""ctypes binding of the C ABI in ``include/kronbatch_b200.h``.

Loads the in-tree ``libkronbatch_b200.so`` (built by ``make lib`` /
``__graft_entry__.build()``). There is deliberately no fallback: if the
library is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# KB_LIB_PATH: load an alternative in-tree build (A/B kernel experiments under tools/)
LIB_PATH = os.environ.get("KB_LIB_PATH") or os.path.join(HERE, "libkronbatch_b200.so")

KB_OK, KB_EINVAL, KB_EOVERFLOW, KB_ECUDA, KB_ENOMEM, KB_EINTERNAL = range(6)
KB_EXEC_ASYNC = 0x1
KB_EXEC_TF32 = 0x2

ABI_SYMBOLS = (
    "kb_skron2",
    "kb_dkron2",
    "kb_skron3",
    "kb_dkron3",
    "kb_kron3_workspace_size",
    "kb_skron1",
    "kb_dkron1",
    "kb_sgemm_a",
    "kb_dgemm_a",
    "kb_version",
    "kb_launch_count",
    "kb_last_path",
    "kb_release_buffers",
    "kb_pooled_bytes",
    "kb_skron2_parts",
    "kb_dkron2_parts",
    "kb_skron3_parts",
    "kb_dkron3_parts",
)


class KbExec(C.Structure):
    _fields_ = [
        ("ndevices", C.c_int32),
        ("devices", C.POINTER(C.c_int32)),
        ("stream", C.c_void_p),
        ("flags", C.c_uint32),
    ]


class KbPart(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("batch_count", C.c_int64),
        ("X", C.c_void_p),
        ("lenx", C.c_int64),
        ("Y", C.c_void_p),
        ("leny", C.c_int64),
        ("stream", C.c_void_p),
    ]


class KronbatchLibraryError(ImportError):
    pass


def _load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise KronbatchLibraryError(
            f"{path} is missing: build the sm_100a library first (`make lib` or __graft_entry__.build()). "
            "There is no CPU fallback.")
    lib = C.CDLL(path)
    i64, vp, ch = C.c_int64, C.c_void_p, C.c_char
    for name, T in (("kb_skron2", C.c_float), ("kb_dkron2", C.c_double)):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [ch, ch, ch, i64, i64, i64, i64, i64, T, vp, i64, i64, vp, i64, i64, vp, i64, i64, i64, T, vp,
                      i64, i64, i64, C.POINTER(KbExec), C.c_char_p, C.c_size_t]
    for name, T in (("kb_skron3", C.c_float), ("kb_dkron3", C.c_double)):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [ch, ch, ch, i64, i64, i64, i64, i64, i64, i64, T, vp, i64, i64, vp, i64, i64, vp, i64, i64, vp,
                      i64, i64, i64, i64, T, vp, i64, i64, i64, i64, vp, i64, C.POINTER(KbExec), C.c_char_p,
                      C.c_size_t]
    for name, T in (("kb_skron1", C.c_float), ("kb_dkron1", C.c_double)):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [ch, i64, i64, i64, T, vp, i64, i64, vp, i64, i64, T, vp, i64, i64, C.POINTER(KbExec),
                      C.c_char_p, C.c_size_t]
    for name, T in (("kb_sgemm_a", C.c_float), ("kb_dgemm_a", C.c_double)):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [ch, ch, i64, i64, i64, i64, T, vp, i64, i64, i64, vp, i64, i64, T, vp, i64, i64, i64,
                      C.POINTER(KbExec), C.c_char_p, C.c_size_t]
    u32, i32 = C.c_uint32, C.c_int32
    for name, T in (("kb_skron2_parts", C.c_float), ("kb_dkron2_parts", C.c_double)):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [ch, ch, ch, i64, i64, i64, i64, T, vp, i64, i64, vp, i64, i64, i64, i64, T, i64, i64, i32,
                      C.POINTER(KbPart), u32, C.c_char_p, C.c_size_t]
    for name, T in (("kb_skron3_parts", C.c_float), ("kb_dkron3_parts", C.c_double)):
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = [ch, ch, ch, i64, i64, i64, i64, i64, i64, T, vp, i64, i64, vp, i64, i64, vp, i64, i64, i64, i64,
                      i64, T, i64, i64, i64, i32, C.POINTER(KbPart), u32, C.c_char_p, C.c_size_t]
    lib.kb_pooled_bytes.restype = C.c_uint64
    lib.kb_pooled_bytes.argtypes = [C.c_int]
    lib.kb_kron3_workspace_size.restype = C.c_int
    lib.kb_kron3_workspace_size.argtypes = [i64, i64, i64, i64, C.POINTER(i64), C.c_char_p, C.c_size_t]
    lib.kb_version.restype = C.c_char_p
    lib.kb_launch_count.restype = C.c_uint64
    lib.kb_last_path.restype = C.c_char_p
    lib.kb_release_buffers.restype = None
    return lib


lib = _load()


def raise_for(rc: int, err) -> None:
    if rc == KB_OK:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    if rc == KB_EINVAL:
        raise ValueError(msg)
    if rc == KB_EOVERFLOW:
        raise OverflowError(msg)
    if rc == KB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg or f"kronbatch_b200 error {rc}")
