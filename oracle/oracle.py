"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers built by ``oracle/Makefile``:

* ``Oracle`` -> ``oracle/liboracle.so``: the plain-C restatement of the
  reference algorithm (``oracle/kron_oracle.c``; every function there cites the
  reference file:line it restates).
* ``Reference`` -> ``oracle/_ref/libkronref.so``: the unmodified reference
  library (``/root/reference/proj``) compiled from its own sources plus
  ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module, and only as the checker / the CPU baseline -- never as the
thing shipped. The product (``paper_1304_7054_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkronref.so")
REF_BLAS_SO = os.path.join(HERE, "_ref", "libkronref_blas.so")

i64 = C.c_int64
vp = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(vp)


def _op(c):
    return C.c_char(c.encode() if isinstance(c, str) else c)


def build():
    """Compile the checkers (liboracle.so; _ref when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class Oracle:
    """The C restatement (``kron_oracle.c``)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        for name, T in (("ko_skron2", C.c_float), ("ko_dkron2", C.c_double)):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = [C.c_char] * 3 + [i64] * 5 + [T, vp, i64, vp, i64, vp, i64, i64, T, vp, i64, i64]
        for name, T in (("ko_skron3", C.c_float), ("ko_dkron3", C.c_double)):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = ([C.c_char] * 3 + [i64] * 7 + [T, vp, i64, vp, i64, vp, i64, vp, i64, i64, i64, T,
                                                       vp, i64, i64, i64])
        for name, T in (("ko_skron1", C.c_float), ("ko_dkron1", C.c_double)):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = [C.c_char, i64, i64, i64, T, vp, i64, vp, i64, T, vp, i64]
        for name, T in (("ko_sgemm_a", C.c_float), ("ko_dgemm_a", C.c_double)):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = [C.c_char, C.c_char, i64, i64, i64, i64, T, vp, i64, i64, vp, i64, T, vp, i64, i64]
        L.ko_generate_batch_f32.argtypes = [C.c_uint64, C.c_int, C.c_int, i64] + [vp] * 5
        L.ko_generate_batch_f64.argtypes = [C.c_uint64, C.c_int, C.c_int, i64] + [vp] * 5
        L.ko_set_fused.argtypes = [C.c_int]
        L.ko_get_fused.restype = C.c_int
        L.ko_kron3_workspace_size.argtypes = [i64, i64, i64, i64, C.POINTER(i64)]
        L.ko_kron3_workspace_size.restype = C.c_int
        L.ko_ref_kron2_apply.argtypes = [i64] * 4 + [vp] * 4
        L.ko_ref_kron3_apply.argtypes = [i64] * 6 + [vp] * 5
        L.ko_kron_matrix.argtypes = [i64, i64, vp, i64, i64, vp, vp]
        L.ko_flops_kron.argtypes = [C.c_int, C.c_int]
        L.ko_flops_kron.restype = C.c_int64
        L.ko_problem_bytes.argtypes = [C.c_int, C.c_int, C.c_int, i64]
        L.ko_problem_bytes.restype = C.c_uint64
        L.ko_rel_err_inf.argtypes = [i64, vp, vp]
        L.ko_rel_err_inf.restype = C.c_double
        L.ko_random_vec_f64.argtypes = [C.c_uint64, i64, vp]

    # -- contraction rule --------------------------------------------------
    def set_fused(self, fused: bool):
        self.lib.ko_set_fused(1 if fused else 0)

    # -- generator ---------------------------------------------------------
    def generate_batch(self, dtype, seed: int, m: int, dims3: bool, batch: int):
        dt = np.dtype(dtype)
        mm = m * m
        entry = mm * m if dims3 else mm
        a = np.empty(mm, dt)
        b = np.empty(mm, dt)
        c = np.empty(mm if dims3 else 0, dt)
        x = np.empty(entry * batch, dt)
        y = np.empty(entry * batch, dt)
        f = self.lib.ko_generate_batch_f32 if dt == np.float32 else self.lib.ko_generate_batch_f64
        f(seed, m, 1 if dims3 else 0, batch, _ptr(a), _ptr(b), _ptr(c) if dims3 else None, _ptr(x), _ptr(y))
        return a, b, c, x, y

    def random_vec(self, seed: int, n: int):
        out = np.empty(n, np.float64)
        self.lib.ko_random_vec_f64(seed, n, _ptr(out))
        return out

    # -- CPU path restatement ----------------------------------------------
    def kron2(self, opa, opb, opx, m_a, n_a, m_b, n_b, batch, alpha, A, lda, B, ldb, X, ldx, sx, beta, Y, ldy, sy):
        f = self.lib.ko_skron2 if Y.dtype == np.float32 else self.lib.ko_dkron2
        f(_op(opa), _op(opb), _op(opx), m_a, n_a, m_b, n_b, batch, alpha, _ptr(A), lda, _ptr(B), ldb, _ptr(X), ldx,
          sx, beta, _ptr(Y), ldy, sy)

    def kron3(self, opa, opb, opc, m_a, n_a, m_b, n_b, m_c, n_c, batch, alpha, A, lda, B, ldb, Cm, ldc, X, ldx, ldx2,
              sx, beta, Y, ldy, ldy2, sy):
        f = self.lib.ko_skron3 if Y.dtype == np.float32 else self.lib.ko_dkron3
        f(_op(opa), _op(opb), _op(opc), m_a, n_a, m_b, n_b, m_c, n_c, batch, alpha, _ptr(A), lda, _ptr(B), ldb,
          _ptr(Cm), ldc, _ptr(X), ldx, ldx2, sx, beta, _ptr(Y), ldy, ldy2, sy)

    def kron1(self, opa, m_a, n_a, batch, alpha, A, lda, X, sx, beta, Y, sy):
        """kron1.hpp:17-62 restated (x entries contiguous n_a at p*sx, y m_a at p*sy)."""
        f = self.lib.ko_skron1 if Y.dtype == np.float32 else self.lib.ko_dkron1
        f(_op(opa), m_a, n_a, batch, alpha, _ptr(A), lda, _ptr(X), sx, beta, _ptr(Y), sy)

    def gemm_a(self, opa, opb, m, n, k, batch, alpha, A, lda, sa, B, ldb, beta, Cm, ldc, sc):
        """gemm_a.hpp:18-76 restated (A^p at p*sa, C^p at p*sc)."""
        f = self.lib.ko_sgemm_a if Cm.dtype == np.float32 else self.lib.ko_dgemm_a
        f(_op(opa), _op(opb), m, n, k, batch, alpha, _ptr(A), lda, sa, _ptr(B), ldb, beta, _ptr(Cm), ldc, sc)

    def kron3_workspace_size(self, m_a, m_b, n_c, batch):
        out = i64(0)
        rc = self.lib.ko_kron3_workspace_size(m_a, m_b, n_c, batch, C.byref(out))
        if rc == -1:
            raise ValueError("kron3_workspace_size: negative dimension")
        if rc == -2:
            raise OverflowError("kron3_workspace_size: m_a*m_b*n_c*batch_count overflows")
        return out.value

    # -- brute-force double oracle -----------------------------------------
    def ref_kron2_apply(self, A, B, X):
        """A (m_a x n_a), B (m_b x n_b), X (n_a x n_b) as Fortran-order 2-D float64 arrays."""
        A, B, X = (np.asfortranarray(v, dtype=np.float64) for v in (A, B, X))
        Y = np.empty((A.shape[0], B.shape[0]), np.float64, order="F")
        self.lib.ko_ref_kron2_apply(A.shape[0], A.shape[1], B.shape[0], B.shape[1], _ptr(A), _ptr(B), _ptr(X),
                                    _ptr(Y))
        return Y

    def ref_kron3_apply(self, A, B, Cm, X):
        A, B, Cm, X = (np.asfortranarray(v, dtype=np.float64) for v in (A, B, Cm, X))
        Y = np.empty((A.shape[0], B.shape[0], Cm.shape[0]), np.float64, order="F")
        self.lib.ko_ref_kron3_apply(A.shape[0], A.shape[1], B.shape[0], B.shape[1], Cm.shape[0], Cm.shape[1],
                                    _ptr(A), _ptr(B), _ptr(Cm), _ptr(X), _ptr(Y))
        return Y

    def kron_matrix(self, A, B):
        A, B = (np.asfortranarray(v, dtype=np.float64) for v in (A, B))
        K = np.empty((A.shape[0] * B.shape[0], A.shape[1] * B.shape[1]), np.float64, order="F")
        self.lib.ko_kron_matrix(A.shape[0], A.shape[1], _ptr(A), B.shape[0], B.shape[1], _ptr(B), _ptr(K))
        return K

    def flops_kron(self, m, dims3):
        r = self.lib.ko_flops_kron(m, 1 if dims3 else 0)
        if r < 0:
            raise ValueError("flops_kron: size must be >= 1")
        return r

    def problem_bytes(self, m, dims3, dbl, batch):
        return self.lib.ko_problem_bytes(m, 1 if dims3 else 0, 1 if dbl else 0, batch)

    @staticmethod
    def rel_err_inf(got, want):
        """max|got - want| / max(1, max|want|)  (tests/test_util.hpp:93-103)."""
        got = np.asarray(got, np.float64).ravel()
        want = np.asarray(want, np.float64).ravel()
        if want.size == 0:
            return 0.0
        d = np.abs(got - want)
        err = np.inf if np.isnan(d).any() else float(d.max())
        return err / max(1.0, float(np.abs(want).max()))


class RefError(Exception):
    pass


class Reference:
    """The unmodified reference library (``oracle/_ref/libkronref.so``)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle ref` where /root/reference exists)")
        L = self.lib = C.CDLL(path)
        for name, T in (("kbref_skron2", C.c_float), ("kbref_dkron2", C.c_double)):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = ([C.c_char] * 3 + [i64] * 5 + [T, vp, i64, i64, i64, i64, vp, i64, i64, i64, i64, vp, i64,
                                                       i64, i64, i64, i64, T, vp, i64, i64, i64, i64, i64, vp,
                                                       C.c_size_t])
        for name, T in (("kbref_skron3", C.c_float), ("kbref_dkron3", C.c_double)):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = ([C.c_char] * 3 + [i64] * 7 + [T] + [vp, i64, i64, i64, i64] * 3 +
                          [vp, i64, i64, i64, i64, i64, i64, i64, T, vp, i64, i64, i64, i64, i64, i64, i64, vp, i64,
                           vp, C.c_size_t])
        # kron1 / gemm_a live in their own library (ref_shim_blas.cpp explains why)
        BL = self.blas = C.CDLL(REF_BLAS_SO) if os.path.exists(REF_BLAS_SO) else None
        for name, T in ((("kbref_skron1", C.c_float), ("kbref_dkron1", C.c_double)) if BL else ()):
            f = getattr(BL, name)
            f.restype = C.c_int
            f.argtypes = [C.c_char, i64, i64, T, vp, i64, i64, i64, i64, vp, i64, i64, i64, i64, T, vp, i64, i64, i64,
                          vp, C.c_size_t]
        for name, T in ((("kbref_sgemm_a", C.c_float), ("kbref_dgemm_a", C.c_double)) if BL else ()):
            f = getattr(BL, name)
            f.restype = C.c_int
            f.argtypes = ([C.c_char, C.c_char, i64, i64, i64, T, vp, i64, i64, i64, i64, i64, i64, vp, i64, i64, i64,
                           i64, T, vp, i64, i64, i64, i64, i64, i64, vp, C.c_size_t])
        L.kbref_generate_batch_f32.argtypes = [C.c_uint64, C.c_int, C.c_int, i64] + [vp] * 5
        L.kbref_generate_batch_f64.argtypes = [C.c_uint64, C.c_int, C.c_int, i64] + [vp] * 5
        L.kbref_has_openmp.restype = C.c_int
        L.kbref_max_threads.restype = C.c_int
        L.kbref_set_threads.argtypes = [C.c_int]
        L.kbref_kron3_workspace_size.argtypes = [i64, i64, i64, i64, C.POINTER(i64), vp, C.c_size_t]
        L.kbref_flops_kron.argtypes = [C.c_int, C.c_int]
        L.kbref_flops_kron.restype = C.c_int64
        L.kbref_problem_bytes.argtypes = [C.c_int, C.c_int, C.c_int, i64]
        L.kbref_problem_bytes.restype = C.c_uint64
        L.kbref_ref_kron2_apply.argtypes = [i64] * 4 + [vp] * 4
        L.kbref_ref_kron3_apply.argtypes = [i64] * 6 + [vp] * 5
        L.kbref_kron_matrix.argtypes = [i64, i64, vp, i64, i64, vp, vp]

    @property
    def has_openmp(self):
        return bool(self.lib.kbref_has_openmp())

    @property
    def max_threads(self):
        return self.lib.kbref_max_threads()

    def set_threads(self, n):
        self.lib.kbref_set_threads(n)

    def _raise(self, rc, err):
        msg = err.value.decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise OverflowError(msg)
        raise RefError(msg)

    def generate_batch(self, dtype, seed, m, dims3, batch):
        dt = np.dtype(dtype)
        mm = m * m
        entry = mm * m if dims3 else mm
        a, b = np.empty(mm, dt), np.empty(mm, dt)
        c = np.empty(mm if dims3 else 0, dt)
        x, y = np.empty(entry * batch, dt), np.empty(entry * batch, dt)
        f = self.lib.kbref_generate_batch_f32 if dt == np.float32 else self.lib.kbref_generate_batch_f64
        f(seed, m, 1 if dims3 else 0, batch, _ptr(a), _ptr(b), _ptr(c) if dims3 else None, _ptr(x), _ptr(y))
        return a, b, c, x, y

    def kron2(self, opa, opb, opx, m_a, n_a, m_b, n_b, batch, alpha, A, a_shape, lda, B, b_shape, ldb, X, x_shape,
              ldx, sx, beta, Y, y_shape, ldy, sy, lens=None):
        """Calls kronbatch::kron2<T> with views built over the given arrays
        (len = array size unless ``lens`` overrides (lena, lenb, lenx, leny))."""
        err = C.create_string_buffer(512)
        la, lb, lx, ly = lens if lens is not None else (A.size, B.size, X.size, Y.size)
        f = self.lib.kbref_skron2 if Y.dtype == np.float32 else self.lib.kbref_dkron2
        rc = f(_op(opa), _op(opb), _op(opx), m_a, n_a, m_b, n_b, batch, alpha, _ptr(A), a_shape[0], a_shape[1], lda,
               la, _ptr(B), b_shape[0], b_shape[1], ldb, lb, _ptr(X), x_shape[0], x_shape[1], ldx, sx, lx, beta,
               _ptr(Y), y_shape[0], y_shape[1], ldy, sy, ly, err, 512)
        if rc:
            self._raise(rc, err)

    def kron3(self, opa, opb, opc, m_a, n_a, m_b, n_b, m_c, n_c, batch, alpha, A, a_shape, lda, B, b_shape, ldb, Cm,
              c_shape, ldc, X, x_dims, ldx, ldx2, sx, beta, Y, y_dims, ldy, ldy2, sy, work, work_cap=None,
              lens=None):
        err = C.create_string_buffer(512)
        la, lb, lc, lx, ly = lens if lens is not None else (A.size, B.size, Cm.size, X.size, Y.size)
        if work_cap is None:
            work_cap = 0 if work is None else work.size
        f = self.lib.kbref_skron3 if Y.dtype == np.float32 else self.lib.kbref_dkron3
        rc = f(_op(opa), _op(opb), _op(opc), m_a, n_a, m_b, n_b, m_c, n_c, batch, alpha, _ptr(A), a_shape[0],
               a_shape[1], lda, la, _ptr(B), b_shape[0], b_shape[1], ldb, lb, _ptr(Cm), c_shape[0], c_shape[1], ldc,
               lc, _ptr(X), x_dims[0], x_dims[1], x_dims[2], ldx, ldx2, sx, lx, beta, _ptr(Y), y_dims[0], y_dims[1],
               y_dims[2], ldy, ldy2, sy, ly, _ptr(work), work_cap, err, 512)
        if rc:
            self._raise(rc, err)

    def kron3_workspace_size(self, m_a, m_b, n_c, batch):
        out = i64(0)
        err = C.create_string_buffer(512)
        rc = self.lib.kbref_kron3_workspace_size(m_a, m_b, n_c, batch, C.byref(out), err, 512)
        if rc:
            self._raise(rc, err)
        return out.value

    def flops_kron(self, m, dims3):
        return self.lib.kbref_flops_kron(m, 1 if dims3 else 0)

    def problem_bytes(self, m, dims3, dbl, batch):
        return self.lib.kbref_problem_bytes(m, 1 if dims3 else 0, 1 if dbl else 0, batch)

    def ref_kron2_apply(self, A, B, X):
        A, B, X = (np.asfortranarray(v, dtype=np.float64) for v in (A, B, X))
        Y = np.empty((A.shape[0], B.shape[0]), np.float64, order="F")
        self.lib.kbref_ref_kron2_apply(A.shape[0], A.shape[1], B.shape[0], B.shape[1], _ptr(A), _ptr(B), _ptr(X),
                                       _ptr(Y))
        return Y

    def ref_kron3_apply(self, A, B, Cm, X):
        A, B, Cm, X = (np.asfortranarray(v, dtype=np.float64) for v in (A, B, Cm, X))
        Y = np.empty((A.shape[0], B.shape[0], Cm.shape[0]), np.float64, order="F")
        self.lib.kbref_ref_kron3_apply(A.shape[0], A.shape[1], B.shape[0], B.shape[1], Cm.shape[0], Cm.shape[1],
                                       _ptr(A), _ptr(B), _ptr(Cm), _ptr(X), _ptr(Y))
        return Y

    def kron_matrix(self, A, B):
        A, B = (np.asfortranarray(v, dtype=np.float64) for v in (A, B))
        K = np.empty((A.shape[0] * B.shape[0], A.shape[1] * B.shape[1]), np.float64, order="F")
        self.lib.kbref_kron_matrix(A.shape[0], A.shape[1], _ptr(A), B.shape[0], B.shape[1], _ptr(B), _ptr(K))
        return K

    def kron1(self, opa, m_a, n_a, alpha, A, a_shape, lda, X, x_size, sx, batch, beta, Y, y_size, sy, lens=None):
        """kronbatch::kron1<T> over views of the given arrays (proj/include/kronbatch/kron1.hpp:17-62)."""
        err = C.create_string_buffer(512)
        la, lx, ly = lens if lens is not None else (A.size, X.size, Y.size)
        f = self.blas.kbref_skron1 if Y.dtype == np.float32 else self.blas.kbref_dkron1
        rc = f(_op(opa), m_a, n_a, alpha, _ptr(A), a_shape[0], a_shape[1], lda, la, _ptr(X), x_size, sx, lx, batch,
               beta, _ptr(Y), y_size, sy, ly, err, 512)
        if rc:
            self._raise(rc, err)

    def gemm_a(self, opa, opb, m, n, k, alpha, A, a_shape, lda, sa, batch, B, b_shape, ldb, beta, Cm, c_shape, ldc, sc,
               hint=0, lens=None):
        """kronbatch::gemm_a<T> over views of the given arrays (proj/include/kronbatch/gemm_a.hpp:18-76)."""
        err = C.create_string_buffer(512)
        la, lb, lc = lens if lens is not None else (A.size, B.size, Cm.size)
        f = self.blas.kbref_sgemm_a if Cm.dtype == np.float32 else self.blas.kbref_dgemm_a
        rc = f(_op(opa), _op(opb), m, n, k, alpha, _ptr(A), a_shape[0], a_shape[1], lda, sa, la, batch, _ptr(B),
               b_shape[0], b_shape[1], ldb, lb, beta, _ptr(Cm), c_shape[0], c_shape[1], ldc, sc, lc, hint, err, 512)
        if rc:
            self._raise(rc, err)
