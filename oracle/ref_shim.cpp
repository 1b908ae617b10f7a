// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile directly from the sources where they lie under
// /root/reference/proj (include/kronbatch/*.hpp, src/reference.cpp,
// tools/bench_support.cpp) into oracle/_ref/libkronref.so. No reference
// source is copied into this repository; this file only builds views over raw
// pointers and forwards to the reference's own templates:
//   kronbatch::kron2<T>            proj/include/kronbatch/kron2.hpp:37-110
//   kronbatch::kron3<T>            proj/include/kronbatch/kron3.hpp:72-166
//   kronbatch::kron3_workspace_size proj/include/kronbatch/kron3.hpp:43-53
//   kronbatch::ref_kron{2,3}_apply proj/src/reference.cpp:162-207
//   kronbench::generate_batch<T>   proj/tools/bench_support.hpp:148-170
//   kronbench::flops_kron / problem_bytes  proj/tools/bench_support.cpp:31-80
// Used by tests/golden/make_golden.py (fixtures), tests/ (pinning the oracle)
// and bench.py --impl reference / cpu_baseline (the reference CPU arm).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "bench_support.hpp"
#include <kronbatch/kronbatch.hpp>

using kronbatch::Array3View;
using kronbatch::BatchView;
using kronbatch::index_t;
using kronbatch::MatrixOp;
using kronbatch::MatrixView;

namespace {

MatrixOp to_op(char c) {
  switch (c) {
    case 'T': case 't': return MatrixOp::Transpose;
    case 'C': case 'c': return MatrixOp::ConjTranspose;
    default: return MatrixOp::NoTranspose;
  }
}

// 0 ok; 1 invalid_argument; 2 overflow_error; 3 other
int fail(const std::exception& e, int code, char* err, std::size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

template <typename T>
int kron2_impl(char opa, char opb, char opx, index_t m_a, index_t n_a,
               index_t m_b, index_t n_b, index_t batch, T alpha, const T* A,
               index_t a_rows, index_t a_cols, index_t lda, index_t lena,
               const T* B, index_t b_rows, index_t b_cols, index_t ldb,
               index_t lenb, const T* X, index_t x_rows, index_t x_cols,
               index_t ldx, index_t sx, index_t lenx, T beta, T* Y,
               index_t y_rows, index_t y_cols, index_t ldy, index_t sy,
               index_t leny, char* err, std::size_t errlen) {
  try {
    kronbatch::KronProblem2D<T> pr;
    pr.op_a = to_op(opa);
    pr.op_b = to_op(opb);
    pr.op_x = to_op(opx);
    pr.m_a = m_a; pr.n_a = n_a; pr.m_b = m_b; pr.n_b = n_b;
    pr.alpha = alpha; pr.beta = beta;
    kronbatch::kron2<T>(
        pr, MatrixView<const T>(A, a_rows, a_cols, lda, lena),
        MatrixView<const T>(B, b_rows, b_cols, ldb, lenb),
        BatchView<MatrixView<const T>>(
            MatrixView<const T>(X, x_rows, x_cols, ldx, lenx), batch, sx),
        BatchView<MatrixView<T>>(MatrixView<T>(Y, y_rows, y_cols, ldy, leny),
                                 batch, sy));
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1, err, errlen);
  } catch (const std::overflow_error& e) {
    return fail(e, 2, err, errlen);
  } catch (const std::exception& e) {
    return fail(e, 3, err, errlen);
  }
}

template <typename T>
int kron3_impl(char opa, char opb, char opc, index_t m_a, index_t n_a,
               index_t m_b, index_t n_b, index_t m_c, index_t n_c,
               index_t batch, T alpha, const T* A, index_t a_rows,
               index_t a_cols, index_t lda, index_t lena, const T* B,
               index_t b_rows, index_t b_cols, index_t ldb, index_t lenb,
               const T* C, index_t c_rows, index_t c_cols, index_t ldc,
               index_t lenc, const T* X, index_t xd1, index_t xd2, index_t xd3,
               index_t ldx, index_t ldx2, index_t sx, index_t lenx, T beta,
               T* Y, index_t yd1, index_t yd2, index_t yd3, index_t ldy,
               index_t ldy2, index_t sy, index_t leny, T* work,
               index_t work_cap, char* err, std::size_t errlen) {
  try {
    kronbatch::KronProblem3D<T> pr;
    pr.op_a = to_op(opa);
    pr.op_b = to_op(opb);
    pr.op_c = to_op(opc);
    pr.m_a = m_a; pr.n_a = n_a; pr.m_b = m_b; pr.n_b = n_b;
    pr.m_c = m_c; pr.n_c = n_c;
    pr.alpha = alpha; pr.beta = beta;
    kronbatch::kron3<T>(
        pr, MatrixView<const T>(A, a_rows, a_cols, lda, lena),
        MatrixView<const T>(B, b_rows, b_cols, ldb, lenb),
        MatrixView<const T>(C, c_rows, c_cols, ldc, lenc),
        BatchView<Array3View<const T>>(
            Array3View<const T>(X, xd1, xd2, xd3, ldx, ldx2, lenx), batch, sx),
        BatchView<Array3View<T>>(
            Array3View<T>(Y, yd1, yd2, yd3, ldy, ldy2, leny), batch, sy),
        kronbatch::Workspace<T>(work, work_cap));
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1, err, errlen);
  } catch (const std::overflow_error& e) {
    return fail(e, 2, err, errlen);
  } catch (const std::exception& e) {
    return fail(e, 3, err, errlen);
  }
}

}  // namespace

extern "C" {



int kbref_has_openmp(void) {
#ifdef _OPENMP
  return 1;
#else
  return 0;
#endif
}

int kbref_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void kbref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

#define KBREF_KRON2(NAME, T)                                                   \
  int NAME(char opa, char opb, char opx, int64_t m_a, int64_t n_a,             \
           int64_t m_b, int64_t n_b, int64_t batch, T alpha, const T* A,       \
           int64_t a_rows, int64_t a_cols, int64_t lda, int64_t lena,          \
           const T* B, int64_t b_rows, int64_t b_cols, int64_t ldb,            \
           int64_t lenb, const T* X, int64_t x_rows, int64_t x_cols,           \
           int64_t ldx, int64_t sx, int64_t lenx, T beta, T* Y,                \
           int64_t y_rows, int64_t y_cols, int64_t ldy, int64_t sy,            \
           int64_t leny, char* err, size_t errlen) {                           \
    return kron2_impl<T>(opa, opb, opx, m_a, n_a, m_b, n_b, batch, alpha, A,   \
                         a_rows, a_cols, lda, lena, B, b_rows, b_cols, ldb,    \
                         lenb, X, x_rows, x_cols, ldx, sx, lenx, beta, Y,      \
                         y_rows, y_cols, ldy, sy, leny, err, errlen);          \
  }
KBREF_KRON2(kbref_skron2, float)
KBREF_KRON2(kbref_dkron2, double)

#define KBREF_KRON3(NAME, T)                                                   \
  int NAME(char opa, char opb, char opc, int64_t m_a, int64_t n_a,             \
           int64_t m_b, int64_t n_b, int64_t m_c, int64_t n_c, int64_t batch,  \
           T alpha, const T* A, int64_t a_rows, int64_t a_cols, int64_t lda,   \
           int64_t lena, const T* B, int64_t b_rows, int64_t b_cols,           \
           int64_t ldb, int64_t lenb, const T* C, int64_t c_rows,              \
           int64_t c_cols, int64_t ldc, int64_t lenc, const T* X,              \
           int64_t xd1, int64_t xd2, int64_t xd3, int64_t ldx, int64_t ldx2,   \
           int64_t sx, int64_t lenx, T beta, T* Y, int64_t yd1, int64_t yd2,   \
           int64_t yd3, int64_t ldy, int64_t ldy2, int64_t sy, int64_t leny,   \
           T* work, int64_t work_cap, char* err, size_t errlen) {              \
    return kron3_impl<T>(opa, opb, opc, m_a, n_a, m_b, n_b, m_c, n_c, batch,   \
                         alpha, A, a_rows, a_cols, lda, lena, B, b_rows,       \
                         b_cols, ldb, lenb, C, c_rows, c_cols, ldc, lenc, X,   \
                         xd1, xd2, xd3, ldx, ldx2, sx, lenx, beta, Y, yd1,     \
                         yd2, yd3, ldy, ldy2, sy, leny, work, work_cap, err,   \
                         errlen);                                              \
  }
KBREF_KRON3(kbref_skron3, float)
KBREF_KRON3(kbref_dkron3, double)

// kron3_workspace_size: 0 ok, 1 invalid_argument, 2 overflow_error
int kbref_kron3_workspace_size(int64_t m_a, int64_t m_b, int64_t n_c,
                               int64_t batch, int64_t* out, char* err,
                               size_t errlen) {
  try {
    kronbatch::KronProblem3D<double> pr;
    pr.m_a = m_a; pr.m_b = m_b; pr.n_c = n_c;
    *out = kronbatch::kron3_workspace_size(pr, batch);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1, err, errlen);
  } catch (const std::overflow_error& e) {
    return fail(e, 2, err, errlen);
  }
}

// generate_batch<T>(seed, m, dims, batch): copies A, B, [C], X, Y out.
#define KBREF_GEN(NAME, T)                                                     \
  int NAME(uint64_t seed, int m, int dims3, int64_t batch, T* a, T* b, T* c,   \
           T* x, T* y) {                                                       \
    auto d = kronbench::generate_batch<T>(                                     \
        seed, m, dims3 ? kronbench::Dims::D3 : kronbench::Dims::D2, batch);    \
    std::memcpy(a, d.a.data(), d.a.size() * sizeof(T));                        \
    std::memcpy(b, d.b.data(), d.b.size() * sizeof(T));                        \
    if (dims3 && c) std::memcpy(c, d.c.data(), d.c.size() * sizeof(T));        \
    std::memcpy(x, d.x.data(), d.x.size() * sizeof(T));                        \
    std::memcpy(y, d.y.data(), d.y.size() * sizeof(T));                        \
    return 0;                                                                  \
  }
KBREF_GEN(kbref_generate_batch_f32, float)
KBREF_GEN(kbref_generate_batch_f64, double)

int64_t kbref_flops_kron(int m, int dims3) {
  try {
    return kronbench::flops_kron(m, dims3 ? kronbench::Dims::D3
                                          : kronbench::Dims::D2);
  } catch (...) {
    return -1;
  }
}

uint64_t kbref_problem_bytes(int m, int dims3, int dbl, int64_t batch) {
  return kronbench::problem_bytes(
      m, dims3 ? kronbench::Dims::D3 : kronbench::Dims::D2,
      dbl ? kronbench::Precision::Double : kronbench::Precision::Single, batch);
}

// Tight double oracles (reference.cpp:162-207).
void kbref_ref_kron2_apply(int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
                           const double* A, const double* B, const double* X,
                           double* Y) {
  const auto y = kronbatch::ref_kron2_apply(
      MatrixView<const double>(A, m_a, n_a, std::max<int64_t>(m_a, 1), m_a * n_a),
      MatrixView<const double>(B, m_b, n_b, std::max<int64_t>(m_b, 1), m_b * n_b),
      MatrixView<const double>(X, n_a, n_b, std::max<int64_t>(n_a, 1), n_a * n_b));
  std::memcpy(Y, y.storage.data(), y.storage.size() * sizeof(double));
}

void kbref_ref_kron3_apply(int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
                           int64_t m_c, int64_t n_c, const double* A,
                           const double* B, const double* C, const double* X,
                           double* Y) {
  const auto y = kronbatch::ref_kron3_apply(
      MatrixView<const double>(A, m_a, n_a, std::max<int64_t>(m_a, 1), m_a * n_a),
      MatrixView<const double>(B, m_b, n_b, std::max<int64_t>(m_b, 1), m_b * n_b),
      MatrixView<const double>(C, m_c, n_c, std::max<int64_t>(m_c, 1), m_c * n_c),
      Array3View<const double>(X, n_a, n_b, n_c, std::max<int64_t>(n_a, 1),
                               std::max<int64_t>(n_a, 1) * n_b, n_a * n_b * n_c));
  std::memcpy(Y, y.storage.data(), y.storage.size() * sizeof(double));
}

void kbref_kron_matrix(int64_t ra, int64_t ca, const double* A, int64_t rb,
                       int64_t cb, const double* B, double* K) {
  const auto k = kronbatch::kron_matrix(
      MatrixView<const double>(A, ra, ca, std::max<int64_t>(ra, 1), ra * ca),
      MatrixView<const double>(B, rb, cb, std::max<int64_t>(rb, 1), rb * cb));
  std::memcpy(K, k.storage.data(), k.storage.size() * sizeof(double));
}

}  // extern "C"
