// oracle/ref_shim_blas.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference's other two operators,
// compiled by oracle/Makefile from /root/reference/proj into
// oracle/_ref/libkronref_blas.so -- a SEPARATE library from libkronref.so on
// purpose: the reference is header-only, so g++'s vectorisation (and with it
// which gemm_axpy_fixed<M> instances are FMA chains) depends on every
// instantiation in the translation unit; instantiating kron1/gemm_a next to
// kron2/kron3 changes the kron2 pattern at n = 2..8. Keeping them apart keeps
// libkronref.so exactly the kron2/kron3 build the parity tests pin.
//   kronbatch::kron1<T>   proj/include/kronbatch/kron1.hpp:17-62
//   kronbatch::gemm_a<T>  proj/include/kronbatch/gemm_a.hpp:18-76
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include <kronbatch/kronbatch.hpp>

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

int fail(const std::exception& e, int code, char* err, std::size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

template <typename T>
int kron1_impl(char opa, index_t m_a, index_t n_a, T alpha, const T* A, index_t a_rows, index_t a_cols,
               index_t lda, index_t lena, const T* X, index_t x_size, index_t sx, index_t lenx, index_t batch,
               T beta, T* Y, index_t y_size, index_t sy, index_t leny, char* err, std::size_t errlen) {
  try {
    kronbatch::kron1<T>(to_op(opa), m_a, n_a, alpha, MatrixView<const T>(A, a_rows, a_cols, lda, lena),
                        BatchView<kronbatch::VectorView<const T>>(kronbatch::VectorView<const T>(X, x_size, lenx),
                                                                  batch, sx),
                        beta, BatchView<kronbatch::VectorView<T>>(kronbatch::VectorView<T>(Y, y_size, leny), batch, sy));
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1, err, errlen);
  } catch (const std::exception& e) {
    return fail(e, 3, err, errlen);
  }
}

template <typename T>
int gemm_a_impl(char opa, char opb, index_t m, index_t n, index_t k, T alpha, const T* A, index_t a_rows,
                index_t a_cols, index_t lda, index_t sa, index_t lena, index_t batch, const T* B, index_t b_rows,
                index_t b_cols, index_t ldb, index_t lenb, T beta, T* C, index_t c_rows, index_t c_cols, index_t ldc,
                index_t sc, index_t lenc, index_t hint, char* err, std::size_t errlen) {
  try {
    kronbatch::gemm_a<T>(to_op(opa), to_op(opb), m, n, k, alpha,
                         BatchView<MatrixView<const T>>(MatrixView<const T>(A, a_rows, a_cols, lda, lena), batch, sa),
                         MatrixView<const T>(B, b_rows, b_cols, ldb, lenb), beta,
                         BatchView<MatrixView<T>>(MatrixView<T>(C, c_rows, c_cols, ldc, lenc), batch, sc), hint);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1, err, errlen);
  } catch (const std::exception& e) {
    return fail(e, 3, err, errlen);
  }
}

}  // namespace

extern "C" {

// kronbatch::kron1<T>   proj/include/kronbatch/kron1.hpp:17-62
#define KBREF_KRON1(NAME, T)                                                                                     \
  int NAME(char opa, int64_t m_a, int64_t n_a, T alpha, const T* A, int64_t a_rows, int64_t a_cols, int64_t lda,  \
           int64_t lena, const T* X, int64_t x_size, int64_t sx, int64_t lenx, int64_t batch, T beta, T* Y,      \
           int64_t y_size, int64_t sy, int64_t leny, char* err, size_t errlen) {                                 \
    return kron1_impl<T>(opa, m_a, n_a, alpha, A, a_rows, a_cols, lda, lena, X, x_size, sx, lenx, batch, beta, Y, \
                         y_size, sy, leny, err, errlen);                                                          \
  }
KBREF_KRON1(kbref_skron1, float)
KBREF_KRON1(kbref_dkron1, double)

// kronbatch::gemm_a<T>  proj/include/kronbatch/gemm_a.hpp:18-76
#define KBREF_GEMMA(NAME, T)                                                                                      \
  int NAME(char opa, char opb, int64_t m, int64_t n, int64_t k, T alpha, const T* A, int64_t a_rows,             \
           int64_t a_cols, int64_t lda, int64_t sa, int64_t lena, int64_t batch, const T* B, int64_t b_rows,      \
           int64_t b_cols, int64_t ldb, int64_t lenb, T beta, T* C, int64_t c_rows, int64_t c_cols, int64_t ldc,  \
           int64_t sc, int64_t lenc, int64_t hint, char* err, size_t errlen) {                                    \
    return gemm_a_impl<T>(opa, opb, m, n, k, alpha, A, a_rows, a_cols, lda, sa, lena, batch, B, b_rows, b_cols,   \
                          ldb, lenb, beta, C, c_rows, c_cols, ldc, sc, lenc, hint, err, errlen);                  \
  }
KBREF_GEMMA(kbref_sgemm_a, float)
KBREF_GEMMA(kbref_dgemm_a, double)

}  // extern "C"
