// kronbatch/kron1.hpp -- drop-in kron1 (reference: proj/include/kronbatch/kron1.hpp:9-62)
// running on B200 through libkronbatch_b200.so.
//
//   y^p <- alpha * op(A) * x^p + beta * y^p,  p = 0 .. batch_count-1
//
// A batched GEMV with A shared across the batch. Same signature, validation
// order and messages, early exits and exception types as the reference; the
// arithmetic is the reference's gemm_axpy with R = x^p (w = fl(alpha x[kk]),
// one fma per term, ascending).
#pragma once

#include <kronbatch/b200.hpp>
#include <kronbatch/types.hpp>
#include <kronbatch/views.hpp>

namespace kronbatch {

template <Element T>
void kron1(MatrixOp op_a, index_t m_a, index_t n_a, T alpha, MatrixView<const T> a, BatchView<VectorView<const T>> x,
           T beta, BatchView<VectorView<T>> y) {
  validate(a, "kron1: A");
  validate_batch(x, "kron1: X");
  validate_batch(y, "kron1: Y");
  const auto [ra, ca] = op_dims(op_a, a.rows, a.cols);
  detail::require(ra == m_a && ca == n_a, "kron1: A",
                  "op(A) is " + detail::dim2s(ra, ca) + ", expected " + detail::dim2s(m_a, n_a));
  detail::require(x.batch_count == y.batch_count, "kron1", "X and Y batch_count differ");
  detail::require(x.base.size == n_a, "kron1: X",
                  "entry length " + std::to_string(x.base.size) + ", expected " + std::to_string(n_a));
  detail::require(y.base.size == m_a, "kron1: Y",
                  "entry length " + std::to_string(y.base.size) + ", expected " + std::to_string(m_a));

  char err[512] = {0};
  const b200::ExecC ex;
  int rc;
  if constexpr (std::same_as<T, float>)
    rc = kb_skron1(b200::op_char(op_a), m_a, n_a, x.batch_count, alpha, a.data, a.ld, a.len, x.base.data,
                   x.batch_stride, x.base.len, beta, y.base.data, y.batch_stride, y.base.len, ex.ptr, err, sizeof err);
  else
    rc = kb_dkron1(b200::op_char(op_a), m_a, n_a, x.batch_count, alpha, a.data, a.ld, a.len, x.base.data,
                   x.batch_stride, x.base.len, beta, y.base.data, y.batch_stride, y.base.len, ex.ptr, err, sizeof err);
  b200::check(rc, err);
}

}  // namespace kronbatch
