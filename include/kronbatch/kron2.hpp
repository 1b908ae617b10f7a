// kronbatch/kron2.hpp -- drop-in kron2 (reference: proj/include/kronbatch/kron2.hpp:9-110)
// running on B200 through libkronbatch_b200.so.
//
//   Y^p <- alpha * op(A) * op(X^p) * op(B)^T + beta * Y^p,  p < batch_count
//   vec(Y^p) = alpha * (op(B) (x) op(A)) vec(op(X^p)) + beta * vec(Y^p)
//
// Same signature, validation order and messages, early exits and exception
// types as the reference; the per-entry work runs in the sm_100a kernels with
// the reference's contraction order (tmp = op(A) op(X), then tmp op(B)^T; one
// fma per term, ascending), so results match the CPU path.
#pragma once

#include <kronbatch/b200.hpp>
#include <kronbatch/types.hpp>
#include <kronbatch/views.hpp>

namespace kronbatch {

template <Element T>
struct KronProblem2D {
  MatrixOp op_a = MatrixOp::NoTranspose;
  MatrixOp op_b = MatrixOp::NoTranspose;
  MatrixOp op_x = MatrixOp::NoTranspose;
  index_t m_a = 0, n_a = 0;
  index_t m_b = 0, n_b = 0;
  T alpha = T(1);
  T beta = T(0);
};

template <Element T>
void kron2(const KronProblem2D<T>& pr, MatrixView<const T> a, MatrixView<const T> b,
           BatchView<MatrixView<const T>> x, BatchView<MatrixView<T>> y) {
  validate(a, "kron2: A");
  validate(b, "kron2: B");
  validate_batch(x, "kron2: X");
  validate_batch(y, "kron2: Y");
  const auto [ra, ca] = op_dims(pr.op_a, a.rows, a.cols);
  const auto [rb, cb] = op_dims(pr.op_b, b.rows, b.cols);
  detail::require(ra == pr.m_a && ca == pr.n_a, "kron2: A",
                  "op(A) is " + detail::dim2s(ra, ca) + ", expected " + detail::dim2s(pr.m_a, pr.n_a));
  detail::require(rb == pr.m_b && cb == pr.n_b, "kron2: B",
                  "op(B) is " + detail::dim2s(rb, cb) + ", expected " + detail::dim2s(pr.m_b, pr.n_b));
  detail::require(x.batch_count == y.batch_count, "kron2", "X and Y batch_count differ");
  const auto [rx, cx] = op_dims(pr.op_x, x.base.rows, x.base.cols);
  detail::require(rx == pr.n_a && cx == pr.n_b, "kron2: X",
                  "op(X) is " + detail::dim2s(rx, cx) + ", expected " + detail::dim2s(pr.n_a, pr.n_b));
  detail::require(y.base.rows == pr.m_a && y.base.cols == pr.m_b, "kron2: Y",
                  "entry is " + detail::dim2s(y.base.rows, y.base.cols) + ", expected " +
                      detail::dim2s(pr.m_a, pr.m_b));

  char err[512] = {0};
  const b200::ExecC ex;
  int rc;
  if constexpr (std::same_as<T, float>)
    rc = kb_skron2(b200::op_char(pr.op_a), b200::op_char(pr.op_b), b200::op_char(pr.op_x), pr.m_a, pr.n_a, pr.m_b,
                   pr.n_b, x.batch_count, pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, x.base.data, x.base.ld,
                   x.batch_stride, x.base.len, pr.beta, y.base.data, y.base.ld, y.batch_stride, y.base.len, ex.ptr,
                   err, sizeof err);
  else
    rc = kb_dkron2(b200::op_char(pr.op_a), b200::op_char(pr.op_b), b200::op_char(pr.op_x), pr.m_a, pr.n_a, pr.m_b,
                   pr.n_b, x.batch_count, pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, x.base.data, x.base.ld,
                   x.batch_stride, x.base.len, pr.beta, y.base.data, y.base.ld, y.batch_stride, y.base.len, ex.ptr,
                   err, sizeof err);
  b200::check(rc, err);
}

}  // namespace kronbatch
