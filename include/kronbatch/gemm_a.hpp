// kronbatch/gemm_a.hpp -- drop-in gemm_a (reference: proj/include/kronbatch/gemm_a.hpp:9-76)
// running on B200 through libkronbatch_b200.so.
//
//   C^p <- alpha * op(A^p) * op(B) + beta * C^p,  p = 0 .. batch_count-1
//
// A batched GEMM with the left matrix varying and B shared. Same signature,
// validation order and messages, early exits and exception types as the
// reference; op_a = N follows the reference's gemm_axpy (w = fl(alpha B_r),
// one fma per term), op_a = T its gemm_dot (dot from 0, then alpha*acc +
// beta*C). parallel_hint only chunks the reference's CPU workers; it cannot
// change results and is ignored here.
#pragma once

#include <kronbatch/b200.hpp>
#include <kronbatch/types.hpp>
#include <kronbatch/views.hpp>

namespace kronbatch {

template <Element T>
void gemm_a(MatrixOp op_a, MatrixOp op_b, index_t m, index_t n, index_t k, T alpha, BatchView<MatrixView<const T>> a,
            MatrixView<const T> b, T beta, BatchView<MatrixView<T>> c, index_t parallel_hint = 0) {
  (void)parallel_hint;
  validate_batch(a, "gemm_a: A");
  validate(b, "gemm_a: B");
  validate_batch(c, "gemm_a: C");
  const auto [ram, rak] = op_dims(op_a, a.base.rows, a.base.cols);
  const auto [rbk, rbn] = op_dims(op_b, b.rows, b.cols);
  detail::require(a.batch_count == c.batch_count, "gemm_a", "A and C batch_count differ");
  detail::require(ram == m && rak == k, "gemm_a: A",
                  "op(A) is " + detail::dim2s(ram, rak) + ", expected " + detail::dim2s(m, k));
  detail::require(rbk == k && rbn == n, "gemm_a: B",
                  "op(B) is " + detail::dim2s(rbk, rbn) + ", expected " + detail::dim2s(k, n));
  detail::require(c.base.rows == m && c.base.cols == n, "gemm_a: C",
                  "entry is " + detail::dim2s(c.base.rows, c.base.cols) + ", expected " + detail::dim2s(m, n));

  char err[512] = {0};
  const b200::ExecC ex;
  int rc;
  if constexpr (std::same_as<T, float>)
    rc = kb_sgemm_a(b200::op_char(op_a), b200::op_char(op_b), m, n, k, a.batch_count, alpha, a.base.data, a.base.ld,
                    a.batch_stride, a.base.len, b.data, b.ld, b.len, beta, c.base.data, c.base.ld, c.batch_stride,
                    c.base.len, ex.ptr, err, sizeof err);
  else
    rc = kb_dgemm_a(b200::op_char(op_a), b200::op_char(op_b), m, n, k, a.batch_count, alpha, a.base.data, a.base.ld,
                    a.batch_stride, a.base.len, b.data, b.ld, b.len, beta, c.base.data, c.base.ld, c.batch_stride,
                    c.base.len, ex.ptr, err, sizeof err);
  b200::check(rc, err);
}

}  // namespace kronbatch
