// kronbatch/kron3.hpp -- drop-in kron3 (reference: proj/include/kronbatch/kron3.hpp:12-166)
// running on B200 through libkronbatch_b200.so.
//
//   vec(Y^p) <- alpha * (op(C) (x) op(B) (x) op(A)) vec(X^p) + beta * vec(Y^p)
//
// Contraction order mode 1 (A) -> mode 2 (B) -> mode 3 (C) as in the
// reference's Algorithm-1 staging, but fused on chip: the caller Workspace is
// still required and capacity-checked first (kron3.hpp:104-109) so existing
// callers behave identically, yet the GPU path never reads or writes it.
#pragma once

#include <span>
#include <stdexcept>
#include <string>

#include <kronbatch/b200.hpp>
#include <kronbatch/types.hpp>
#include <kronbatch/views.hpp>

namespace kronbatch {

template <Element T>
struct KronProblem3D {
  MatrixOp op_a = MatrixOp::NoTranspose;
  MatrixOp op_b = MatrixOp::NoTranspose;
  MatrixOp op_c = MatrixOp::NoTranspose;
  index_t m_a = 0, n_a = 0;
  index_t m_b = 0, n_b = 0;
  index_t m_c = 0, n_c = 0;
  T alpha = T(1);
  T beta = T(0);
};

/// Caller scratch of the reference's two-stage kron3 (m_a*m_b*n_c per entry).
template <Element T>
struct Workspace {
  T* data = nullptr;
  index_t capacity = 0;

  constexpr Workspace() = default;
  constexpr Workspace(std::span<T> buf) : data(buf.data()), capacity(static_cast<index_t>(buf.size())) {}
  constexpr Workspace(T* d, index_t cap) : data(d), capacity(cap) {}
};

/// m_a*m_b*n_c*batch_count; std::overflow_error past index_t.
template <Element T>
index_t kron3_workspace_size(const KronProblem3D<T>& pr, index_t batch_count) {
  detail::require(pr.m_a >= 0 && pr.m_b >= 0 && pr.n_c >= 0 && batch_count >= 0, "kron3_workspace_size",
                  "negative dimension");
  index_t out = 0;
  char err[256] = {0};
  b200::check(kb_kron3_workspace_size(pr.m_a, pr.m_b, pr.n_c, batch_count, &out, err, sizeof err), err);
  return out;
}

template <Element T>
void kron3(const KronProblem3D<T>& pr, MatrixView<const T> a, MatrixView<const T> b, MatrixView<const T> c,
           BatchView<Array3View<const T>> x, BatchView<Array3View<T>> y, Workspace<T> work) {
  validate(a, "kron3: A");
  validate(b, "kron3: B");
  validate(c, "kron3: C");
  validate_batch(x, "kron3: X");
  validate_batch(y, "kron3: Y");
  const auto [ra, ca] = op_dims(pr.op_a, a.rows, a.cols);
  const auto [rb, cb] = op_dims(pr.op_b, b.rows, b.cols);
  const auto [rc, cc] = op_dims(pr.op_c, c.rows, c.cols);
  detail::require(ra == pr.m_a && ca == pr.n_a, "kron3: A",
                  "op(A) is " + detail::dim2s(ra, ca) + ", expected " + detail::dim2s(pr.m_a, pr.n_a));
  detail::require(rb == pr.m_b && cb == pr.n_b, "kron3: B",
                  "op(B) is " + detail::dim2s(rb, cb) + ", expected " + detail::dim2s(pr.m_b, pr.n_b));
  detail::require(rc == pr.m_c && cc == pr.n_c, "kron3: C",
                  "op(C) is " + detail::dim2s(rc, cc) + ", expected " + detail::dim2s(pr.m_c, pr.n_c));
  detail::require(x.batch_count == y.batch_count, "kron3", "X and Y batch_count differ");
  detail::require(x.base.dim1 == pr.n_a && x.base.dim2 == pr.n_b && x.base.dim3 == pr.n_c, "kron3: X",
                  "entry dims do not match n_a x n_b x n_c");
  detail::require(y.base.dim1 == pr.m_a && y.base.dim2 == pr.m_b && y.base.dim3 == pr.m_c, "kron3: Y",
                  "entry dims do not match m_a x m_b x m_c");

  char err[512] = {0};
  const b200::ExecC ex;
  int rc_;
  if constexpr (std::same_as<T, float>)
    rc_ = kb_skron3(b200::op_char(pr.op_a), b200::op_char(pr.op_b), b200::op_char(pr.op_c), pr.m_a, pr.n_a, pr.m_b,
                    pr.n_b, pr.m_c, pr.n_c, x.batch_count, pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, c.data,
                    c.ld, c.len, x.base.data, x.base.ld, x.base.ld2, x.batch_stride, x.base.len, pr.beta, y.base.data,
                    y.base.ld, y.base.ld2, y.batch_stride, y.base.len, work.data, work.capacity, ex.ptr, err,
                    sizeof err);
  else
    rc_ = kb_dkron3(b200::op_char(pr.op_a), b200::op_char(pr.op_b), b200::op_char(pr.op_c), pr.m_a, pr.n_a, pr.m_b,
                    pr.n_b, pr.m_c, pr.n_c, x.batch_count, pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, c.data,
                    c.ld, c.len, x.base.data, x.base.ld, x.base.ld2, x.batch_stride, x.base.len, pr.beta, y.base.data,
                    y.base.ld, y.base.ld2, y.batch_stride, y.base.len, work.data, work.capacity, ex.ptr, err,
                    sizeof err);
  b200::check(rc_, err);
}

}  // namespace kronbatch
