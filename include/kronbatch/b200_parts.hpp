// kronbatch/b200_parts.hpp -- C++ face of kb_?kron{2,3}_parts (not in the
// reference API): one kron2 / kron3 over a batch that is already split over
// several GPUs (e.g. one device-resident slice per GPU, as a data-parallel
// caller holds it). Every part is validated before anything runs; the parts
// run concurrently, one per device, with no collective; the call returns when
// all are done (or all are queued, asynchronous = true with device buffers).
// Results are bit-identical to one call over the concatenated batch.
#pragma once

#include <span>
#include <vector>

#include <kronbatch/kron2.hpp>
#include <kronbatch/kron3.hpp>

namespace kronbatch {
namespace b200 {

template <Element T, class XView, class YView>
struct Part {
  std::int32_t device = 0;          // GPU that runs the part (where device buffers live)
  BatchView<XView> x;               // the part's entries; same entry layout in every part
  BatchView<YView> y;
  void* stream = nullptr;           // cudaStream_t on `device`; nullptr => library stream
};
template <Element T>
using Part2 = Part<T, MatrixView<const T>, MatrixView<T>>;
template <Element T>
using Part3 = Part<T, Array3View<const T>, Array3View<T>>;

template <class P>
std::vector<kb_part> to_c_parts(std::span<const P> parts) {
  std::vector<kb_part> out;
  out.reserve(parts.size());
  for (const P& p : parts)
    out.push_back(kb_part{p.device, p.x.batch_count, p.x.base.data, p.x.base.len, p.y.base.data, p.y.base.len,
                          p.stream});
  return out;
}

template <Element T>
void kron2_parts(const KronProblem2D<T>& pr, MatrixView<const T> a, MatrixView<const T> b,
                 std::span<const Part2<T>> parts, bool asynchronous = false) {
  if (parts.empty()) return;
  const auto& x0 = parts[0].x;
  const auto& y0 = parts[0].y;
  const std::vector<kb_part> cp = to_c_parts(parts);
  char err[1024] = {0};
  const std::uint32_t flags = asynchronous ? KB_EXEC_ASYNC : 0u;
  int rc;
  if constexpr (std::same_as<T, float>)
    rc = kb_skron2_parts(op_char(pr.op_a), op_char(pr.op_b), op_char(pr.op_x), pr.m_a, pr.n_a, pr.m_b, pr.n_b,
                         pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, x0.base.ld, x0.batch_stride, pr.beta,
                         y0.base.ld, y0.batch_stride, (std::int32_t)cp.size(), cp.data(), flags, err, sizeof err);
  else
    rc = kb_dkron2_parts(op_char(pr.op_a), op_char(pr.op_b), op_char(pr.op_x), pr.m_a, pr.n_a, pr.m_b, pr.n_b,
                         pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, x0.base.ld, x0.batch_stride, pr.beta,
                         y0.base.ld, y0.batch_stride, (std::int32_t)cp.size(), cp.data(), flags, err, sizeof err);
  check(rc, err);
}

template <Element T>
void kron3_parts(const KronProblem3D<T>& pr, MatrixView<const T> a, MatrixView<const T> b, MatrixView<const T> c,
                 std::span<const Part3<T>> parts, bool asynchronous = false) {
  if (parts.empty()) return;
  const auto& x0 = parts[0].x;
  const auto& y0 = parts[0].y;
  const std::vector<kb_part> cp = to_c_parts(parts);
  char err[1024] = {0};
  const std::uint32_t flags = asynchronous ? KB_EXEC_ASYNC : 0u;
  int rc;
  if constexpr (std::same_as<T, float>)
    rc = kb_skron3_parts(op_char(pr.op_a), op_char(pr.op_b), op_char(pr.op_c), pr.m_a, pr.n_a, pr.m_b, pr.n_b,
                         pr.m_c, pr.n_c, pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, c.data, c.ld, c.len,
                         x0.base.ld, x0.base.ld2, x0.batch_stride, pr.beta, y0.base.ld, y0.base.ld2,
                         y0.batch_stride, (std::int32_t)cp.size(), cp.data(), flags, err, sizeof err);
  else
    rc = kb_dkron3_parts(op_char(pr.op_a), op_char(pr.op_b), op_char(pr.op_c), pr.m_a, pr.n_a, pr.m_b, pr.n_b,
                         pr.m_c, pr.n_c, pr.alpha, a.data, a.ld, a.len, b.data, b.ld, b.len, c.data, c.ld, c.len,
                         x0.base.ld, x0.base.ld2, x0.batch_stride, pr.beta, y0.base.ld, y0.base.ld2,
                         y0.batch_stride, (std::int32_t)cp.size(), cp.data(), flags, err, sizeof err);
  check(rc, err);
}

}  // namespace b200
}  // namespace kronbatch
