// kb_fast_switch.cu -- size switch of the square n <= 16 fast path: square
// problems (m_a = n_a = m_b = ... = n) go to the per-size kernels, anything
// else returns cudaErrorNotSupported (the runtime then runs the generic kernel).
#include "kb_kernels.h"
#include "kb_sizes.h"

namespace kb {

#define KB_CASE2(N) \
  case N:           \
    return kron2_size<T, N>(p, ha, hw, sm_count, s);
#define KB_CASE3(N) \
  case N:           \
    return kron3_size<T, N>(p, ha, hb, hc, sm_count, s);

template <typename T>
cudaError_t launch_kron2_fast(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s) {
  if (p.m_a != p.n_a || p.m_a != p.m_b || p.m_a != p.n_b) return cudaErrorNotSupported;
  switch (p.m_a) {
    KB_CASE2(1) KB_CASE2(2) KB_CASE2(3) KB_CASE2(4) KB_CASE2(5) KB_CASE2(6) KB_CASE2(7) KB_CASE2(8)
    KB_CASE2(9) KB_CASE2(10) KB_CASE2(11) KB_CASE2(12) KB_CASE2(13) KB_CASE2(14) KB_CASE2(15) KB_CASE2(16)
    default: return cudaErrorNotSupported;
  }
}

template <typename T>
cudaError_t launch_kron3_fast(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                              cudaStream_t s) {
  if (p.m_a != p.n_a || p.m_a != p.m_b || p.m_a != p.n_b || p.m_a != p.m_c || p.m_a != p.n_c)
    return cudaErrorNotSupported;
  switch (p.m_a) {
    KB_CASE3(1) KB_CASE3(2) KB_CASE3(3) KB_CASE3(4) KB_CASE3(5) KB_CASE3(6) KB_CASE3(7) KB_CASE3(8)
    KB_CASE3(9) KB_CASE3(10) KB_CASE3(11) KB_CASE3(12) KB_CASE3(13) KB_CASE3(14) KB_CASE3(15) KB_CASE3(16)
    default: return cudaErrorNotSupported;
  }
}

#undef KB_CASE2
#undef KB_CASE3

template cudaError_t launch_kron2_fast<float>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t launch_kron2_fast<double>(const Kron2Params<double>&, const double*, const double*, int,
                                               cudaStream_t);
template cudaError_t launch_kron3_fast<float>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                              cudaStream_t);
template cudaError_t launch_kron3_fast<double>(const Kron3Params<double>&, const double*, const double*,
                                               const double*, int, cudaStream_t);

}  // namespace kb
