// kb_kernels.h -- internal launch interface between the host runtime
// (kb_runtime.cu) and the sm_100a kernels (kb_generic.cu, kb_fast*.cu).
#pragma once

#include <cuda_runtime.h>

#include "kb_device.cuh"

namespace kb {

// Shape-generic kernels: any dims / ops / strides. `scratch` (grid * per-CTA
// intermediate elements) is only used when the per-entry intermediates exceed
// the 48 KiB shared-memory budget.
template <typename T>
cudaError_t launch_kron2_generic(const Kron2Params<T>& p, T* scratch, long long scratch_elems, int grid,
                                 cudaStream_t s);
template <typename T>
cudaError_t launch_kron3_generic(const Kron3Params<T>& p, T* scratch, long long scratch_elems, int grid,
                                 cudaStream_t s);
// Y <- init(beta) for the alpha == 0 / empty-sum path.
template <typename T>
cudaError_t launch_scale(T* Y, long long batch, long long d1, long long d2, long long d3, long long ld,
                         long long ld2, long long sy, int beta_mode, T beta, int grid, cudaStream_t s);

// Strided batch copy (padded <-> tight entry layouts) for the square
// fast paths on padded / strided callers: entry elements only, padding untouched.
template <typename T>
cudaError_t launch_repack(const T* src, long long s_ld, long long s_ld2, long long s_stride, T* dst, long long d_ld,
                          long long d_ld2, long long d_stride, int d1, int d2, int d3, long long batch, int sm_count,
                          cudaStream_t s);

// Square n <= 16 register-blocked kernels. Return cudaErrorNotSupported
// (without launching) when the layout does not meet the fast-path
// preconditions (tight entries, vector alignment); the caller then uses the
// generic kernel. The constant matrices come as HOST arrays, op-resolved and
// alpha-folded (n*n each): ha = A_r col-major, hw/hc = fl(alpha*B_r / C_r)
// row-major, hb = B_r row-major; they are passed as kernel parameters.
template <typename T>
cudaError_t launch_kron2_fast(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s);
template <typename T>
cudaError_t launch_kron3_fast(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                              cudaStream_t s);

// kron1 / gemm_a (kb_blas.cu): any shape, op, stride; one thread per output.
template <typename T>
cudaError_t launch_kron1(const T* A, long long lda, int opa, const T* X, long long sx, T* Y, long long sy,
                         long long m, long long n, long long batch, T alpha, int beta_mode, T beta, int sm_count,
                         cudaStream_t s);
// kron1 square n <= 16, contiguous x / y entries, host-resolved A_r (col-major).
template <typename T>
cudaError_t launch_kron1_sq(int n, const T* ha, const T* X, T* Y, long long batch, T alpha, int beta_mode, T beta,
                            int sm_count, cudaStream_t s);
template <typename T>
cudaError_t launch_gemm_a_sq(int n, bool opt, const T* hw, const T* A, T* Cm, long long batch, T alpha, int beta_mode,
                             T beta, int sm_count, cudaStream_t s);
template <typename T>
cudaError_t launch_gemm_a(const T* A, long long lda, long long sa, int opa, const T* B, long long ldb, int opb, T* Cm,
                          long long ldc, long long sc, long long m, long long n, long long k, long long batch, T alpha,
                          int beta_mode, T beta, int sm_count, cudaStream_t s);

// 3-D fp32 n = 16 on tcgen05 tensor cores with 3xTF32 compensation
// (tolerance-level parity, not bit-exact). Same host constant layouts.
cudaError_t launch_kron3_tc(const Kron3Params<float>& p, const float* ha, const float* hb, const float* hc,
                            int sm_count, cudaStream_t s);

}  // namespace kb
