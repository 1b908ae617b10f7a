// kb_generic.cu -- general-shape sm_100a kernels for kron2 / kron3.
//
// These cover every shape, op and stride combination the reference API
// accepts (rectangular, n > 16, padded leading dimensions / batch strides,
// ConjTranspose == Transpose). They follow the reference contraction exactly
// (kron2.hpp:95-107, kron3.hpp:147-163, detail.hpp:38-117):
//   kron2: tmp(i,c) = sum_l A_r(i,l) Xop(l,c)                (init 0, l ascending)
//          Y(i,j)  = init + sum_m tmp(i,m) * fl(alpha*B_r(j,m)) (m ascending)
//   kron3: per plane N: t1 = A_r X(:,:,N);  T2(:,:,N) = t1 B_r^T  (alpha 1, beta 0)
//          Y(i,j,k) = init + sum_N T2(i,j,N) * fl(alpha*C_r(k,N))
// One CTA owns one batch entry at a time (grid-stride over entries); the
// per-entry intermediates live in shared memory when they fit, otherwise in a
// per-CTA slice of a device scratch buffer (the library's internal pool; the
// caller's kron3 Workspace is not touched -- it is a CPU-path artefact).
// The square n <= 16 fast paths are in kb_fast.cu.
#include "kb_device.cuh"
#include "kb_kernels.h"

namespace kb {

template <typename T>
__global__ void __launch_bounds__(256) kron2_generic_kernel(Kron2Params<T> p, T* scratch, int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const long long tsz = p.m_a * p.n_b;
  T* tmp = use_smem ? reinterpret_cast<T*>(smem_raw) : scratch + (long long)blockIdx.x * tsz;
  const long long ysz = p.m_a * p.m_b;
  for (long long e = blockIdx.x; e < p.batch; e += gridDim.x) {
    const T* x = p.X + e * p.sx;
    T* y = p.Y + e * p.sy;
    // stage 1: tmp = op(A) * op(X^e)    (kron2.hpp:96-103)
    for (long long t = threadIdx.x; t < tsz; t += blockDim.x) {
      const long long i = t % p.m_a, c = t / p.m_a;
      T acc = T(0);
      for (long long l = 0; l < p.n_a; ++l)
        acc = fma_rn(op_at(p.A, p.lda, p.opa, i, l), op_at(x, p.ldx, p.opx, l, c), acc);
      tmp[t] = acc;
    }
    __syncthreads();
    // stage 2: Y = alpha * tmp * op(B)^T + beta * Y    (kron2.hpp:105-107)
    for (long long t = threadIdx.x; t < ysz; t += blockDim.x) {
      const long long i = t % p.m_a, j = t / p.m_a;
      T* yij = y + i + j * p.ldy;
      T acc = beta_init(p.beta_mode, p.beta, p.beta_mode == kBetaZero ? T(0) : *yij);
      for (long long m = 0; m < p.n_b; ++m)
        acc = fma_rn(tmp[i + m * p.m_a], mul_rn(p.alpha, op_at(p.B, p.ldb, p.opb, j, m)), acc);
      *yij = acc;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(256) kron3_generic_kernel(Kron3Params<T> p, T* scratch, int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const long long t1sz = p.m_a * p.n_b;
  const long long t2sz = p.m_a * p.m_b * p.n_c;
  T* base = use_smem ? reinterpret_cast<T*>(smem_raw) : scratch + (long long)blockIdx.x * (t1sz + t2sz);
  T* t1 = base;
  T* t2 = base + t1sz;
  const long long mab = p.m_a * p.m_b;
  const long long ysz = mab * p.m_c;
  for (long long e = blockIdx.x; e < p.batch; e += gridDim.x) {
    const T* x = p.X + e * p.sx;
    T* y = p.Y + e * p.sy;
    // stage 1 per plane (kron3.hpp:147-156)
    for (long long N = 0; N < p.n_c; ++N) {
      const T* xp = x + N * p.ldx2;
      for (long long t = threadIdx.x; t < t1sz; t += blockDim.x) {
        const long long i = t % p.m_a, c = t / p.m_a;
        T acc = T(0);
        for (long long l = 0; l < p.n_a; ++l) acc = fma_rn(op_at(p.A, p.lda, p.opa, i, l), xp[l + c * p.ldx], acc);
        t1[t] = acc;
      }
      __syncthreads();
      T* t2p = t2 + N * mab;
      for (long long t = threadIdx.x; t < mab; t += blockDim.x) {
        const long long i = t % p.m_a, j = t / p.m_a;
        T acc = T(0);
        for (long long m = 0; m < p.n_b; ++m) acc = fma_rn(t1[i + m * p.m_a], op_at(p.B, p.ldb, p.opb, j, m), acc);
        t2p[t] = acc;
      }
      __syncthreads();
    }
    // stage 2: Y(:,j,:) = alpha * T2(:,j,:) * op(C)^T + beta * Y   (kron3.hpp:158-163)
    for (long long t = threadIdx.x; t < ysz; t += blockDim.x) {
      const long long i = t % p.m_a, j = (t / p.m_a) % p.m_b, k = t / mab;
      T* yv = y + i + j * p.ldy + k * p.ldy2;
      T acc = beta_init(p.beta_mode, p.beta, p.beta_mode == kBetaZero ? T(0) : *yv);
      for (long long N = 0; N < p.n_c; ++N)
        acc = fma_rn(t2[i + j * p.m_a + N * mab], mul_rn(p.alpha, op_at(p.C, p.ldc, p.opc, k, N)), acc);
      *yv = acc;
    }
    __syncthreads();
  }
}

// Y <- init(beta) only: the empty-sum / alpha == 0 path (kron2.hpp:67-79,
// kron3.hpp:113-128). A, B, C, X are never read. Element (i, j[, k]) of entry e.
template <typename T>
__global__ void __launch_bounds__(256) scale_kernel(T* Y, long long batch, long long d1, long long d2, long long d3,
                                                    long long ld, long long ld2, long long sy, int beta_mode,
                                                    T beta) {
  const long long per = d1 * d2 * d3;
  const long long total = per * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / per, r = t % per;
    const long long i = r % d1, j = (r / d1) % d2, k = r / (d1 * d2);
    T* y = Y + e * sy + i + j * ld + k * ld2;
    *y = beta_mode == kBetaZero ? T(0) : mul_rn(*y, beta);
  }
}

// ---------------------------------------------------------------- launch --

template <typename T>
cudaError_t launch_kron2_generic(const Kron2Params<T>& p, T* scratch, long long scratch_elems, int grid,
                                 cudaStream_t s) {
  const size_t tbytes = sizeof(T) * (size_t)(p.m_a * p.n_b);
  const int use_smem = tbytes <= 48 * 1024;
  if (!use_smem && scratch_elems < (long long)grid * p.m_a * p.n_b) return cudaErrorInvalidValue;
  kron2_generic_kernel<T><<<grid, 256, use_smem ? tbytes : 0, s>>>(p, scratch, use_smem);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_kron3_generic(const Kron3Params<T>& p, T* scratch, long long scratch_elems, int grid,
                                 cudaStream_t s) {
  const long long elems = p.m_a * p.n_b + p.m_a * p.m_b * p.n_c;
  const size_t tbytes = sizeof(T) * (size_t)elems;
  const int use_smem = tbytes <= 48 * 1024;
  if (!use_smem && scratch_elems < (long long)grid * elems) return cudaErrorInvalidValue;
  kron3_generic_kernel<T><<<grid, 256, use_smem ? tbytes : 0, s>>>(p, scratch, use_smem);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scale(T* Y, long long batch, long long d1, long long d2, long long d3, long long ld,
                         long long ld2, long long sy, int beta_mode, T beta, int grid, cudaStream_t s) {
  scale_kernel<T><<<grid, 256, 0, s>>>(Y, batch, d1, d2, d3, ld, ld2, sy, beta_mode, beta);
  return cudaGetLastError();
}

// Strided batch copy: entry p, element (i, j, k) of d1 x d2 x d3 from
// src[p*s_stride + i + j*s_ld + k*s_ld2] to dst[p*d_stride + i + j*d_ld + k*d_ld2].
// Thread per element in (i fastest) order: the tight side is fully coalesced,
// the strided side reads / writes runs of d1 contiguous elements. Only entry
// elements are touched (padding of either layout is never read or written).
template <typename T>
__global__ void __launch_bounds__(256) repack_kernel(const T* __restrict__ src, long long s_ld, long long s_ld2,
                                                     long long s_stride, T* __restrict__ dst, long long d_ld,
                                                     long long d_ld2, long long d_stride, int d1, int d2, int d3,
                                                     long long total) {
  const long long per = (long long)d1 * d2 * d3;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / per;
    const int r = (int)(t - p * per);
    const int i = r % d1, jk = r / d1, j = jk % d2, k = jk / d2;
    dst[p * d_stride + i + j * d_ld + k * d_ld2] = src[p * s_stride + i + j * s_ld + k * s_ld2];
  }
}

// Square entries (n <= 16, the repack path of the fast kernels): the entry
// shape is compile-time, and a CTA walks groups of EPB whole entries (~2K
// elements) with a FIXED per-thread set of U element slots, so the index split
// and the in-entry offsets of both layouts are computed once per thread; per
// element only the group base moves (thread per element in tight order: the
// tight side is fully coalesced, the strided side reads / writes runs of n).
template <typename T, int N, int D3>
__global__ void __launch_bounds__(256) repack_sq_kernel(const T* __restrict__ src, long long s_ld, long long s_ld2,
                                                        long long s_stride, T* __restrict__ dst, long long d_ld,
                                                        long long d_ld2, long long d_stride, long long batch) {
  constexpr int PER = N * N * D3;
  constexpr int EPB = PER >= 2048 ? 1 : 2048 / PER;  // entries per group
  constexpr int TOT = EPB * PER;
  constexpr int U = (TOT + 255) / 256;
  long long soff[U], doff[U];
  int eix[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int t = (int)threadIdx.x + 256 * u;
    const int e = t / PER, r = t - e * PER;
    const int i = r % N, jk = r / N, j = jk % N, k = jk / N;
    eix[u] = t < TOT ? e : EPB;  // EPB: slot unused
    soff[u] = e * s_stride + i + j * s_ld + k * s_ld2;
    doff[u] = e * d_stride + i + j * d_ld + k * d_ld2;
  }
  pdl_enter();  // launched with programmatic serialization: the previous kernel's tail overlaps this launch
  for (long long g = blockIdx.x; g * EPB < batch; g += gridDim.x) {
    const long long p0 = g * EPB;
    const int left = batch - p0 < EPB ? (int)(batch - p0) : EPB;
    const T* sg = src + p0 * s_stride;
    T* dg = dst + p0 * d_stride;
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (eix[u] < left) v[u] = sg[soff[u]];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (eix[u] < left) dg[doff[u]] = v[u];
  }
}

template <typename T, int N>
static bool launch_repack_sq(const T* src, long long s_ld, long long s_ld2, long long s_stride, T* dst, long long d_ld,
                             long long d_ld2, long long d_stride, int n, int d3, long long total, int grid,
                             cudaStream_t s) {
  if constexpr (N > 1) {
    if (n != N) return launch_repack_sq<T, N - 1>(src, s_ld, s_ld2, s_stride, dst, d_ld, d_ld2, d_stride, n, d3, total,
                                                  grid, s);
  } else if (n != 1) {
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256u);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto kern = d3 == 1 ? repack_sq_kernel<T, N, 1> : repack_sq_kernel<T, N, N>;
  const long long per = (long long)N * N * (d3 == 1 ? 1 : N), epb = per >= 2048 ? 1 : 2048 / per;
  const long long batch = total / per, groups = (batch + epb - 1) / epb;
  cfg.gridDim = dim3((unsigned)(groups < grid ? groups : grid));
  cudaLaunchKernelEx(&cfg, kern, src, s_ld, s_ld2, s_stride, dst, d_ld, d_ld2, d_stride, batch);
  return true;
}

template <typename T>
cudaError_t launch_repack(const T* src, long long s_ld, long long s_ld2, long long s_stride, T* dst, long long d_ld,
                          long long d_ld2, long long d_stride, int d1, int d2, int d3, long long batch, int sm_count,
                          cudaStream_t s) {
  const long long total = batch * d1 * d2 * d3;
  if (total <= 0) return cudaSuccess;
  const long long want = (total + 255) / 256, cap = (long long)sm_count * 16;
  const int grid = (int)(want < cap ? want : cap);
  if (d1 == d2 && d1 >= 1 && d1 <= 16 && (d3 == 1 || d3 == d1) &&
      launch_repack_sq<T, 16>(src, s_ld, s_ld2, s_stride, dst, d_ld, d_ld2, d_stride, d1, d3, total, grid, s))
    return cudaGetLastError();
  repack_kernel<T><<<grid, 256, 0, s>>>(src, s_ld, s_ld2, s_stride, dst, d_ld, d_ld2, d_stride, d1, d2, d3, total);
  return cudaGetLastError();
}

template cudaError_t launch_repack<float>(const float*, long long, long long, long long, float*, long long, long long,
                                          long long, int, int, int, long long, int, cudaStream_t);
template cudaError_t launch_repack<double>(const double*, long long, long long, long long, double*, long long,
                                           long long, long long, int, int, int, long long, int, cudaStream_t);

template cudaError_t launch_kron2_generic<float>(const Kron2Params<float>&, float*, long long, int, cudaStream_t);
template cudaError_t launch_kron2_generic<double>(const Kron2Params<double>&, double*, long long, int, cudaStream_t);
template cudaError_t launch_kron3_generic<float>(const Kron3Params<float>&, float*, long long, int, cudaStream_t);
template cudaError_t launch_kron3_generic<double>(const Kron3Params<double>&, double*, long long, int, cudaStream_t);
template cudaError_t launch_scale<float>(float*, long long, long long, long long, long long, long long, long long,
                                         long long, int, float, int, cudaStream_t);
template cudaError_t launch_scale<double>(double*, long long, long long, long long, long long, long long, long long,
                                          long long, int, double, int, cudaStream_t);

}  // namespace kb
