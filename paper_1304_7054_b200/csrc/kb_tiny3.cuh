// kb_tiny3.cuh -- 3-D kernel for tiny entries (n <= 4: 4 .. 256 bytes of fp32).
//
// One thread per entry: a warp cooperatively moves 32 contiguous entries
// HBM -> smem with coalesced loads (entry stride padded to an odd word count,
// so the per-thread reads below are bank-conflict-free), each lane runs the
// three contractions of its entry entirely in registers with A_r, B_r and
// fl(alpha C_r) as constant-bank (uniform register) operands, and the warp
// writes the 32 results back with coalesced stores. Same per-element FMA
// chains as the reference (kron3.hpp:147-163 / detail.hpp:38-59): T1 = A_r X
// (l ascending, from 0), T2 = T1 B_r^T (m ascending, from 0), Y = init +
// T2 fl(alpha C_r)^T (n ascending). No CTA barrier, no TMA: at these sizes
// the per-entry TMA / mbarrier work of the tiled kernels costs more than the
// bytes.
#pragma once

#include "kb_fast.cuh"

namespace kb {

template <typename T, int N>
struct Tiny3 {
  static constexpr int E = N * N * N;
  static constexpr int SE = E % 2 ? E : E + 1;  // odd element stride: per-lane entry reads hit distinct banks
  static constexpr int WARPS = 8;
  static constexpr size_t smem_bytes() { return sizeof(T) * (size_t)WARPS * 32 * SE; }
};

template <typename T, int N>
__global__ void __launch_bounds__(Tiny3<T, N>::WARPS * 32)
    kron3_tiny_kernel(const Kron3Params<T> p, const __grid_constant__ SqConsts3<T, N> kc, const long long ngroups) {
  using K = Tiny3<T, N>;
  constexpr int E = K::E, SE = K::SE, NN = N * N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* sm = reinterpret_cast<T*>(smem_raw) + warp * 32 * SE;
  for (long long g = (long long)blockIdx.x * K::WARPS + warp; g < ngroups; g += (long long)gridDim.x * K::WARPS) {
    const long long first = g * 32;
    const int valid = (int)(p.batch - first < 32 ? p.batch - first : 32);
    const T* xg = p.X + first * E;
    for (int idx = lane; idx < valid * E; idx += 32) sm[(idx / E) * SE + idx % E] = xg[idx];
    __syncwarp();
    if (lane < valid) {
      T v[E];
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = sm[lane * SE + k];
      // mode 1: T1(:, m, n) = A_r X(:, m, n), column by column in place
#pragma unroll
      for (int c = 0; c < NN; ++c) {
        T t[N];
#pragma unroll
        for (int i = 0; i < N; ++i) t[i] = T(0);
#pragma unroll
        for (int l = 0; l < N; ++l)
#pragma unroll
          for (int i = 0; i < N; ++i) t[i] = fma_rn(kc.a[i + l * N], v[l + c * N], t[i]);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i + c * N] = t[i];
      }
      // mode 2: T2(i, :, n) = T1(i, :, n) B_r^T, row by row in place
#pragma unroll
      for (int n = 0; n < N; ++n)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          T t[N];
#pragma unroll
          for (int j = 0; j < N; ++j) t[j] = T(0);
#pragma unroll
          for (int m = 0; m < N; ++m)
#pragma unroll
            for (int j = 0; j < N; ++j) t[j] = fma_rn(v[i + m * N + n * NN], kc.b[j * N + m], t[j]);
#pragma unroll
          for (int j = 0; j < N; ++j) v[i + j * N + n * NN] = t[j];
        }
      // mode 3: Y(i, j, :) = init + T2(i, j, :) fl(alpha C_r)^T, fiber by fiber
      const T* yp = p.Y + (first + lane) * p.sy;
#pragma unroll
      for (int f = 0; f < NN; ++f) {
        T t[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
          t[k] = p.beta_mode == kBetaZero ? T(0) : beta_init(p.beta_mode, p.beta, yp[f + k * NN]);
#pragma unroll
        for (int n = 0; n < N; ++n)
#pragma unroll
          for (int k = 0; k < N; ++k) t[k] = fma_rn(v[f + n * NN], kc.c[k * N + n], t[k]);
#pragma unroll
        for (int k = 0; k < N; ++k) sm[lane * SE + f + k * NN] = t[k];
      }
    }
    __syncwarp();
    T* yg = p.Y + first * E;
    for (int idx = lane; idx < valid * E; idx += 32) yg[idx] = sm[(idx / E) * SE + idx % E];
    __syncwarp();
  }
}

}  // namespace kb
