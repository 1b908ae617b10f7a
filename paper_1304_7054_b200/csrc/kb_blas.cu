// kb_blas.cu -- the two other batched operators of the reference's umbrella
// API (README.md:19-24), on the same launcher as kron2/kron3:
//
//   kron1  (proj/include/kronbatch/kron1.hpp:17-62): y^p <- alpha op(A) x^p + beta y^p,
//          shared A, a batched GEMV. Reference arithmetic: gemm_axpy with
//          R = x^p (detail.hpp:38-117): per element init from beta, then
//          acc = fma(A_r(i, kk), fl(alpha x[kk]), acc), kk ascending.
//   gemm_a (proj/include/kronbatch/gemm_a.hpp:18-76): C^p <- alpha op(A^p) op(B) + beta C^p,
//          varying A, shared B. op_a = N: gemm_axpy with S = A^p, R = B_r
//          (w = fl(alpha B_r(kk, c))); op_a = T: gemm_dot (detail.hpp:119-135):
//          acc = sum_kk A^p(kk, i) B_r(kk, c) from 0, then
//          fma(alpha, acc, beta == 0 ? 0 : fl(beta C)).
//
// Both are HBM-bound streaming operators (AI ~ n/4 .. n/2 flop/B). At square
// n <= 16 with contiguous entries kron1 runs kron1_sq_kernel and gemm_a
// gemm_a_sq_kernel (below); the general kernels use one thread
// per output element, consecutive threads on consecutive rows of one entry so
// the per-entry operand reads broadcast through L1 and the output writes are
// coalesced; the shared matrix is read through the read-only path (it stays
// in L1/L2). Any shape, op and stride; identical arithmetic to the CPU path.
#include <cstdlib>

#include "kb_kernels.h"

namespace kb {

template <typename T>
__global__ void kron1_kernel(const T* __restrict__ A, long long lda, int opa, const T* __restrict__ X,
                             long long sx, T* __restrict__ Y, long long sy, long long m, long long n,
                             long long batch, T alpha, int beta_mode, T beta) {
  const long long total = batch * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / m, i = t - p * m;
    const T* x = X + p * sx;
    T* y = Y + p * sy + i;
    T acc = beta_mode == kBetaZero ? T(0) : beta_init(beta_mode, beta, *y);
    for (long long kk = 0; kk < n; ++kk) {
      const T w = mul_rn(alpha, __ldg(x + kk));
      acc = fma_rn(__ldg(opa ? A + kk + i * lda : A + i + kk * lda), w, acc);
    }
    *y = acc;
  }
}

template <typename T>
__global__ void gemm_a_kernel(const T* __restrict__ A, long long lda, long long sa, int opa,
                              const T* __restrict__ B, long long ldb, int opb, T* __restrict__ Cm, long long ldc,
                              long long sc, long long m, long long n, long long k, long long batch, T alpha,
                              int beta_mode, T beta) {
  const long long per = m * n, total = batch * per;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / per, r = t - p * per, c = r / m, i = r - c * m;
    const T* a = A + p * sa;
    T* out = Cm + p * sc + i + c * ldc;
    auto b_at = [&](long long kk) { return __ldg(opb ? B + c + kk * ldb : B + kk + c * ldb); };  // B_r(kk, c)
    if (!opa) {  // gemm_axpy: init, then + A(i, kk) * fl(alpha B_r(kk, c))
      T acc = beta_mode == kBetaZero ? T(0) : beta_init(beta_mode, beta, *out);
      for (long long kk = 0; kk < k; ++kk) acc = fma_rn(__ldg(a + i + kk * lda), mul_rn(alpha, b_at(kk)), acc);
      *out = acc;
    } else {  // gemm_dot: plain dot from 0, then alpha * acc + beta * C
      T acc = T(0);
      for (long long kk = 0; kk < k; ++kk) acc = fma_rn(__ldg(a + kk + i * lda), b_at(kk), acc);
      const T init = beta_mode == kBetaZero ? T(0) : mul_rn(beta, *out);
      *out = fma_rn(alpha, acc, init);
    }
  }
}

// ---- kron1, square n <= 16 with contiguous entries: one thread per entry.
// A warp stages its 32 entries' x through smem with coalesced loads (odd
// element stride, so the per-lane reads are conflict-free), each lane forms
// y = init + A_r fl(alpha x) with A_r column pairs from the constant bank
// (FFMA2 R.F32 x UR.F32x2 -- two rows, one scalar), and the warp writes the
// results back coalesced.
template <typename T, int N>
struct K1Consts {
  T a[N * N];  // a[i + l*N] = A_r(i, l)
};

template <typename T, int N>
__global__ void __launch_bounds__(256) kron1_sq_kernel(const T* __restrict__ X, T* __restrict__ Y, long long batch,
                                                       T alpha, int beta_mode, T beta,
                                                       const __grid_constant__ K1Consts<T, N> kc) {
  constexpr int SE = N % 2 ? N : N + 1;
  __shared__ T sm[8][32 * SE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* s = sm[warp];
  const long long ngroups = (batch + 31) / 32;
  for (long long g = (long long)blockIdx.x * 8 + warp; g < ngroups; g += (long long)gridDim.x * 8) {
    const long long first = g * 32;
    const int valid = (int)(batch - first < 32 ? batch - first : 32);
    if (valid == 32) {  // full group: all N loads of this lane in flight before the smem stores
      T v[N];
#pragma unroll
      for (int t = 0; t < N; ++t) v[t] = __ldcs(X + first * N + lane + 32 * t);
#pragma unroll
      for (int t = 0; t < N; ++t) {
        const int idx = lane + 32 * t;
        s[(idx / N) * SE + idx % N] = v[t];
      }
    } else {
      for (int idx = lane; idx < valid * N; idx += 32) s[(idx / N) * SE + idx % N] = X[first * N + idx];
    }
    __syncwarp();
    if (lane < valid) {
      T acc[N];
      const T* yp = Y + (first + lane) * N;
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = beta_mode == kBetaZero ? T(0) : beta_init(beta_mode, beta, yp[i]);
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const T w = mul_rn(alpha, s[lane * SE + l]);
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int i = 0; i + 1 < N; i += 2) {
            const float2 d = ffma2_s(make_float2(kc.a[i + l * N], kc.a[i + 1 + l * N]), w,
                                     make_float2(acc[i], acc[i + 1]));
            acc[i] = d.x;
            acc[i + 1] = d.y;
          }
          if constexpr (N % 2) acc[N - 1] = fma_rn(kc.a[N - 1 + l * N], w, acc[N - 1]);
        } else {
#pragma unroll
          for (int i = 0; i < N; ++i) acc[i] = fma_rn(kc.a[i + l * N], w, acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < N; ++i) s[lane * SE + i] = acc[i];  // this lane's own slot: no cross-lane hazard
    }
    __syncwarp();
    if (valid == 32) {
#pragma unroll
      for (int t = 0; t < N; ++t) {
        const int idx = lane + 32 * t;
        __stcs(Y + first * N + idx, s[(idx / N) * SE + idx % N]);
      }
    } else {
      for (int idx = lane; idx < valid * N; idx += 32) Y[first * N + idx] = s[(idx / N) * SE + idx % N];
    }
    __syncwarp();
  }
}

template <typename T, int N>
static cudaError_t launch_kron1_sq_n(const T* ha, const T* X, T* Y, long long batch, T alpha, int beta_mode, T beta,
                                     int sm_count, cudaStream_t s) {
  K1Consts<T, N> kc;
  for (int i = 0; i < N * N; ++i) kc.a[i] = ha[i];
  const long long want = ((batch + 31) / 32 + 7) / 8;
  const int grid = (int)(want < (long long)sm_count * 8 ? want : (long long)sm_count * 8);
  kron1_sq_kernel<T, N><<<grid > 0 ? grid : 1, 256, 0, s>>>(X, Y, batch, alpha, beta_mode, beta, kc);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_kron1_sq(int n, const T* ha, const T* X, T* Y, long long batch, T alpha, int beta_mode, T beta,
                            int sm_count, cudaStream_t s) {
  switch (n) {
#define KB_K1(N) \
  case N: return launch_kron1_sq_n<T, N>(ha, X, Y, batch, alpha, beta_mode, beta, sm_count, s);
    KB_K1(1) KB_K1(2) KB_K1(3) KB_K1(4) KB_K1(5) KB_K1(6) KB_K1(7) KB_K1(8)
    KB_K1(9) KB_K1(10) KB_K1(11) KB_K1(12) KB_K1(13) KB_K1(14) KB_K1(15) KB_K1(16)
#undef KB_K1
    default: return cudaErrorNotSupported;
  }
}

// ---- gemm_a, square n <= 16 with tight entries (lda = n, entry stride n*n):
// one thread per (entry, output column c). A CTA tile of E = 256/n entries is
// copied to smem (fp64: element-granular cp.async, two stages, so the next
// tile is in flight while this one computes; fp32: one stage, loads batched in
// registers -- the faster choice per dtype), with op(A) resolved on the way in (column kk of
// op(A) contiguous at an even stride CS, entries padded apart, so the row-pair
// reads are 8-byte LDS that the n threads of one entry broadcast). Thread c
// runs the reference's per-column order: op N (gemm_axpy) acc = init, then
// acc_i = fma(op(A)(i, kk), w(kk, c), acc_i) with w = fl(alpha B_r) folded on
// the host; op T (gemm_dot) acc from 0 with w = B_r, then fma(alpha, acc, init).
// Rows pair into FFMA2 (two rows, one scalar). Results go back through the same
// smem tile so the C stores are coalesced.
template <typename T, int N>
struct GaConsts {
  T w[N * N];  // w[kk + c*N] = fl(alpha B_r(kk, c)) (op_a N) or B_r(kk, c) (op_a T)
};

template <typename T, int N>
struct GaTile {
  // column stride: fp32 a multiple of 4 (16-byte LDS of 4 rows), fp64 even;
  // the pad shifts consecutive columns across banks for the op-T staging stores
  static constexpr int CS = sizeof(T) == 4 ? (N % 4 == 0 ? N + 4 : (N + 3) / 4 * 4) : (N % 2 ? N + 1 : N + 2);
  static constexpr int EST = (N * CS + 3) / 4 * 4 + 4;       // entry stride (16-B multiple, bank-shifted)
  static constexpr int E = 256 / N;                           // entries per tile
  // fp64: two cp.async stages (measured faster); fp32: one stage, register-batched loads
  static constexpr bool PIPE = sizeof(T) == 8;
  static constexpr int STAGES = PIPE ? 2 : 1;
};

template <typename T, int N, bool OPT>
__global__ void __launch_bounds__(256) gemm_a_sq_kernel(const T* __restrict__ A, T* __restrict__ Cm, long long batch,
                                                        T alpha, int beta_mode, T beta,
                                                        const __grid_constant__ GaConsts<T, N> gc) {
  using G = GaTile<T, N>;
  constexpr int NN = N * N, CS = G::CS, EST = G::EST, E = G::E, TS = E * EST;
  extern __shared__ __align__(16) unsigned char ga_smem[];
  T* sa = reinterpret_cast<T*>(ga_smem);  // two stages of TS: tile t computes while tile t+1 lands
  T* sw = sa + G::STAGES * TS;
  const int tid = threadIdx.x;
  for (int i = tid; i < NN; i += 256) sw[(i % N) * N + i / N] = gc.w[i];  // sw[kk*N + c]: lanes c read consecutive words
  const int el = tid / N, c = tid % N;
  const long long ntiles = (batch + E - 1) / E;
  // element-granular async copies resolve op(A) on the way in: op N r = i + kk*N,
  // op T r = kk + i*N (A^p(kk, i) = op(A)(i, kk)); always one commit group per call
  auto issue = [&](long long tile, int st) {
    if (tile < ntiles) {
      const long long first = tile * E;
      const int lim = (int)(batch - first < E ? batch - first : E) * NN;
      const T* src = A + first * NN;
      T* dst = sa + st * TS;
#pragma unroll 4
      for (int g = tid; g < lim; g += 256) {
        const int e = g / NN, r = g - e * NN;
        const int i = OPT ? r / N : r % N, kk = OPT ? r % N : r / N;
        cp_async<sizeof(T)>(dst + e * EST + i + kk * CS, src + g, true);
      }
    }
    cp_async_commit();
  };
  int st = 0;
  if constexpr (G::PIPE) issue(blockIdx.x, 0);
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, st ^= (G::PIPE ? 1 : 0)) {
    const long long first = tile * E;
    const int valid = (int)(batch - first < E ? batch - first : E);
    __syncthreads();  // the stage being refilled (previous output staging) is drained; sw is filled
    if constexpr (G::PIPE) {
      issue(tile + gridDim.x, st ^ 1);
      cp_async_wait<1>();
    } else {
      // one stage: all of this thread's loads in flight before the first smem store
      constexpr int LPT = (E * NN + 255) / 256;
      const int lim = valid * NN;
      const T* src = A + first * NN;
      T v[LPT];
#pragma unroll
      for (int t = 0; t < LPT; ++t)
        if (tid + t * 256 < lim) v[t] = __ldcs(src + tid + t * 256);
#pragma unroll
      for (int t = 0; t < LPT; ++t) {
        const int g = tid + t * 256;
        if (g < lim) {
          const int e = g / NN, r = g - e * NN;
          const int i = OPT ? r / N : r % N, kk = OPT ? r % N : r / N;
          sa[e * EST + i + kk * CS] = v[t];
        }
      }
    }
    __syncthreads();  // this tile's op(A) is visible to every thread
    T* sst = sa + st * TS;
    T acc[N];
    const bool act = el < valid;
    T* cg = Cm + (first + el) * NN + c * N;  // column c of this thread's C entry
    if (act) {
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = OPT || beta_mode == kBetaZero ? T(0) : beta_init(beta_mode, beta, cg[i]);
      const T* ae = sst + el * EST;
#pragma unroll
      for (int kk = 0; kk < N; ++kk) {
        const T w = sw[kk * N + c];
        const T* col = ae + kk * CS;
        if constexpr (sizeof(T) == 4) {
          float a[(N + 3) / 4 * 4];
#pragma unroll
          for (int i = 0; i < N; i += 4) *reinterpret_cast<float4*>(a + i) = *reinterpret_cast<const float4*>(col + i);
#pragma unroll
          for (int i = 0; i + 1 < N; i += 2) {
            const float2 d = ffma2_s(make_float2(a[i], a[i + 1]), w, make_float2(acc[i], acc[i + 1]));
            acc[i] = d.x;
            acc[i + 1] = d.y;
          }
          if constexpr (N % 2) acc[N - 1] = fma_rn(a[N - 1], w, acc[N - 1]);
        } else {
#pragma unroll
          for (int i = 0; i < N; ++i) acc[i] = fma_rn(col[i], w, acc[i]);
        }
      }
      if constexpr (OPT) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const T init = beta_mode == kBetaZero ? T(0) : mul_rn(beta, cg[i]);
          acc[i] = fma_rn(alpha, acc[i], init);
        }
      }
    }
    __syncthreads();  // every thread is done reading op(A) out of this stage
    if (act) {
#pragma unroll
      for (int i = 0; i < N; ++i) sst[el * EST + i + c * CS] = acc[i];
    }
    __syncthreads();
    T* dst = Cm + first * NN;
#pragma unroll 4
    for (int g = tid; g < valid * NN; g += 256) {
      const int e = g / NN, r = g - e * NN;
      __stcs(dst + g, sst[e * EST + r % N + (r / N) * CS]);
    }
  }
  if constexpr (G::PIPE) cp_async_wait<0>();
}

// Warp-granular variant (the default for most sizes): each warp owns WE = 32/n entries (lane -> entry
// lane/n, column lane%n) in a private smem slice; no CTA barrier after the
// one-time w fill, so warps drift freely and hide each other's load latency.
template <typename T, int N>
struct GaWarp {
  static constexpr int CS = GaTile<T, N>::CS, EST = GaTile<T, N>::EST;
  static constexpr int WE = 32 / N;             // entries per warp group
  static constexpr int LPT = (WE * N * N + 31) / 32;  // loads per lane per group
  static constexpr int WARPS = 8;
};

template <typename T, int N, bool OPT>
__global__ void __launch_bounds__(256) gemm_a_sqw_kernel(const T* __restrict__ A, T* __restrict__ Cm, long long batch,
                                                         T alpha, int beta_mode, T beta,
                                                         const __grid_constant__ GaConsts<T, N> gc) {
  using G = GaWarp<T, N>;
  constexpr int NN = N * N, CS = G::CS, EST = G::EST, WE = G::WE, LPT = G::LPT;
  __shared__ __align__(16) T sa_all[G::WARPS * WE * EST];
  __shared__ T sw[NN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < NN; i += 256) sw[(i % N) * N + i / N] = gc.w[i];  // sw[kk*N + c]
  __syncthreads();
  T* sa = sa_all + warp * WE * EST;
  const int el = lane / N, c = lane % N;
  const long long ngroups = (batch + WE - 1) / WE;
  for (long long grp = (long long)blockIdx.x * G::WARPS + warp; grp < ngroups; grp += (long long)gridDim.x * G::WARPS) {
    const long long first = grp * WE;
    const int valid = (int)(batch - first < WE ? batch - first : WE);
    const int lim = valid * NN;
    const T* src = A + first * NN;
    {
      T v[LPT];
#pragma unroll
      for (int t = 0; t < LPT; ++t)
        if (lane + 32 * t < lim) v[t] = __ldcs(src + lane + 32 * t);
#pragma unroll
      for (int t = 0; t < LPT; ++t) {
        const int g = lane + 32 * t;
        if (g < lim) {
          const int e = g / NN, r = g - e * NN;
          const int i = OPT ? r / N : r % N, kk = OPT ? r % N : r / N;
          sa[e * EST + i + kk * CS] = v[t];
        }
      }
    }
    __syncwarp();
    T acc[N];
    const bool act = el < valid;
    T* cg = Cm + (first + el) * NN + c * N;
    if (act) {
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = OPT || beta_mode == kBetaZero ? T(0) : beta_init(beta_mode, beta, cg[i]);
      const T* ae = sa + el * EST;
#pragma unroll
      for (int kk = 0; kk < N; ++kk) {
        const T w = sw[kk * N + c];
        const T* col = ae + kk * CS;
        if constexpr (sizeof(T) == 4) {
          float a[(N + 3) / 4 * 4];
#pragma unroll
          for (int i = 0; i < N; i += 4) *reinterpret_cast<float4*>(a + i) = *reinterpret_cast<const float4*>(col + i);
#pragma unroll
          for (int i = 0; i + 1 < N; i += 2) {
            const float2 d = ffma2_s(make_float2(a[i], a[i + 1]), w, make_float2(acc[i], acc[i + 1]));
            acc[i] = d.x;
            acc[i + 1] = d.y;
          }
          if constexpr (N % 2) acc[N - 1] = fma_rn(a[N - 1], w, acc[N - 1]);
        } else {
#pragma unroll
          for (int i = 0; i < N; ++i) acc[i] = fma_rn(col[i], w, acc[i]);
        }
      }
      if constexpr (OPT) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const T init = beta_mode == kBetaZero ? T(0) : mul_rn(beta, cg[i]);
          acc[i] = fma_rn(alpha, acc[i], init);
        }
      }
    }
    __syncwarp();  // the warp is done reading op(A) out of its slice
    if (act) {
#pragma unroll
      for (int i = 0; i < N; ++i) sa[el * EST + i + c * CS] = acc[i];
    }
    __syncwarp();
    T* dst = Cm + first * NN;
#pragma unroll
    for (int t = 0; t < LPT; ++t) {
      const int g = lane + 32 * t;
      if (g < lim) __stcs(dst + g, sa[(g / NN) * EST + (g % NN) % N + ((g % NN) / N) * CS]);
    }
    __syncwarp();
  }
}

template <typename T, int N>
static cudaError_t launch_gemm_a_sq_n(bool opt, const T* hw, const T* A, T* Cm, long long batch, T alpha,
                                      int beta_mode, T beta, int sm_count, cudaStream_t s) {
  GaConsts<T, N> gc;
  for (int i = 0; i < N * N; ++i) gc.w[i] = hw[i];
  // warp-granular kernel by default; the CTA-tile kernel where it measured
  // faster (fp64 n = 12-15, profiles/r01_gemm_a_square.txt). KB_GA_WARP=0/1 forces one.
  static const int wv = [] { const char* e = std::getenv("KB_GA_WARP"); return e ? std::atoi(e) : -1; }();
  constexpr bool warp_default = !(sizeof(T) == 8 && N >= 12 && N <= 15);
  if (wv == 1 || (wv < 0 && warp_default)) {
    auto kw = opt ? gemm_a_sqw_kernel<T, N, true> : gemm_a_sqw_kernel<T, N, false>;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kw, 256, 0) != cudaSuccess || occ < 1) occ = 1;
    const long long ng = (batch + GaWarp<T, N>::WE - 1) / GaWarp<T, N>::WE;
    const long long want = (ng + 7) / 8, cap = (long long)sm_count * occ;
    const int grid = (int)(want < cap ? want : cap);
    kw<<<grid > 0 ? grid : 1, 256, 0, s>>>(A, Cm, batch, alpha, beta_mode, beta, gc);
    return cudaGetLastError();
  }
  const long long ntiles = (batch + GaTile<T, N>::E - 1) / GaTile<T, N>::E;
  auto kern = opt ? gemm_a_sq_kernel<T, N, true> : gemm_a_sq_kernel<T, N, false>;
  using G = GaTile<T, N>;
  const size_t smem = sizeof(T) * ((size_t)G::STAGES * G::E * G::EST + N * N);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem) != cudaSuccess || occ < 1) occ = 1;
  const long long cap = (long long)sm_count * occ;
  const int grid = (int)(ntiles < cap ? ntiles : cap);
  kern<<<grid > 0 ? grid : 1, 256, smem, s>>>(A, Cm, batch, alpha, beta_mode, beta, gc);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_gemm_a_sq(int n, bool opt, const T* hw, const T* A, T* Cm, long long batch, T alpha, int beta_mode,
                             T beta, int sm_count, cudaStream_t s) {
  switch (n) {
#define KB_GA(N) \
  case N: return launch_gemm_a_sq_n<T, N>(opt, hw, A, Cm, batch, alpha, beta_mode, beta, sm_count, s);
    KB_GA(1) KB_GA(2) KB_GA(3) KB_GA(4) KB_GA(5) KB_GA(6) KB_GA(7) KB_GA(8)
    KB_GA(9) KB_GA(10) KB_GA(11) KB_GA(12) KB_GA(13) KB_GA(14) KB_GA(15) KB_GA(16)
#undef KB_GA
    default: return cudaErrorNotSupported;
  }
}

template <typename T>
cudaError_t launch_kron1(const T* A, long long lda, int opa, const T* X, long long sx, T* Y, long long sy,
                         long long m, long long n, long long batch, T alpha, int beta_mode, T beta, int sm_count,
                         cudaStream_t s) {
  const long long total = batch * m;
  const int threads = 256;
  const long long want = (total + threads - 1) / threads;
  const int grid = (int)(want < (long long)sm_count * 16 ? want : (long long)sm_count * 16);
  kron1_kernel<T><<<grid, threads, 0, s>>>(A, lda, opa, X, sx, Y, sy, m, n, batch, alpha, beta_mode, beta);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_gemm_a(const T* A, long long lda, long long sa, int opa, const T* B, long long ldb, int opb, T* Cm,
                          long long ldc, long long sc, long long m, long long n, long long k, long long batch, T alpha,
                          int beta_mode, T beta, int sm_count, cudaStream_t s) {
  const long long total = batch * m * n;
  const int threads = 256;
  const long long want = (total + threads - 1) / threads;
  const int grid = (int)(want < (long long)sm_count * 16 ? want : (long long)sm_count * 16);
  gemm_a_kernel<T><<<grid, threads, 0, s>>>(A, lda, sa, opa, B, ldb, opb, Cm, ldc, sc, m, n, k, batch, alpha,
                                            beta_mode, beta);
  return cudaGetLastError();
}

template cudaError_t launch_kron1_sq<float>(int, const float*, const float*, float*, long long, float, int, float, int,
                                            cudaStream_t);
template cudaError_t launch_kron1_sq<double>(int, const double*, const double*, double*, long long, double, int, double,
                                             int, cudaStream_t);
template cudaError_t launch_gemm_a_sq<float>(int, bool, const float*, const float*, float*, long long, float, int,
                                             float, int, cudaStream_t);
template cudaError_t launch_gemm_a_sq<double>(int, bool, const double*, const double*, double*, long long, double, int,
                                              double, int, cudaStream_t);
template cudaError_t launch_kron1<float>(const float*, long long, int, const float*, long long, float*, long long,
                                         long long, long long, long long, float, int, float, int, cudaStream_t);
template cudaError_t launch_kron1<double>(const double*, long long, int, const double*, long long, double*, long long,
                                          long long, long long, long long, double, int, double, int, cudaStream_t);
template cudaError_t launch_gemm_a<float>(const float*, long long, long long, int, const float*, long long, int,
                                          float*, long long, long long, long long, long long, long long, long long,
                                          float, int, float, int, cudaStream_t);
template cudaError_t launch_gemm_a<double>(const double*, long long, long long, int, const double*, long long, int,
                                           double*, long long, long long, long long, long long, long long, long long,
                                           double, int, double, int, cudaStream_t);

}  // namespace kb
