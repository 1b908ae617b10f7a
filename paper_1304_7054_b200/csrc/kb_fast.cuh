// kb_fast.cuh -- register-blocked sm_100a kernels for square n <= 16 kron2 / kron3.
//
// Hot path of the reference (kron2.hpp:92-107 / kron3.hpp:138-163 running
// detail.hpp:38-59 gemm_axpy_fixed<M> inside detail.hpp:156-180 run_chunked),
// re-designed for B200 instead of translated:
//
// * The op-resolved constant matrices are staged ONCE per persistent CTA in
//   shared memory (A in a per-row-block layout, w = fl(alpha*B_r) / B_r /
//   fl(alpha*C_r) row-major so a row is one broadcast vector load).
// * Operands stream HBM -> shared memory with cp.async (16 B LDGSTS when the
//   entry size allows), multi-stage ring, so loads of entry group g+S-1 are in
//   flight while group g computes. No register staging, no HBM round trip of
//   any intermediate: the 2-D tmp and the 3-D T1/T2 stay in registers / smem.
// * "row-owner" register blocking: TPI threads cooperate on one n x n entry
//   (or 3-D plane); thread q owns R = ceil(n/TPI) rows I_q of tmp and of Y,
//   so both contractions of kron2 run out of registers with the scalar
//   operand broadcast from smem; pairs of rows go through FFMA2
//   (fma.rn.f32x2) with a broadcast scalar -- two different output elements
//   per instruction, each still accumulated in ascending order.
// * Entry slots in smem are padded (constexpr slot_stride) so the IPW entries
//   a warp reads in one LDS phase fall into disjoint bank groups.
// * 3-D: mode-1 + mode-2 run per plane exactly like 2-D (alpha 1, beta 0),
//   T2 overwrites its own X plane in smem, then mode-3 fibers are read back
//   and contracted with fl(alpha*C_r): no workspace traffic.
// Output goes straight from registers to HBM with vector stores.
#pragma once

#include "kb_device.cuh"

namespace kb {

// ---------------------------------------------------------- configuration --

constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }

// widest element vector width (16/8/4-byte) dividing n for element size `es`
__host__ __device__ constexpr int vec_width(int n, int es) {
  return (n % (16 / es) == 0) ? 16 / es : ((es == 4 && n % 2 == 0) ? 2 : 1);
}

// Worst shared-memory bank multiplicity when `ways` accesses, `width`
// elements wide, start at k*stride (k < ways).
__host__ __device__ constexpr int bank_conflicts(int s, int width, int ways, int es) {
  int cnt[32] = {};
  const int wb = width * es / 4 > 0 ? width * es / 4 : 1;  // banks per access
  int worst = 0;
  for (int k = 0; k < ways; ++k)
    for (int b = 0; b < wb; ++b) {
      const int bank = (int)(((long long)k * s * es / 4 + b) % 32);
      if (++cnt[bank] > worst) worst = cnt[bank];
    }
  return worst;
}

// Smallest stride >= base, multiple of `align`, minimising the bank
// multiplicity of `ways` strided accesses (1 == conflict-free).
__host__ __device__ constexpr int bank_spread_stride(int base, int align, int width, int ways, int es) {
  const int first = ((base + align - 1) / align) * align;
  int best = first, best_c = 1 << 30;
  for (int s = first; s <= first + 32 * align; s += align) {
    const int c = bank_conflicts(s, width, ways, es);
    if (c < best_c) {
      best_c = c;
      best = s;
      if (c == 1) break;
    }
  }
  return best;
}

__host__ __device__ constexpr int align16_elems(int elems, int es) { return ((elems * es + 15) / 16) * 16 / es; }

template <typename T, int N>
struct SqCfg {
  static constexpr int ES = sizeof(T);
  // threads per entry (2-D) / per plane (3-D), and rows each owns
  static constexpr int TPI = ES == 4 ? (N <= 4 ? 1 : (N <= 10 ? 2 : 4)) : (N <= 4 ? 1 : (N <= 8 ? 2 : (N <= 12 ? 4 : 8)));
  static constexpr int R = ceil_div(N, TPI);
  static constexpr int IPW = 32 / TPI;  // entries (planes) per warp pass
  static constexpr int NN = N * N;
  static constexpr int VXC = vec_width(NN, ES);  // cp.async chunk (elements)
  static constexpr int VXR = vec_width(N, ES);   // smem column read width
  static constexpr int VR = vec_width(R, ES);    // R-row vector width (smem)
  // global Y row-block vector width: must also divide N so tight layouts align
  static constexpr int VY = vec_width(R % 4 == 0 && N % 4 == 0 ? 4 : (R % 2 == 0 && N % 2 == 0 ? 2 : 1), ES);
  static constexpr int VN = vec_width(N, ES);    // row-of-constant read width
  static constexpr int LANES_PER_PHASE = 128 / (VXR * ES) < 32 ? 128 / (VXR * ES) : 32;
  static constexpr int PLANES_PER_PHASE = LANES_PER_PHASE / TPI > 0 ? LANES_PER_PHASE / TPI : 1;
  // padded per-entry (2-D) / per-plane (3-D) stride in smem, in elements
  static constexpr int SLOT = bank_spread_stride(NN, VXC > VXR ? VXC : VXR, VXR, PLANES_PER_PHASE, ES);
  // A row-block layout: Ablk[q][l][R] with q-stride QS
  static constexpr int QS = bank_spread_stride(N * R, VR, VR, TPI < 128 / (VR * ES) ? TPI : 128 / (VR * ES), ES);
  // R-row vector accesses into an smem plane (T2 write / fiber read) are aligned
  static constexpr bool PLANE_VEC = (N % VR == 0) && (SLOT % VR == 0);
  // 16-byte aligned element offsets of the smem constants (A blocks, rows)
  static constexpr int A_ELEMS = align16_elems(TPI * QS, ES);
  static constexpr int ROW_ELEMS = align16_elems(N * N, ES);
};

// ------------------------------------------------------- constant staging --

// Ablk[q*QS + l*R + r] = A_r(q*R + r, l) (0 for padded rows >= N)
template <typename T, int N>
__device__ __forceinline__ void stage_a(T* ablk, const T* A, long long lda, int opa) {
  using C = SqCfg<T, N>;
  for (int t = threadIdx.x; t < C::TPI * N * C::R; t += blockDim.x) {
    const int r = t % C::R, l = (t / C::R) % N, q = t / (C::R * N);
    const int i = q * C::R + r;
    ablk[q * C::QS + l * C::R + r] = i < N ? op_at(A, lda, opa, i, l) : T(0);
  }
}

// W[j*N + m] = scale * M_r(j, m) (row j contiguous); scale applied as fl(alpha*x)
template <typename T, int N>
__device__ __forceinline__ void stage_rows(T* w, const T* M, long long ldm, int opm, T alpha, bool scale) {
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) {
    const int m = t % N, j = t / N;
    const T v = op_at(M, ldm, opm, j, m);
    w[j * N + m] = scale ? mul_rn(alpha, v) : v;
  }
}

// ------------------------------------------------------------- contraction --

// tmp(I_q, m) = sum_l A_r(I_q, l) Xop(l, m) for all m, from one smem plane.
// OPX = 0: plane holds Xop column-major (column m contiguous); m-outer.
// OPX = 1: plane holds X stored (= Xop^T), i.e. row l of Xop contiguous; l-outer.
template <typename T, int N, int OPX, int MB>
__device__ __forceinline__ void mode1(T (&t)[N][SqCfg<T, N>::R], const T* __restrict__ xs,
                                      const T* __restrict__ aq) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R;
#pragma unroll
  for (int m = 0; m < N; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) t[m][r] = T(0);
  if constexpr (OPX == 0) {
#pragma unroll
    for (int m0 = 0; m0 < N; m0 += MB) {
      T xc[MB][N];
#pragma unroll
      for (int mm = 0; mm < MB; ++mm)
        if (m0 + mm < N) lds_n<N, C::VXR>(xc[mm], xs + (m0 + mm) * N);
#pragma unroll
      for (int l = 0; l < N; ++l) {
        T a[R];
        lds_n<R, C::VR>(a, aq + l * R);
#pragma unroll
        for (int mm = 0; mm < MB; ++mm)
          if (m0 + mm < N) axpy_rows<R>(t[m0 + mm], a, xc[mm][l]);
      }
    }
  } else {
#pragma unroll
    for (int l = 0; l < N; ++l) {
      T xr[N];
      lds_n<N, C::VXR>(xr, xs + l * N);
      T a[R];
      lds_n<R, C::VR>(a, aq + l * R);
#pragma unroll
      for (int m = 0; m < N; ++m) axpy_rows<R>(t[m], a, xr[m]);
    }
  }
}

// ---------------------------------------------------------------- kron2 ---

// Launch/tiling policy; V selects a tuning variant (V = 0 is the default).
template <typename T, int N, int V = 0>
struct Kron2Fast {
  using C = SqCfg<T, N>;
  static constexpr int WARPS = V == 2 ? 4 : (V == 3 ? 12 : 8);
  static constexpr int STAGES = V == 2 ? 4 : (V == 3 ? 2 : 3);
  static constexpr int MB = V == 1 ? 2 : 4;  // X columns held per mode-1 block
  static constexpr int JB = V == 3 ? 4 : 2;  // Y columns per mode-2 block
  static constexpr int RING = C::IPW * C::SLOT;  // elements per warp stage
  static constexpr size_t smem_bytes() {
    return sizeof(T) * ((size_t)C::A_ELEMS + (size_t)C::ROW_ELEMS + (size_t)WARPS * STAGES * RING);
  }
};

template <typename T, int N, int OPX, int V>
__global__ void __launch_bounds__(Kron2Fast<T, N, V>::WARPS * 32)
    kron2_sq_kernel(const Kron2Params<T> p, const long long ngroups) {
  using K = Kron2Fast<T, N, V>;
  using C = SqCfg<T, N>;
  constexpr int R = C::R, TPI = C::TPI, IPW = C::IPW, NN = C::NN, VXC = C::VXC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ablk = reinterpret_cast<T*>(smem_raw);
  T* wrow = ablk + C::A_ELEMS;
  T* ring = wrow + C::ROW_ELEMS;

  stage_a<T, N>(ablk, p.A, p.lda, p.opa);
  stage_rows<T, N>(wrow, p.B, p.ldb, p.opb, p.alpha, true);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wring = ring + warp * K::STAGES * K::RING;
  const long long gw = (long long)blockIdx.x * K::WARPS + warp;
  const long long gstride = (long long)gridDim.x * K::WARPS;

  // cp.async one group of IPW entries into a stage (zero-fill past the batch)
  auto issue = [&](long long g, int stage) {
    if (g < ngroups) {
      T* dst = wring + stage * K::RING;
      constexpr int CPI = NN / VXC;  // chunks per entry
      for (int c = lane; c < IPW * CPI; c += 32) {
        const int e = c / CPI, r = c % CPI;
        const long long item = g * IPW + e;
        const bool ok = item < p.batch;
        const T* src = p.X + (ok ? item : 0) * p.sx + r * VXC;
        cp_async<VXC * sizeof(T)>(dst + e * C::SLOT + r * VXC, src, ok);
      }
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < K::STAGES - 1; ++s) issue(gw + s * gstride, s);

  const int slot = lane / TPI, q = lane % TPI;
  const T* aq = ablk + q * C::QS;
  int stage = 0;
  for (long long g = gw; g < ngroups; g += gstride) {
    issue(g + (K::STAGES - 1) * gstride, (stage + K::STAGES - 1) % K::STAGES);
    cp_async_wait<K::STAGES - 1>();
    __syncwarp();
    const long long item = g * IPW + slot;
    if (slot < IPW && item < p.batch) {
      const T* xs = wring + stage * K::RING + slot * C::SLOT;
      T t[N][R];
      mode1<T, N, OPX, K::MB>(t, xs, aq);
      T* yb = p.Y + item * p.sy + q * R;
      const int rows = N - q * R;  // valid rows of this block (>= R unless padded)
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += K::JB) {
        T w[K::JB][N];
        T y[K::JB][R];
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj) {
          if (j0 + jj < N) {
            lds_n<N, C::VN>(w[jj], wrow + (j0 + jj) * N);
            if (p.beta_mode == kBetaZero) {
#pragma unroll
              for (int r = 0; r < R; ++r) y[jj][r] = T(0);
            } else {
              T* yc = yb + (long long)(j0 + jj) * p.ldy;
              if (R * TPI == N || rows >= R) {
                ldg_n<R, C::VY>(y[jj], yc);
              } else {
#pragma unroll
                for (int r = 0; r < R; ++r) y[jj][r] = r < rows ? yc[r] : T(0);
              }
#pragma unroll
              for (int r = 0; r < R; ++r) y[jj][r] = beta_init(p.beta_mode, p.beta, y[jj][r]);
            }
          }
        }
#pragma unroll
        for (int m = 0; m < N; ++m)
#pragma unroll
          for (int jj = 0; jj < K::JB; ++jj)
            if (j0 + jj < N) axpy_rows<R>(y[jj], t[m], w[jj][m]);
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj) {
          if (j0 + jj < N) {
            T* yc = yb + (long long)(j0 + jj) * p.ldy;
            if (R * TPI == N || rows >= R) {
              stg_n<R, C::VY>(yc, y[jj]);
            } else {
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (r < rows) yc[r] = y[jj][r];
            }
          }
        }
      }
    }
    __syncwarp();
    stage = (stage + 1) % K::STAGES;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- kron3 ---

template <typename T, int N, int V = 0>
struct Kron3Fast {
  using C = SqCfg<T, N>;
  static constexpr int PT = N * C::TPI;  // threads per entry
  static constexpr int MAXT = V == 0 ? 256 : (V == 3 ? 64 : 128);
  static constexpr int IT = (MAXT / PT) > 0 ? MAXT / PT : 1;  // entries per tile
  static constexpr int THREADS = IT * PT;
  static constexpr int STAGES = 2;
  static constexpr int MB = (V == 2 || V == 3) ? 2 : 4;
  static constexpr int JB = 2;
  static constexpr int KB = 2;
  static constexpr int ITEM = N * C::SLOT;  // padded entry stride (planes at SLOT)
  static constexpr int TILE = IT * ITEM;
  static constexpr size_t smem_bytes() {
    return sizeof(T) * ((size_t)C::A_ELEMS + 2 * (size_t)C::ROW_ELEMS + (size_t)STAGES * TILE);
  }
};

template <typename T, int N, int V>
__global__ void __launch_bounds__(Kron3Fast<T, N, V>::THREADS)
    kron3_sq_kernel(const Kron3Params<T> p, const long long ntiles) {
  using K = Kron3Fast<T, N, V>;
  using C = SqCfg<T, N>;
  constexpr int R = C::R, TPI = C::TPI, NN = C::NN, VXC = C::VXC, IT = K::IT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ablk = reinterpret_cast<T*>(smem_raw);
  T* brow = ablk + C::A_ELEMS;  // B_r rows (stage 1b: alpha 1, exact)
  T* crow = brow + C::ROW_ELEMS;        // fl(alpha*C_r) rows
  T* tiles = crow + C::ROW_ELEMS;

  stage_a<T, N>(ablk, p.A, p.lda, p.opa);
  stage_rows<T, N>(brow, p.B, p.ldb, p.opb, T(1), false);
  stage_rows<T, N>(crow, p.C, p.ldc, p.opc, p.alpha, true);
  __syncthreads();

  const int tid = threadIdx.x;
  auto issue = [&](long long tile, int stage) {
    if (tile < ntiles) {
      T* dst = tiles + stage * K::TILE;
      constexpr int CPP = NN / VXC;       // chunks per plane
      constexpr int CPE = N * CPP;        // chunks per entry
      for (int c = tid; c < IT * CPE; c += K::THREADS) {
        const int e = c / CPE, rr = c % CPE, n = rr / CPP, r = rr % CPP;
        const long long item = tile * IT + e;
        const bool ok = item < p.batch;
        const T* src = p.X + (ok ? item : 0) * p.sx + (long long)n * NN + r * VXC;
        cp_async<VXC * sizeof(T)>(dst + e * K::ITEM + n * C::SLOT + r * VXC, src, ok);
      }
    }
    cp_async_commit();
  };

  issue(blockIdx.x, 0);
  const int task = tid / TPI, q = tid % TPI;  // plane task: entry task/N, plane task%N
  const int te = task / N, tn = task % N;
  const T* aq = ablk + q * C::QS;
  // mode-3 fiber block: entry fe, column j, rows I_q
  const int fe = tid / K::PT, fj = (tid % K::PT) / TPI;
  int stage = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    issue(tile + gridDim.x, stage ^ 1);
    cp_async_wait<1>();
    __syncthreads();
    T* buf = tiles + stage * K::TILE;
    const int rows = N - q * R;
    // ---- modes 1 and 2 on plane (te, tn): T2(I_q, :, tn) -> in place
    {
      T* xs = buf + te * K::ITEM + tn * C::SLOT;
      T t[N][R];
      mode1<T, N, 0, K::MB>(t, xs, aq);
      T t2[N][R];
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += K::JB) {
        T w[K::JB][N];
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj)
          if (j0 + jj < N) {
            lds_n<N, C::VN>(w[jj], brow + (j0 + jj) * N);
#pragma unroll
            for (int r = 0; r < R; ++r) t2[j0 + jj][r] = T(0);
          }
#pragma unroll
        for (int m = 0; m < N; ++m)
#pragma unroll
          for (int jj = 0; jj < K::JB; ++jj)
            if (j0 + jj < N) axpy_rows<R>(t2[j0 + jj], t[m], w[jj][m]);
      }
      __syncwarp();  // all TPI threads of this plane finished reading X
#pragma unroll
      for (int j = 0; j < N; ++j) {
        T* dst = xs + j * N + q * R;
        if (R * TPI == N || rows >= R) {
          if constexpr (C::PLANE_VEC) {
            // aligned vector store into smem
#pragma unroll
            for (int r = 0; r < R; r += C::VR) {
              if constexpr (C::VR * sizeof(T) == 16 && sizeof(T) == 4)
                *reinterpret_cast<float4*>(dst + r) = make_float4(t2[j][r], t2[j][r + 1], t2[j][r + 2], t2[j][r + 3]);
              else if constexpr (C::VR * sizeof(T) == 16)
                *reinterpret_cast<double2*>(dst + r) = make_double2(t2[j][r], t2[j][r + 1]);
              else if constexpr (C::VR == 2 && sizeof(T) == 4)
                *reinterpret_cast<float2*>(dst + r) = make_float2(t2[j][r], t2[j][r + 1]);
              else
                dst[r] = t2[j][r];
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) dst[r] = t2[j][r];
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < rows) dst[r] = t2[j][r];
        }
      }
    }
    __syncthreads();
    // ---- mode 3 on fibers (fe, fj, I_q): Y(I_q, fj, k) for all k
    {
      const long long item = tile * IT + fe;
      if (item < p.batch) {
        const T* fb = buf + fe * K::ITEM + fj * N + q * R;
        T f[N][R];
#pragma unroll
        for (int n = 0; n < N; ++n) {
          if (R * TPI == N || rows >= R) {
            if constexpr (C::PLANE_VEC)
              lds_n<R, C::VR>(f[n], fb + n * C::SLOT);
            else {
#pragma unroll
              for (int r = 0; r < R; ++r) f[n][r] = fb[n * C::SLOT + r];
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) f[n][r] = r < rows ? fb[n * C::SLOT + r] : T(0);
          }
        }
        T* yb = p.Y + item * p.sy + (long long)fj * p.ldy + q * R;
#pragma unroll
        for (int k0 = 0; k0 < N; k0 += K::KB) {
          T w[K::KB][N];
          T y[K::KB][R];
#pragma unroll
          for (int kk = 0; kk < K::KB; ++kk) {
            if (k0 + kk < N) {
              lds_n<N, C::VN>(w[kk], crow + (k0 + kk) * N);
              if (p.beta_mode == kBetaZero) {
#pragma unroll
                for (int r = 0; r < R; ++r) y[kk][r] = T(0);
              } else {
                const T* yc = yb + (long long)(k0 + kk) * p.ldy2;
                if (R * TPI == N || rows >= R) {
                  ldg_n<R, C::VY>(y[kk], yc);
                } else {
#pragma unroll
                  for (int r = 0; r < R; ++r) y[kk][r] = r < rows ? yc[r] : T(0);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) y[kk][r] = beta_init(p.beta_mode, p.beta, y[kk][r]);
              }
            }
          }
#pragma unroll
          for (int n = 0; n < N; ++n)
#pragma unroll
            for (int kk = 0; kk < K::KB; ++kk)
              if (k0 + kk < N) axpy_rows<R>(y[kk], f[n], w[kk][n]);
#pragma unroll
          for (int kk = 0; kk < K::KB; ++kk) {
            if (k0 + kk < N) {
              T* yc = yb + (long long)(k0 + kk) * p.ldy2;
              if (R * TPI == N || rows >= R) {
                stg_n<R, C::VY>(yc, y[kk]);
              } else {
#pragma unroll
                for (int r = 0; r < R; ++r)
                  if (r < rows) yc[r] = y[kk][r];
              }
            }
          }
        }
      }
    }
    __syncthreads();
    stage ^= 1;
  }
  cp_async_wait<0>();
}

}  // namespace kb
