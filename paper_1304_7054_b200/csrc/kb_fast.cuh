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
  // (odd n: entries stay contiguous, SLOT = NN, so a group of entries lands
  //  with one bulk copy of its 16-byte-aligned span; odd NN spreads banks anyway)
  static constexpr int SLOT = (NN * ES) % 16 == 0 ? bank_spread_stride(NN, VXC > VXR ? VXC : VXR, VXR, PLANES_PER_PHASE, ES)
                                                  : NN;
  // A row-block layout: Ablk[q][l][R] with q-stride QS
  static constexpr int QS = bank_spread_stride(N * R, VR, VR, TPI < 128 / (VR * ES) ? TPI : 128 / (VR * ES), ES);
  // R-row vector accesses into an smem plane (T2 write / fiber read) are aligned
  static constexpr bool PLANE_VEC = (N % VR == 0) && (SLOT % VR == 0);
  // 16-byte aligned element offsets of the smem constants (A blocks, rows)
  static constexpr int A_ELEMS = align16_elems(TPI * QS, ES);
  static constexpr int ROW_ELEMS = align16_elems(N * N, ES);
};

// Op-resolved constant matrices, passed BY VALUE as __grid_constant__ kernel
// parameters: the broadcast operands of the second/third contractions are read
// straight from the constant bank into uniform registers (LDCU -> FFMA2 UR
// operand), so they cost no shared-memory wavefronts and no LDS issue slots.
//   a[i + l*N] = A_r(i, l)            (staged once into smem per CTA)
//   w[j*N + m] = fl(alpha * B_r(j, m)) (2-D)
//   b[j*N + m] = B_r(j, m), c[k*N + n] = fl(alpha * C_r(k, n)) (3-D)
template <typename T, int N>
struct SqConsts2 {
  T a[N * N];
  T w[N * N];
};
template <typename T, int N>
struct SqConsts3 {
  T a[N * N];
  T b[N * N];
  T c[N * N];
};

// ------------------------------------------------------- constant staging --

// Ablk[q*QS + l*R + r] = A_r(q*R + r, l) from the resolved parameter copy
template <typename T, int N>
__device__ __forceinline__ void stage_a_param(T* ablk, const T (&a)[N * N]) {
  using C = SqCfg<T, N>;
  for (int t = threadIdx.x; t < C::TPI * N * C::R; t += blockDim.x) {
    const int r = t % C::R, l = (t / C::R) % N, q = t / (C::R * N);
    const int i = q * C::R + r;
    ablk[q * C::QS + l * C::R + r] = i < N ? a[i + l * N] : T(0);
  }
}

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
// All loops below are fully unrolled; operands are fetched from smem in
// vector chunks right before use so that only the accumulators stay live.
// Each accumulator receives its terms in ascending contraction index.

// tmp(I_q, m) = sum_l A_r(I_q, l) Xop(l, m) for all m, from one smem plane.
// OPX = 0: plane holds Xop column-major (column m contiguous): m-blocks of MB
//          columns, l in chunks of VXR (MB * R/2 independent FFMA2 chains).
// OPX = 1: plane holds X as stored (= Xop^T): row l of Xop contiguous; l-outer.
template <typename T, int N, int OPX, int MB>
__device__ __forceinline__ void mode1(T (&t)[N][SqCfg<T, N>::R], const T* __restrict__ xs,
                                      const T* __restrict__ aq) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R, LC = C::VXR;
#pragma unroll
  for (int m = 0; m < N; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) t[m][r] = T(0);
  if constexpr (OPX == 0) {
#pragma unroll
    for (int m0 = 0; m0 < N; m0 += MB) {
#pragma unroll
      for (int l0 = 0; l0 < N; l0 += LC) {
        T xc[MB][LC];
        T a[LC][R];
#pragma unroll
        for (int mm = 0; mm < MB; ++mm)
          if (m0 + mm < N) lds_vec<LC>(xc[mm], xs + (m0 + mm) * N + l0);
#pragma unroll
        for (int ll = 0; ll < LC; ++ll) lds_n<R, C::VR>(a[ll], aq + (l0 + ll) * R);
#pragma unroll
        for (int ll = 0; ll < LC; ++ll)
#pragma unroll
          for (int mm = 0; mm < MB; ++mm)
            if (m0 + mm < N) axpy_rows<R>(t[m0 + mm], a[ll], xc[mm][ll]);
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

// Mode 1 (OPX = 0) with this thread's A rows held in registers: ar[l][r] =
// A_r(q*R + r, l). Saves the per-m-block A re-reads (smem wavefronts).
template <typename T, int N, int MB>
__device__ __forceinline__ void mode1_areg(T (&t)[N][SqCfg<T, N>::R], const T* __restrict__ xs,
                                           const T (&ar)[N][SqCfg<T, N>::R]) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R, LC = C::VXR;
#pragma unroll
  for (int m = 0; m < N; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) t[m][r] = T(0);
#pragma unroll
  for (int m0 = 0; m0 < N; m0 += MB) {
#pragma unroll
    for (int l0 = 0; l0 < N; l0 += LC) {
      T xc[MB][LC];
#pragma unroll
      for (int mm = 0; mm < MB; ++mm)
        if (m0 + mm < N) lds_vec<LC>(xc[mm], xs + (m0 + mm) * N + l0);
#pragma unroll
      for (int ll = 0; ll < LC; ++ll)
#pragma unroll
        for (int mm = 0; mm < MB; ++mm)
          if (m0 + mm < N) axpy_rows<R>(t[m0 + mm], ar[l0 + ll], xc[mm][ll]);
    }
  }
}

// out[jj] (+)= sum_m t[m] * w(j0+jj, m) for jj < JB, m ascending; w rows
// contiguous in smem (broadcast reads), fetched VN elements at a time.
template <typename T, int N, int JB>
__device__ __forceinline__ void contract_rows(T (&out)[JB][SqCfg<T, N>::R], const T (&t)[N][SqCfg<T, N>::R],
                                              const T* __restrict__ wrow, int j0) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R, VN = C::VN;
#pragma unroll
  for (int m0 = 0; m0 < N; m0 += VN) {
    T wv[JB][VN];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj)
      if (j0 + jj < N) lds_vec<VN>(wv[jj], wrow + (j0 + jj) * N + m0);
#pragma unroll
    for (int mm = 0; mm < VN; ++mm)
#pragma unroll
      for (int jj = 0; jj < JB; ++jj)
        if (j0 + jj < N) axpy_rows<R>(out[jj], t[m0 + mm], wv[jj][mm]);
  }
}

// Same contraction with the w rows read from a __grid_constant__ parameter
// (compile-time offsets -> constant bank -> uniform registers).
template <typename T, int N, int JB>
__device__ __forceinline__ void contract_rows_c(T (&out)[JB][SqCfg<T, N>::R], const T (&t)[N][SqCfg<T, N>::R],
                                                const T (&w)[N * N], int j0) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R;
#pragma unroll
  for (int m = 0; m < N; ++m)
#pragma unroll
    for (int jj = 0; jj < JB; ++jj)
      if (j0 + jj < N) axpy_rows<R>(out[jj], t[m], w[(j0 + jj) * N + m]);
}

// Y(I_q, j) block init from beta (detail.hpp:45-51), reading the prior only when needed.
template <typename T, int N>
__device__ __forceinline__ void init_y(T (&y)[SqCfg<T, N>::R], const T* yc, int rows, int beta_mode, T beta) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R;
  if (beta_mode == kBetaZero) {
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] = T(0);
    return;
  }
  if (R * C::TPI == N || rows >= R) {
    ldg_n<R, C::VY>(y, yc);
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] = r < rows ? yc[r] : T(0);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) y[r] = beta_init(beta_mode, beta, y[r]);
}

template <typename T, int N>
__device__ __forceinline__ void store_y(T* yc, const T (&y)[SqCfg<T, N>::R], int rows) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R;
  if (R * C::TPI == N || rows >= R) {
    stg_n<R, C::VY>(yc, y);
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r < rows) yc[r] = y[r];
  }
}

// Store R rows (the valid prefix when the block is padded) to smem.
template <typename T, int N>
__device__ __forceinline__ void sts_rows(T* dst, const T (&v)[SqCfg<T, N>::R], int rows) {
  using C = SqCfg<T, N>;
  constexpr int R = C::R;
  if (R * C::TPI == N || rows >= R) {
    if constexpr (C::PLANE_VEC) {
#pragma unroll
      for (int r = 0; r < R; r += C::VR) {
        if constexpr (C::VR * sizeof(T) == 16 && sizeof(T) == 4)
          *reinterpret_cast<float4*>(dst + r) = make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]);
        else if constexpr (C::VR * sizeof(T) == 16)
          *reinterpret_cast<double2*>(dst + r) = make_double2(v[r], v[r + 1]);
        else if constexpr (C::VR == 2 && sizeof(T) == 4)
          *reinterpret_cast<float2*>(dst + r) = make_float2(v[r], v[r + 1]);
        else
          dst[r] = v[r];
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r] = v[r];
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r < rows) dst[r] = v[r];
  }
}

// ------------------------------------------------------ staged Y copy-out --
// Y blocks staged in shared memory (same element layout as the tight global
// entry / plane) leave with coalesced VW-element vector stores: consecutive
// threads write consecutive chunks, so a warp instruction covers 32 chunks of
// one contiguous span instead of 32 scattered R-row pieces. Used when the
// row-block stores would be narrower than 16 bytes (n % 4 != 0 fp32 ...).
//   chunk c of `nent` entries x `planes` planes x CPP chunks per plane:
//   smem  src + e*ent_stride + pl*plane_stride + r*VW
//   HBM   Y + e*sy + pl*NN + r*VW
template <typename T, int NN, int VW>
__device__ __forceinline__ void copy_out(T* __restrict__ Y, long long sy, const T* __restrict__ src, int ent_stride,
                                         int plane_stride, int planes, int nent, int tid, int nthreads) {
  constexpr int CPP = NN / VW;
  const int total = nent * planes * CPP;
  for (int c = tid; c < total; c += nthreads) {
    const int ep = c / CPP, r = c - ep * CPP;
    const int e = ep / planes, pl = ep - e * planes;
    T v[VW];
    lds_vec<VW>(v, src + e * ent_stride + pl * plane_stride + r * VW);
    stg_n<VW, VW>(Y + e * sy + (long long)pl * NN + r * VW, v);
  }
}

// ---------------------------------------------------------------- kron2 ---

// Launch/tiling policy; V selects a tuning variant (V = 0 is the default).
template <typename T, int N, int V = 0>
struct Kron2Fast {
  using C = SqCfg<T, N>;
  static constexpr bool F32 = sizeof(T) == 4;
  // V0 (default): 8 warps x 3 stages (two groups in flight per warp: 6.4 TB/s
  // at n = 16 fp32); V1: 12 x 2; V2: 16 x 1; V3: 12 x 2 with MB = JB = 2.
  static constexpr int WARPS = V == 0 ? 8 : (V == 1 ? 12 : (V == 2 ? 16 : 12));
  static constexpr int STAGES = V == 0 ? 3 : (V == 1 ? 2 : (V == 2 ? 1 : 2));
  static constexpr int MB = V == 3 ? 2 : 4;  // X columns per mode-1 block
  static constexpr int JB = V == 3 ? 2 : 4;  // Y columns per mode-2 block
  // whole entries are 16-byte multiples: one cp.async.bulk per entry
  static constexpr bool BULK = (C::NN * sizeof(T)) % 16 == 0;
  // odd n: + slack for the span copy's 16-byte rounding; stages stay 16-byte aligned
  static constexpr int RING = BULK ? C::IPW * C::SLOT
                                   : (C::IPW * C::SLOT + 32 / (int)sizeof(T) + 16 / (int)sizeof(T) - 1) /
                                         (16 / (int)sizeof(T)) * (16 / (int)sizeof(T));
  static constexpr size_t smem_bytes() {
    return sizeof(T) * ((size_t)C::A_ELEMS + (size_t)WARPS * STAGES * RING) +
           sizeof(unsigned long long) * WARPS * STAGES;
  }
};

template <typename T, int N, int OPX, int V, bool YS>
__global__ void __launch_bounds__(Kron2Fast<T, N, V>::WARPS * 32)
    kron2_sq_kernel(const Kron2Params<T> p, const __grid_constant__ SqConsts2<T, N> kc, const long long ngroups) {
  constexpr bool ystage = YS;  // Y staged through the entry's smem slot (compile-time: no dead code in the other)
  using K = Kron2Fast<T, N, V>;
  using C = SqCfg<T, N>;
  constexpr int R = C::R, TPI = C::TPI, IPW = C::IPW, NN = C::NN, VXC = C::VXC, S = K::STAGES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ablk = reinterpret_cast<T*>(smem_raw);
  T* ring = ablk + C::A_ELEMS;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + K::WARPS * S * K::RING);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // odd n with contiguous entries: one span bulk copy per group (mbarrier);
  // any other odd-n layout: element cp.async (commit groups)
  const bool span = !K::BULK && p.sx == NN;
  const bool use_bar = K::BULK || span;
  if (use_bar) {
    if (lane == 0)
      for (int s = 0; s < S; ++s) mbar_init(&bars[warp * S + s], 1);
    mbar_fence_init();
  }
  stage_a_param<T, N>(ablk, kc.a);
  __syncthreads();

  T* wring = ring + warp * S * K::RING;
  unsigned long long* wbar = bars + warp * S;
  const long long gw = (long long)blockIdx.x * K::WARPS + warp;
  const long long gstride = (long long)gridDim.x * K::WARPS;

  // ystage with a tight Y whose 16-byte phase matches the stage image: bulk
  // stores (odd n: one span per group; padded slots: one per entry) instead of
  // copy_out; a stage is refilled after this lane's stores have read it
  const bool ybulk = ystage && use_bar && p.ldy == N &&
                     (K::BULK ? (p.sy * (long long)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.Y) & 15) == 0
                              : p.sy == NN && ((reinterpret_cast<uintptr_t>(p.X) ^ reinterpret_cast<uintptr_t>(p.Y)) & 15) == 0);
  // start loading group g (IPW entries) into `stage`
  auto issue = [&](long long g, int stage) {
    if (g >= ngroups) {
      if (!use_bar) cp_async_commit();
      return;
    }
    if (ystage && use_bar) bulk_wait_read();
    T* dst = wring + stage * K::RING;
    const long long first = g * IPW;
    const int valid = (int)(p.batch - first < IPW ? p.batch - first : IPW);
    if constexpr (K::BULK) {
      if (lane == 0) mbar_arrive_expect_tx(&wbar[stage], (unsigned)(valid * NN * sizeof(T)));
      __syncwarp();
      if (lane < valid) bulk_g2s(dst + lane * C::SLOT, p.X + (first + lane) * p.sx, NN * sizeof(T), &wbar[stage]);
    } else if (span) {
      if (lane == 0) {
        uintptr_t lo, hi;
        group_span(p.X, p.batch, (long long)NN, first, valid, lo, hi);
        span_g2s<T>(dst, lo, hi, &wbar[stage]);
      }
    } else {
      constexpr int CPI = NN / VXC;  // chunks per entry
#pragma unroll 4
      for (int c = lane; c < IPW * CPI; c += 32) {
        const int e = c / CPI, r = c - e * CPI;
        const bool ok = e < valid;
        const T* src = p.X + (first + (ok ? e : 0)) * p.sx + r * VXC;
        cp_async<VXC * sizeof(T)>(dst + e * C::SLOT + r * VXC, src, ok);
      }
      cp_async_commit();
    }
  };

  // warm L2 with this warp's first groups while the previous kernel drains (hint only)
  if (p.prefetch && use_bar) {
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
      const long long g = gw + s * gstride;
      if (g >= ngroups) break;
      const long long first = g * IPW;
      const int valid = (int)(p.batch - first < IPW ? p.batch - first : IPW);
      if constexpr (K::BULK) {
        if (lane < valid) prefetch_l2(p.X + (first + lane) * p.sx, NN * sizeof(T));
      } else if (lane == 0) {
        uintptr_t lo, hi;
        group_span(p.X, p.batch, (long long)NN, first, valid, lo, hi);
        prefetch_l2_span(lo, hi);
      }
    }
  }
  pdl_enter();  // no global access before the previous kernel on the stream has completed
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(gw + s * gstride, s);

  const int slot = lane / TPI, q = lane % TPI;
  const T* aq = ablk + q * C::QS;
  const int rows = N - q * R;  // valid rows of this block (>= R unless padded)
  int stage = 0;
  unsigned phase = 0;  // parity of the current use of `stage`
  for (long long g = gw; g < ngroups; g += gstride) {
    issue(g + (S - 1) * gstride, (stage + S - 1) % S);
    if (use_bar) {
      mbar_wait(&wbar[stage], phase);
    } else {
      cp_async_wait<S - 1>();
      __syncwarp();
    }
    const long long item = g * IPW + slot;
    T* sbase = wring + stage * K::RING;  // entry 0 of the group (span copies land shifted)
    if (!K::BULK && span) sbase += (reinterpret_cast<uintptr_t>(p.X + g * IPW * NN) & 15) / sizeof(T);
    T* xs = sbase + slot * C::SLOT;
    if constexpr (ystage) {
      // Y(I_q, j) goes into the entry's own smem slot (X is dead once every
      // lane of the entry finished mode 1), then leaves with coalesced stores.
      T t[N][R];
      if (item < p.batch) mode1<T, N, OPX, K::MB>(t, xs, aq);
      __syncwarp();
      if (item < p.batch) {
        const T* yb = p.Y + item * p.sy + q * R;
#pragma unroll
        for (int j0 = 0; j0 < N; j0 += K::JB) {
          T y[K::JB][R];
#pragma unroll
          for (int jj = 0; jj < K::JB; ++jj)
            if (j0 + jj < N) init_y<T, N>(y[jj], yb + (long long)(j0 + jj) * p.ldy, rows, p.beta_mode, p.beta);
          contract_rows_c<T, N, K::JB>(y, t, kc.w, j0);
#pragma unroll
          for (int jj = 0; jj < K::JB; ++jj)
            if (j0 + jj < N) sts_rows<T, N>(xs + (j0 + jj) * N + q * R, y[jj], rows);
        }
      }
      __syncwarp();
      const long long first = g * IPW;
      const int valid = (int)(p.batch - first < IPW ? p.batch - first : IPW);
      if (ybulk) {
        fence_proxy_async();  // staged Y (generic writes) -> the bulk stores (async proxy)
        __syncwarp();
        if constexpr (K::BULK) {
          if (lane < valid) {
            bulk_s2g(p.Y + (first + lane) * p.sy, sbase + lane * C::SLOT, NN * sizeof(T));
            bulk_commit();
          }
        } else {
          const uintptr_t lo = reinterpret_cast<uintptr_t>(p.Y + first * NN);
          span_s2g<T>(lo, lo + (uintptr_t)valid * NN * sizeof(T), wring + stage * K::RING, lane);
        }
      } else {
        copy_out<T, NN, VXC>(p.Y + first * p.sy, p.sy, sbase, C::SLOT, 0, 1, valid, lane, 32);
      }
      if (use_bar) fence_proxy_async();  // generic smem accesses before the TMA refill
    } else if (item < p.batch) {
      T t[N][R];
      mode1<T, N, OPX, K::MB>(t, xs, aq);
      T* yb = p.Y + item * p.sy + q * R;
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += K::JB) {
        T y[K::JB][R];
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj)
          if (j0 + jj < N) init_y<T, N>(y[jj], yb + (long long)(j0 + jj) * p.ldy, rows, p.beta_mode, p.beta);
        contract_rows_c<T, N, K::JB>(y, t, kc.w, j0);
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj)
          if (j0 + jj < N) store_y<T, N>(yb + (long long)(j0 + jj) * p.ldy, y[jj], rows);
      }
    }
    __syncwarp();  // the stage is refilled by the next issue()
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (!use_bar) cp_async_wait<0>();
  if (ystage && use_bar) bulk_wait_all();  // the stages stay valid until the last store has read them
}

// ---------------------------------------------------------------- kron3 ---

// Worst bank multiplicity of one LDS/STS phase in which lane k accesses
// `width` elements at (k / tpi) * stride + (k % tpi) * r (equal addresses broadcast).
__host__ __device__ constexpr int phase_conflicts(int stride, int tpi, int r, int width, int es) {
  const int lanes = 128 / (width * es) < 32 ? 128 / (width * es) : 32;
  int cnt[32] = {};
  int worst = 0;
  const int wb = width * es / 4 > 0 ? width * es / 4 : 1;
  for (int k = 0; k < lanes; ++k) {
    const long long off = (long long)(k / tpi) * stride + (long long)(k % tpi) * r;
    bool dup = false;
    for (int k2 = 0; k2 < k && !dup; ++k2) dup = (long long)(k2 / tpi) * stride + (long long)(k2 % tpi) * r == off;
    if (dup) continue;
    for (int b = 0; b < wb; ++b) {
      const int bank = (int)((off * es / 4 + b) % 32);
      if (++cnt[bank] > worst) worst = cnt[bank];
    }
  }
  return worst;
}

// 3-D plane stride: conflict-free mode-1 column reads (planes of a phase at
// k*stride, TPI lanes broadcasting) AND conflict-free T2 row-block writes
// (lane (s, q) at s*stride + q*R); a multiple of 16 bytes for bulk copies.
template <typename T, int N>
__host__ __device__ constexpr int plane_stride3() {
  using C = SqCfg<T, N>;
  const int es = sizeof(T);
  int align = C::VXC > C::VXR ? C::VXC : C::VXR;
  if ((C::NN * es) % 16 == 0) align = 16 / es;
  const int first = ((C::NN + align - 1) / align) * align;
  int best = first, best_c = 1 << 30;
  for (int s = first; s <= first + 64 * align; s += align) {
    if (s % C::VR) continue;
    const int cr = phase_conflicts(s, C::TPI, 0, C::VXR, es);
    const int cw = C::PLANE_VEC ? phase_conflicts(s, C::TPI, C::R, C::VR, es) : 1;
    const int c = cr > cw ? cr : cw;
    if (c < best_c) {
      best_c = c;
      best = s;
      if (c == 1) break;
    }
  }
  return best;
}

template <typename T, int N, int V = 0>
struct Kron3Fast {
  using C = SqCfg<T, N>;
  static constexpr int PT = N * C::TPI;  // threads per entry (one plane task + one fiber block each)
  // V0 (default): one entry per 64-thread CTA at n = 16 (barriers span 2 warps,
  // 6 CTAs/SM); V1: ~128 threads; V2: ~256; V3: ~128, single-stage ring.
  static constexpr int MAXT = V == 0 ? 64 : (V == 2 ? 256 : 128);
  static constexpr int IT = (MAXT / PT) > 0 ? MAXT / PT : 1;  // entries per tile
  static constexpr int THREADS = IT * PT;
  static constexpr int STAGES = V == 3 ? 1 : 2;
  // resident CTAs/SM targeted (register cap): ~12 warps per SM
  static constexpr int MINB = V == 3 ? 4 : (384 / THREADS > 0 ? 384 / THREADS : 1);
  static constexpr int MB = 4;
  static constexpr bool AREG = sizeof(T) == 4 && C::R * N <= 64;  // A rows live in registers
  static constexpr int JB = sizeof(T) == 4 ? 4 : 4;
  static constexpr int KB = JB;
  static constexpr bool BULK = (C::NN * sizeof(T)) % 16 == 0;  // one cp.async.bulk per plane
  static constexpr int PS = plane_stride3<T, N>();             // plane stride in smem
  static constexpr int ITEM = N * PS;                          // entry stride in smem
  static constexpr int TILE = IT * ITEM;
  static constexpr size_t smem_bytes() {
    return sizeof(T) * ((size_t)C::A_ELEMS + (size_t)STAGES * TILE) + sizeof(unsigned long long) * STAGES;
  }
};

template <typename T, int N, int V, bool YS>
__global__ void __launch_bounds__(Kron3Fast<T, N, V>::THREADS, Kron3Fast<T, N, V>::MINB)
    kron3_sq_kernel(const Kron3Params<T> p, const __grid_constant__ SqConsts3<T, N> kc, const long long ntiles) {
  constexpr bool ystage = YS;
  using K = Kron3Fast<T, N, V>;
  using C = SqCfg<T, N>;
  constexpr int R = C::R, TPI = C::TPI, NN = C::NN, VXC = C::VXC, IT = K::IT, PS = K::PS, S = K::STAGES;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ablk = reinterpret_cast<T*>(smem_raw);
  T* tiles = ablk + C::A_ELEMS;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(tiles + S * K::TILE);

  const int tid = threadIdx.x;
  if constexpr (K::BULK) {
    if (tid == 0)
      for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  stage_a_param<T, N>(ablk, kc.a);
  __syncthreads();

  // start loading tile `tile` (IT entries, N planes each) into `stage`; warp 0 issues
  auto issue = [&](long long tile, int stage) {
    if (tile >= ntiles) {
      if constexpr (!K::BULK) cp_async_commit();
      return;
    }
    T* dst = tiles + stage * K::TILE;
    const long long first = tile * IT;
    const int valid = (int)(p.batch - first < IT ? p.batch - first : IT);
    if constexpr (K::BULK) {
      if (tid < 32) {
        if (tid == 0) mbar_arrive_expect_tx(&bars[stage], (unsigned)(valid * N * NN * sizeof(T)));
        __syncwarp();
        for (int pl = tid; pl < valid * N; pl += 32) {
          const int e = pl / N, n = pl - e * N;
          bulk_g2s(dst + e * K::ITEM + n * PS, p.X + (first + e) * p.sx + (long long)n * NN, NN * sizeof(T),
                   &bars[stage]);
        }
      }
    } else {
      constexpr int CPP = NN / VXC;  // chunks per plane
      constexpr int CPE = N * CPP;   // chunks per entry
      for (int c = tid; c < IT * CPE; c += K::THREADS) {
        const int e = c / CPE, rr = c - e * CPE, n = rr / CPP, r = rr - n * CPP;
        const bool ok = e < valid;
        const T* src = p.X + (first + (ok ? e : 0)) * p.sx + (long long)n * NN + r * VXC;
        cp_async<VXC * sizeof(T)>(dst + e * K::ITEM + n * PS + r * VXC, src, ok);
      }
      cp_async_commit();
    }
  };

  const int task = tid / TPI, q = tid % TPI;  // plane task: entry task/N, plane task%N
  const int te = task / N, tn = task % N;
  const T* aq = ablk + q * C::QS;
  const int fe = te, fj = tn;  // mode-3 fiber block (entry fe, column j = fj, rows I_q)
  const int rows = N - q * R;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(blockIdx.x + (long long)s * gridDim.x, s);
  int stage = 0;
  unsigned phase = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if constexpr (S == 1) {
      issue(tile, 0);
    } else {
      issue(tile + (long long)(S - 1) * gridDim.x, (stage + S - 1) % S);
    }
    if constexpr (K::BULK) {
      mbar_wait(&bars[stage], phase);
    } else {
      cp_async_wait<S - 1>();
      __syncthreads();
    }
    T* buf = tiles + stage * K::TILE;
    // ---- modes 1 and 2 on plane (te, tn); T2(I_q, :, tn) overwrites the X plane
    {
      T* xs = buf + te * K::ITEM + tn * PS;
      T t[N][R];
      if constexpr (K::AREG) {
        T ar[N][R];  // reloaded per tile: live only through mode 1
#pragma unroll
        for (int l = 0; l < N; ++l) lds_n<R, C::VR>(ar[l], aq + l * R);
        mode1_areg<T, N, K::MB>(t, xs, ar);
      } else
        mode1<T, N, 0, K::MB>(t, xs, aq);
      __syncwarp();  // every lane of this warp finished reading its X plane
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += K::JB) {
        T t2[K::JB][R];
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj)
#pragma unroll
          for (int r = 0; r < R; ++r) t2[jj][r] = T(0);
        contract_rows_c<T, N, K::JB>(t2, t, kc.b, j0);
#pragma unroll
        for (int jj = 0; jj < K::JB; ++jj)
          if (j0 + jj < N) sts_rows<T, N>(xs + (j0 + jj) * N + q * R, t2[jj], rows);
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
              lds_n<R, C::VR>(f[n], fb + n * PS);
            else {
#pragma unroll
              for (int r = 0; r < R; ++r) f[n][r] = fb[n * PS + r];
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) f[n][r] = r < rows ? fb[n * PS + r] : T(0);
          }
        }
        T* yb = p.Y + item * p.sy + (long long)fj * p.ldy + q * R;
#pragma unroll
        for (int k0 = 0; k0 < N; k0 += K::KB) {
          T y[K::KB][R];
#pragma unroll
          for (int kk = 0; kk < K::KB; ++kk)
            if (k0 + kk < N) init_y<T, N>(y[kk], yb + (long long)(k0 + kk) * p.ldy2, rows, p.beta_mode, p.beta);
          contract_rows_c<T, N, K::KB>(y, f, kc.c, k0);
          if constexpr (ystage) {
            // Y(I_q, fj, k) overwrites T2(I_q, fj, n = k): exactly the fiber
            // this thread read above, so no other thread is affected.
            T* fw = buf + fe * K::ITEM + fj * N + q * R;
#pragma unroll
            for (int kk = 0; kk < K::KB; ++kk)
              if (k0 + kk < N) sts_rows<T, N>(fw + (k0 + kk) * PS, y[kk], rows);
          } else {
#pragma unroll
            for (int kk = 0; kk < K::KB; ++kk)
              if (k0 + kk < N) store_y<T, N>(yb + (long long)(k0 + kk) * p.ldy2, y[kk], rows);
          }
        }
      }
    }
    if constexpr (ystage) {
      __syncthreads();
      const long long first = tile * IT;
      const int valid = (int)(p.batch - first < IT ? p.batch - first : IT);
      copy_out<T, NN, VXC>(p.Y + first * p.sy, p.sy, buf, K::ITEM, PS, N, valid, tid, K::THREADS);
    }
    if constexpr (K::BULK) fence_proxy_async();  // generic T2 writes before the next TMA refill
    __syncthreads();
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
  if constexpr (!K::BULK) cp_async_wait<0>();
}

}  // namespace kb
