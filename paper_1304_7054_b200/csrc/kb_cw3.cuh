// kb_cw3.cuh -- "column-wise" square 3-D kernel (kron3, even n <= 16).
//
// Same arithmetic as the reference stage order (kron3.hpp:147-163, each
// gemm_axpy_fixed of detail.hpp:38-59 an ascending FMA chain per element),
// re-mapped so that EVERY contraction takes its shared operand from the
// constant bank (uniform registers) instead of registers or shared memory:
//
//   mode 1 (column owner):  T1(:, m, n) = A_r * X(:, m, n)
//     a thread owns whole X columns (CA of them); FFMA2 pairs two ROWS i, i+1
//     of its column: {T1(i,m,n), T1(i+1,m,n)} += {A(i,l), A(i+1,l)} * X(l,m,n)
//     -- the A pair is a uniform-register pair (SASS `FFMA2 R, R.F32,
//     UR.F32x2`), the X element a per-thread scalar. T1 overwrites the X
//     column in shared memory (same thread, same addresses).
//   mode 2 (row owner, R = 2): T2(I_q, j, n) = sum_m T1(I_q, m, n) B_r(j, m)
//     row pair from smem x uniform scalar B_r(j, m); overwrites T1(I_q, :, n).
//   mode 3 (row owner, R = 2): Y(I_q, j, k) = init + sum_n T2(I_q, j, n) Cw(k, n)
//     with Cw = fl(alpha * C_r); Y leaves registers straight to HBM.
//
// Versus kb_fast.cuh's kron3_sq_kernel this drops the A rows held in
// registers (64 per thread) and most broadcast LDS traffic, so a tile runs
// with ~80 registers per thread and twice the warps per SM. Tiles of IT
// entries land by one cp.async.bulk per plane into a padded plane stride PS
// chosen so that all three phases' shared-memory accesses are conflict-free.
#pragma once

#include "kb_fast.cuh"

#ifndef KB_CW_UNROLL
#define KB_CW_UNROLL 16  // contraction-loop unroll of the column-wise kernels (code size vs loop overhead)
#endif

namespace kb {

constexpr int kCwUnroll = KB_CW_UNROLL;

template <typename T, int N>
struct SqConstsCw3 {
  // column stride: even, so every row pair {i, i+1} (i even) of every column is
  // an 8-byte-aligned constant-bank pair (one UR.F32x2 FFMA2 operand, no UMOVs)
  static constexpr int LD = N % 2 ? N + 1 : N;
  T a[N * LD];   // a[l*LD + i]  = A_r(i, l)          (column l contiguous: row pairs)
  T bt[N * LD];  // bt[m*LD + j] = B_r(j, m)          (all j of one m contiguous)
  T ct[N * LD];  // ct[n*LD + k] = fl(alpha*C_r(k, n))
};

// Bank multiplicity of one shared-memory access phase: `lanes` lanes, lane k at
// word offset off(k) (4-byte words), each touching `words` consecutive words.
// Identical addresses broadcast.
template <typename F>
__host__ __device__ constexpr int phase_banks(F off, int lanes, int words) {
  int cnt[32] = {};
  int worst = 0;
  for (int k = 0; k < lanes; ++k) {
    bool dup = false;
    for (int k2 = 0; k2 < k && !dup; ++k2) dup = off(k2) == off(k);
    if (dup) continue;
    for (int w = 0; w < words; ++w) {
      const int b = (int)((off(k) + w) % 32);
      if (++cnt[b] > worst) worst = cnt[b];
    }
  }
  return worst;
}

template <typename T, int N, int V = 0>
struct Cw3 {
  static constexpr int ES = sizeof(T);
  // rows per mode-2/3 task (odd n: the last task has 1). V3: one row per
  // task -- twice the threads per entry (n = 16: 256), FFMA2 then pairs two
  // output COLUMNS with a uniform-register constant pair, like mode 1
  static constexpr int R = V == 3 ? 1 : 2;
  static constexpr int TPI = (N + R - 1) / R;  // tasks per plane / per fiber column
  static constexpr int NN = N * N;
  // entries per tile: ~256 threads of mode-2/3 tasks (fp32, V0/V1), ~128
  // (fp64; fp32 V2: 4-warp CTAs, so each SM sub-partition interleaves warps
  // of six independent CTAs instead of three)
  static constexpr int MAXT = ES == 4 && V != 2 ? 256 : 128;
  // V2 / fp64: the smallest tile (entries) whose mode-2/3 tasks fill their
  // warps to >= 93 % (n = 10: 3 entries = 150 of 160 threads, not 2 = 100 of
  // 128), at most 384 threads; V0/V1: as many entries as fit MAXT threads
  // V6 "warp-plane": each warp owns PPW whole planes for modes 1 AND 2, so the
  // mode-1 -> mode-2 dependency is intra-warp (__syncwarp); tiles hold the
  // fewest entries whose planes split evenly over warps (n = 10: 6 planes per
  // warp, 3 entries = 5 warps)
  static constexpr bool WP = V == 6;
  static constexpr int PPW = 32 / TPI > 0 ? 32 / TPI : 1;
  __host__ __device__ static constexpr int pick_it() {
    if (V == 6) {
      for (int it = 1; it <= 32; ++it)
        if ((it * N) % PPW == 0 && it * N / PPW <= 12) return it;
      return 1;
    }
    if (V == 4) return 1;  // one entry per CTA: CTA barriers span only that entry's warps
    if (ES == 4 && V != 2 && V != 3) return MAXT / (N * TPI) > 0 ? MAXT / (N * TPI) : 1;
    int best = 1, best_idle = 1 << 30;
    for (int it = 1; it * N * TPI <= 384 || it == 1; ++it) {
      const int t = it * N * TPI, w = (t + 31) / 32 * 32;
      const int idle = (w - t) * 1000 / w;  // per mille
      if (idle * 100 <= 7 * 1000) return it;
      if (idle < best_idle) {
        best_idle = idle;
        best = it;
      }
    }
    return best;
  }
  static constexpr int IT = pick_it();
  static constexpr int NP = IT * N;           // planes per tile
  static constexpr int NTASK = NP * TPI;      // mode-2 and mode-3 tasks per tile
  static constexpr int THREADS = WP ? (NP + PPW - 1) / PPW * 32 : (NTASK + 31) / 32 * 32;
  static constexpr int NCOL = NP * N;         // mode-1 columns per tile
  static constexpr int CA = WP ? (PPW * N + 31) / 32 : (NCOL + THREADS - 1) / THREADS;
  static constexpr int STAGES = V == 1 ? 1 : 2;
  // resident CTAs the register budget targets (~24 warps per SM)
  static constexpr int MINB_AUTO = 768 / ((IT * N * TPI + 31) / 32 * 32) > 0 ? 768 / ((IT * N * TPI + 31) / 32 * 32) : 1;
  static constexpr int MINB = V == 6 ? (768 / THREADS > 0 ? 768 / THREADS : 1)
                             : V == 4 ? MINB_AUTO
                             : V == 3 ? (ES == 4 ? 4 : 3)
                                     : (ES == 4 ? (V == 1 ? 4 : (V == 2 ? MINB_AUTO : 3)) : (V == 1 ? MINB_AUTO : 3));
  static constexpr int VXR = vec_width(N, ES);  // column read width (elements)
  // planes are 16-byte multiples (even n): one cp.async.bulk per plane into a
  // padded plane stride. Otherwise (odd n) the tile's entries are contiguous
  // in HBM and land with ONE bulk copy of the 16-byte-aligned span covering
  // them (<= 12 bytes either side, never crossing a page: an unaligned end is
  // not a page boundary) at plane stride NN, shifted by the span's offset.
  static constexpr bool BULK = (NN * ES) % 16 == 0;
  static constexpr int VR = BULK ? vec_width(R, ES) : 1;       // smem row-pair width
  static constexpr int VRY = N % 2 == 0 ? vec_width(R, ES) : 1;  // HBM Y row-pair width
  static constexpr int SLACK = BULK ? 0 : 32 / ES;              // span rounding (elements)
  // mode-2 plane permutation: 4 plane groups of a warp's 16-lane phases
  // spread across the banks (see plane_of_task)
  static constexpr bool PERM = N % 4 == 0 && TPI * 4 <= 32;

  __host__ __device__ static constexpr int plane_of_group(int g) {
    if (!PERM) return g;
    const int e = g / N, gi = g % N;
    return e * N + gi / 4 + (N / 4) * (gi % 4);
  }

  // worst bank multiplicity over the three phases for plane stride ps (elements)
  __host__ __device__ static constexpr int conflicts(int ps) {
    const int wpe = ES / 4;  // words per element
    const int item = N * ps;
    int worst = 1;
    // mode-1 column reads: lanes 0..(128/(VXR*ES))-1 own columns c = lane
    {
      const int lanes = 128 / (VXR * ES) < 32 ? 128 / (VXR * ES) : 32;
      auto off = [&](int k) {
        const int P = WP ? k % PPW : k % NP, m = WP ? k / PPW : k / NP;
        return ((P / N) * item + (P % N) * ps + m * N) * wpe;
      };
      const int c = phase_banks(off, lanes, VXR * wpe);
      worst = c > worst ? c : worst;
    }
    // mode-2 row-pair reads: task t -> (group g = t / TPI, q = t % TPI), m = 0
    {
      const int lanes = 128 / (VR * ES) < 32 ? 128 / (VR * ES) : 32;
      auto off = [&](int k) {
        const int P = WP ? k / TPI : plane_of_group(k / TPI), q = k % TPI;
        return ((P / N) * item + (P % N) * ps + q * R) * wpe;
      };
      const int c = phase_banks(off, lanes, VR * wpe);
      worst = c > worst ? c : worst;
    }
    return worst;
  }
  __host__ __device__ static constexpr int plane_stride() {
    if (!BULK) return NN;
    const int align = 16 / ES;
    int best = (NN + align - 1) / align * align, best_c = 1 << 30;
    for (int s = best; s <= best + 64 * align; s += align) {
      const int c = conflicts(s);
      if (c < best_c) {
        best_c = c;
        best = s;
        if (c == 1) break;
      }
    }
    return best;
  }
  static constexpr int PS = plane_stride();
  static constexpr int ITEM = N * PS;
  static constexpr int TILE = (IT * ITEM + SLACK + 16 / ES - 1) / (16 / ES) * (16 / ES);
  static constexpr size_t smem_bytes() { return (size_t)ES * STAGES * TILE + 8 * STAGES; }
};

// {acc[i], acc[i+1]} += {a[i], a[i+1]} * s  (a from the constant bank: FFMA2 with a UR pair;
// odd n: the last row is a scalar FFMA)
__device__ __forceinline__ void axpy_pairs_c(float* acc, const float* a, float s, int n) {
#pragma unroll
  for (int i = 0; i + 1 < n; i += 2) {
    const float2 d = ffma2_s(make_float2(a[i], a[i + 1]), s, make_float2(acc[i], acc[i + 1]));
    acc[i] = d.x;
    acc[i + 1] = d.y;
  }
  if (n % 2) acc[n - 1] = __fmaf_rn(a[n - 1], s, acc[n - 1]);
}
__device__ __forceinline__ void axpy_pairs_c(double* acc, const double* a, double s, int n) {
#pragma unroll
  for (int i = 0; i < n; ++i) acc[i] = __fma_rn(a[i], s, acc[i]);
}

template <typename T, int N, int V, bool B0>
__global__ void __launch_bounds__(Cw3<T, N, V>::THREADS, Cw3<T, N, V>::MINB)
    kron3_cw_kernel(const Kron3Params<T> p, const __grid_constant__ SqConstsCw3<T, N> kc, const long long ntiles) {
  using K = Cw3<T, N, V>;
  // B0: beta == 0 known at compile time (Y never read; the beta paths are not in the binary)
  const int beta_mode = B0 ? kBetaZero : p.beta_mode;
  constexpr int R = K::R, TPI = K::TPI, NN = K::NN, IT = K::IT, NP = K::NP, PS = K::PS, S = K::STAGES;
  constexpr int ITEM = K::ITEM;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tiles = reinterpret_cast<T*>(smem_raw);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(tiles + S * K::TILE);
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  mbar_fence_init();
  __syncthreads();

  auto issue = [&](long long tile, int stage) {
    if (tile >= ntiles || tid >= 32) return;
    T* dst = tiles + stage * K::TILE;
    const long long first = tile * IT;
    const int valid = (int)(p.batch - first < IT ? p.batch - first : IT);
    if constexpr (K::BULK) {
      if (tid == 0) mbar_arrive_expect_tx(&bars[stage], (unsigned)(valid * N * NN * sizeof(T)));
      __syncwarp();
      for (int pl = tid; pl < valid * N; pl += 32) {
        const int e = pl / N, n = pl - e * N;
        bulk_g2s(dst + e * ITEM + n * PS, p.X + (first + e) * p.sx + (long long)n * NN, NN * sizeof(T), &bars[stage]);
      }
    } else if (tid == 0) {
      uintptr_t lo, hi;
      group_span(p.X, p.batch, p.sx, first, valid, lo, hi);
      span_g2s<T>(dst, lo, hi, &bars[stage]);
    }
  };

  // per-thread task coordinates (fixed for the kernel)
  const bool task_ok = tid < K::NTASK;
  const int q = tid % TPI;
  const int j3 = (tid / TPI) % N, e3 = tid / (TPI * N);        // mode-3 fiber column / entry
  const int wid = tid >> 5, lid = tid & 31;
  // mode-2 task: warp-plane (V6) = this warp's planes, else entry-major groups
  const bool m2_ok = K::WP ? (lid < K::PPW * TPI && wid * K::PPW + lid / TPI < NP) : task_ok;
  const int P2 = K::WP ? wid * K::PPW + lid / TPI : K::plane_of_group(tid / TPI);
  const int q2 = K::WP ? lid % TPI : q;

#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(blockIdx.x + (long long)s * gridDim.x, s);
  int stage = 0;
  unsigned phase = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if constexpr (S == 1)
      issue(tile, 0);
    else
      issue(tile + (long long)(S - 1) * gridDim.x, (stage + S - 1) % S);
    mbar_wait(&bars[stage], phase);
    const long long first = tile * IT;
    const int valid = (int)(p.batch - first < IT ? p.batch - first : IT);
    T* buf = tiles + stage * K::TILE;
    if constexpr (!K::BULK) buf += (reinterpret_cast<uintptr_t>(p.X + first * p.sx) & 15) / sizeof(T);

    // ---- mode 1: columns c = tid + k*THREADS (plane P = c % NP, column m = c / NP)
    {
      T acc[K::CA][N];
      T* col[K::CA];
      bool cok[K::CA];
#pragma unroll
      for (int k = 0; k < K::CA; ++k) {
        int P, m;
        if constexpr (K::WP) {
          const int c = lid + 32 * k;
          P = wid * K::PPW + c % K::PPW;
          m = c / K::PPW;
          cok[k] = c < K::PPW * N && P < NP;
        } else {
          const int c = tid + k * K::THREADS;
          P = c % NP;
          m = c / NP;
          cok[k] = K::CA * K::THREADS == K::NCOL || c < K::NCOL;
        }
        col[k] = buf + (P / N) * ITEM + (P % N) * PS + m * N;
#pragma unroll
        for (int i = 0; i < N; ++i) acc[k][i] = T(0);
      }
#pragma unroll kCwUnroll
      for (int l0 = 0; l0 < N; l0 += K::VXR) {
        T x[K::CA][K::VXR];
#pragma unroll
        for (int k = 0; k < K::CA; ++k)
          if (cok[k]) lds_vec<K::VXR>(x[k], col[k] + l0);
#pragma unroll
        for (int ll = 0; ll < K::VXR; ++ll)
#pragma unroll
          for (int k = 0; k < K::CA; ++k) axpy_pairs_c(acc[k], kc.a + (l0 + ll) * kc.LD, x[k][ll], N);
      }
#pragma unroll
      for (int k = 0; k < K::CA; ++k)
        if (cok[k])
#pragma unroll
          for (int i = 0; i < N; i += K::VXR) {
            T v[K::VXR];
#pragma unroll
            for (int u = 0; u < K::VXR; ++u) v[u] = acc[k][i + u];
            if constexpr (K::VXR * sizeof(T) == 16 && sizeof(T) == 4)
              *reinterpret_cast<float4*>(col[k] + i) = make_float4(v[0], v[1], v[2], v[3]);
            else if constexpr (K::VXR * sizeof(T) == 16)
              *reinterpret_cast<double2*>(col[k] + i) = make_double2(v[0], v[1]);
            else if constexpr (K::VXR == 2 && sizeof(T) == 4)
              *reinterpret_cast<float2*>(col[k] + i) = make_float2(v[0], v[1]);
            else
#pragma unroll
              for (int u = 0; u < K::VXR; ++u) col[k][i + u] = v[u];
          }
    }
    if constexpr (K::WP)
      __syncwarp();  // this warp's planes are complete in T1
    else
      __syncthreads();

    // ---- mode 2: T2(I_q, j, P2) = sum_m T1(I_q, m, P2) B_r(j, m), in place
    if constexpr (R == 1) {  // one row: FFMA2 pairs columns j, j+1 (uniform B_r pair)
      if (m2_ok) {
        T* pl = buf + (P2 / N) * ITEM + (P2 % N) * PS + q2;
        T acc[N];
#pragma unroll
        for (int j = 0; j < N; ++j) acc[j] = T(0);
#pragma unroll kCwUnroll
        for (int m = 0; m < N; ++m) axpy_pairs_c(acc, kc.bt + m * kc.LD, pl[m * N], N);
#pragma unroll
        for (int j = 0; j < N; ++j) pl[j * N] = acc[j];
      }
    } else if (m2_ok) {
      const bool two2 = N % 2 == 0 || q2 * R + 1 < N;
      T* pl = buf + (P2 / N) * ITEM + (P2 % N) * PS + q2 * R;
      T acc[N][R];
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[j][r] = T(0);
#pragma unroll kCwUnroll
      for (int m = 0; m < N; ++m) {
        T t[R];
        lds_rows<R, K::VR>(t, pl + m * N, two2);
#pragma unroll
        for (int j = 0; j < N; ++j) axpy_rows<R>(acc[j], t, kc.bt[m * kc.LD + j]);
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if constexpr (K::VR == 2 && sizeof(T) == 4)
          *reinterpret_cast<float2*>(pl + j * N) = make_float2(acc[j][0], acc[j][1]);
        else if constexpr (K::VR == 2)
          *reinterpret_cast<double2*>(pl + j * N) = make_double2(acc[j][0], acc[j][1]);
        else {
          pl[j * N] = acc[j][0];
          if (two2) pl[j * N + 1] = acc[j][1];  // odd n: last task owns one row
        }
      }
    }
    __syncthreads();

    // ---- mode 3: Y(I_q, j3, k) = init + sum_n T2(I_q, j3, n) Cw(k, n)
    if constexpr (R == 1) {  // one row: FFMA2 pairs k, k+1 (uniform Cw pair)
      if (task_ok && e3 < valid) {
        const T* fb = buf + e3 * ITEM + j3 * N + q;
        T* yb = p.Y + (first + e3) * p.sy + (long long)j3 * p.ldy + q;
        T acc[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
          acc[k] = beta_mode == kBetaZero ? T(0) : beta_init(beta_mode, p.beta, yb[(long long)k * p.ldy2]);
#pragma unroll kCwUnroll
        for (int n = 0; n < N; ++n) axpy_pairs_c(acc, kc.ct + n * kc.LD, fb[n * PS], N);
#pragma unroll
        for (int k = 0; k < N; ++k) yb[(long long)k * p.ldy2] = acc[k];
      }
    } else if (task_ok && e3 < valid) {
      const bool two = N % 2 == 0 || q * R + 1 < N;
      const T* fb = buf + e3 * ITEM + j3 * N + q * R;
      T* yb = p.Y + (first + e3) * p.sy + (long long)j3 * p.ldy + q * R;
      T acc[N][R];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (beta_mode == kBetaZero) {
          acc[k][0] = T(0);
          acc[k][1] = T(0);
        } else {
          T y0[R];
          if (K::VRY == 2 || two) {
            ldg_n<R, K::VRY>(y0, yb + (long long)k * p.ldy2);
          } else {
            y0[0] = yb[(long long)k * p.ldy2];
            y0[1] = T(0);
          }
          acc[k][0] = beta_init(beta_mode, p.beta, y0[0]);
          acc[k][1] = beta_init(beta_mode, p.beta, y0[1]);
        }
      }
#pragma unroll kCwUnroll
      for (int n = 0; n < N; ++n) {
        T f[R];
        lds_rows<R, K::VR>(f, fb + n * PS, two);
#pragma unroll
        for (int k = 0; k < N; ++k) axpy_rows<R>(acc[k], f, kc.ct[n * kc.LD + k]);
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (K::VRY == 2 || two)
          stg_n<R, K::VRY>(yb + (long long)k * p.ldy2, acc[k]);
        else
          yb[(long long)k * p.ldy2] = acc[k][0];
      }
    }
    fence_proxy_async();  // generic smem writes before the stage's next TMA refill
    __syncthreads();
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
}

}  // namespace kb

namespace kb {

// ----------------------------------------------------------------------------
// n = 16 "warp-plane" variant of the column-wise kernel: one entry per
// 128-thread CTA, and warp w owns planes 4w .. 4w+3 in BOTH mode 1
// (64 columns, two per lane) and mode 2 (8 row pairs per plane), so the
// mode-1 -> mode-2 dependency is intra-warp (__syncwarp) and only mode 3
// (fibers across all 16 planes) needs a CTA barrier. The stage is handed back
// to the TMA without a barrier either: each warp fences its generic smem
// accesses against the async proxy and bumps a per-stage counter; the warp
// that completes the count issues the refill (tile + S*grid).
// Shared-memory banks (fp32): plane stride 264 floats puts the warp's four
// planes 8 banks apart, so a mode-2 half-warp phase (4 planes x 4 row pairs)
// is conflict-free; the mode-1 16-byte column reads (4 planes x 2 columns per
// 8-lane phase) take a 2-way conflict -- 16 instructions per thread per entry.
// fp64: stride 258 doubles, mode-2 phases are one plane's 8 row pairs
// (conflict-free), mode 1 again 2-way.
// EARLY: mode 3 first pulls its whole fiber (16 row pairs) into registers and
// hands the stage back BEFORE its 256 FMAs, so the refill overlaps mode 3.
template <typename T, int S, bool EARLY = false>
struct Cwp3 {
  static constexpr int N = 16, NN = 256, R = 2, THREADS = 128;
  static constexpr int ES = sizeof(T);
  static constexpr int PS = ES == 4 ? 264 : 258;  // 1056 B / 2064 B: 16-B aligned TMA destinations
  static constexpr int MINB = 6;
  static constexpr size_t smem_bytes() { return (size_t)ES * S * N * PS + 16 * S; }
};

__device__ __forceinline__ unsigned atom_add_acq_rel_cta(unsigned* addr, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(addr)), "r"(v) : "memory");
  return old;
}

template <typename T, int S, bool EARLY, bool B0>
__global__ void __launch_bounds__(128, Cwp3<T, S, EARLY>::MINB)
    kron3_cwp_kernel(const Kron3Params<T> p, const __grid_constant__ SqConstsCw3<T, 16> kc, const long long ntiles) {
  using K = Cwp3<T, S, EARLY>;
  const int beta_mode = B0 ? kBetaZero : p.beta_mode;
  constexpr int N = 16, NN = 256, R = 2, PS = K::PS, ITEM = N * PS;
  constexpr int VXR = 16 / sizeof(T);  // column chunk (16 bytes)
  constexpr int VR = 2;                // row pair
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tiles = reinterpret_cast<T*>(smem_raw);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(tiles + S * ITEM);
  unsigned* cnt = reinterpret_cast<unsigned*>(bars + S);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&bars[s], 1);
      cnt[s] = 0;
    }
  }
  mbar_fence_init();
  __syncthreads();

  // this warp loads entry `tile` into `stage`: lanes 0..15 one plane each
  auto issue = [&](long long tile, int stage) {
    if (tile >= ntiles) return;
    if (lane == 0) mbar_arrive_expect_tx(&bars[stage], (unsigned)(N * NN * sizeof(T)));
    __syncwarp();
    if (lane < N)
      bulk_g2s(tiles + stage * ITEM + lane * PS, p.X + tile * p.sx + (long long)lane * NN, NN * sizeof(T), &bars[stage]);
  };
  if (warp == 0)
#pragma unroll
    for (int s = 0; s < S; ++s) issue(blockIdx.x + (long long)s * gridDim.x, s);

  // mode-1 columns: plane 4w + (lane&3), columns lane>>2 and (lane>>2) + 8
  const int p1 = 4 * warp + (lane & 3), m1 = lane >> 2;
  // mode-2 row pair: fp32 plane 4w + ((lane>>2)&3), rows 2*((lane&3) + 4*(lane>>4));
  //                  fp64 plane 4w + (lane>>3), rows 2*(lane&7)
  const int p2 = 4 * warp + (sizeof(T) == 4 ? ((lane >> 2) & 3) : (lane >> 3));
  const int q2 = sizeof(T) == 4 ? ((lane & 3) + 4 * (lane >> 4)) : (lane & 7);
  // mode-3 fiber: column j = tid>>3, rows 2*(tid&7)
  const int j3 = tid >> 3, q3 = tid & 7;

  int stage = 0;
  unsigned phase = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    mbar_wait(&bars[stage], phase);
    T* buf = tiles + stage * ITEM;

    // ---- mode 1 (column owner): T1(:, m, P) = A_r X(:, m, P), in place
    {
      T* c0 = buf + p1 * PS + m1 * N;
      T* c1 = c0 + 8 * N;
      T acc0[N], acc1[N];
#pragma unroll
      for (int i = 0; i < N; ++i) acc0[i] = acc1[i] = T(0);
#pragma unroll
      for (int l0 = 0; l0 < N; l0 += VXR) {
        T x0[VXR], x1[VXR];
        lds_vec<VXR>(x0, c0 + l0);
        lds_vec<VXR>(x1, c1 + l0);
#pragma unroll
        for (int ll = 0; ll < VXR; ++ll) {
          axpy_pairs_c(acc0, kc.a + (l0 + ll) * kc.LD, x0[ll], N);
          axpy_pairs_c(acc1, kc.a + (l0 + ll) * kc.LD, x1[ll], N);
        }
      }
#pragma unroll
      for (int i = 0; i < N; i += VXR) {
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(c0 + i) = make_float4(acc0[i], acc0[i + 1], acc0[i + 2], acc0[i + 3]);
          *reinterpret_cast<float4*>(c1 + i) = make_float4(acc1[i], acc1[i + 1], acc1[i + 2], acc1[i + 3]);
        } else {
          *reinterpret_cast<double2*>(c0 + i) = make_double2(acc0[i], acc0[i + 1]);
          *reinterpret_cast<double2*>(c1 + i) = make_double2(acc1[i], acc1[i + 1]);
        }
      }
    }
    __syncwarp();  // this warp's planes are complete in T1

    // ---- mode 2 (row owner): T2(I_q, j, P) = sum_m T1(I_q, m, P) B_r(j, m), in place
    {
      T* pl = buf + p2 * PS + q2 * R;
      T acc[N][R];
#pragma unroll
      for (int j = 0; j < N; ++j) acc[j][0] = acc[j][1] = T(0);
#pragma unroll
      for (int m = 0; m < N; ++m) {
        T t[R];
        lds_vec<VR>(t, pl + m * N);
#pragma unroll
        for (int j = 0; j < N; ++j) axpy_rows<R>(acc[j], t, kc.bt[m * kc.LD + j]);
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if constexpr (sizeof(T) == 4)
          *reinterpret_cast<float2*>(pl + j * N) = make_float2(acc[j][0], acc[j][1]);
        else
          *reinterpret_cast<double2*>(pl + j * N) = make_double2(acc[j][0], acc[j][1]);
      }
    }
    __syncthreads();  // mode 3 reads fibers across all 16 planes

    // ---- mode 3: Y(I_q, j, k) = init + sum_n T2(I_q, j, n) Cw(k, n)
    {
      const T* fb = buf + j3 * N + q3 * R;
      T* yb = p.Y + tile * p.sy + (long long)j3 * p.ldy + q3 * R;
      T acc[N][R];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (beta_mode == kBetaZero) {
          acc[k][0] = acc[k][1] = T(0);
        } else {
          T y0[R];
          ldg_n<R, VR>(y0, yb + (long long)k * p.ldy2);
          acc[k][0] = beta_init(beta_mode, p.beta, y0[0]);
          acc[k][1] = beta_init(beta_mode, p.beta, y0[1]);
        }
      }
      // hand the stage back: the last warp through issues its refill
      auto release = [&]() {
        fence_proxy_async();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) {
          last = atom_add_acq_rel_cta(&cnt[stage], 1u) == 3u;
          if (last) cnt[stage] = 0;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) issue(tile + (long long)S * gridDim.x, stage);
      };
      if constexpr (EARLY) {
        T f[N][R];
#pragma unroll
        for (int n = 0; n < N; ++n) lds_vec<VR>(f[n], fb + n * PS);
        release();
#pragma unroll
        for (int n = 0; n < N; ++n)
#pragma unroll
          for (int k = 0; k < N; ++k) axpy_rows<R>(acc[k], f[n], kc.ct[n * kc.LD + k]);
      } else {
#pragma unroll
        for (int n = 0; n < N; ++n) {
          T f[R];
          lds_vec<VR>(f, fb + n * PS);
#pragma unroll
          for (int k = 0; k < N; ++k) axpy_rows<R>(acc[k], f, kc.ct[n * kc.LD + k]);
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) stg_n<R, VR>(yb + (long long)k * p.ldy2, acc[k]);
      if constexpr (!EARLY) release();
    }
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
}

}  // namespace kb

namespace kb {

// ----------------------------------------------------------------------------
// Software-pipelined warp-plane kernel (n = 16): each warp runs modes 1+2 of
// entry k+1 BEFORE mode 3 of entry k, so by the time it needs every warp's
// mode-2 planes of entry k (an mbarrier with one arrival per warp) the other
// warps have long arrived -- the CTA-wide wait of kron3_cwp_kernel turns into
// an almost always already-completed phase check. Three stages: entry k
// (mode 3), entry k+1 (modes 1/2), entry k+2 landing by TMA; the last warp to
// finish mode 3 of entry k refills its stage with entry k+3.
template <typename T>
struct Cwpp3 {
  static constexpr int N = 16, NN = 256, R = 2, THREADS = 128, S = 3;
  static constexpr int ES = sizeof(T);
  static constexpr int PS = Cwp3<T, 2>::PS;
  static constexpr int MINB = ES == 4 ? 4 : 2;
  static constexpr size_t smem_bytes() { return (size_t)ES * S * N * PS + 32 * S; }
};

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(128, Cwpp3<T>::MINB)
    kron3_cwpp_kernel(const Kron3Params<T> p, const __grid_constant__ SqConstsCw3<T, 16> kc, const long long ntiles) {
  using K = Cwpp3<T>;
  constexpr int N = 16, NN = 256, R = 2, PS = K::PS, ITEM = N * PS, S = K::S;
  constexpr int VXR = 16 / sizeof(T);
  constexpr int VR = 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tiles = reinterpret_cast<T*>(smem_raw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(tiles + S * ITEM);
  unsigned long long* t2done = full + S;
  unsigned* cnt = reinterpret_cast<unsigned*>(t2done + S);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&t2done[s], 4);
      cnt[s] = 0;
    }
  }
  mbar_fence_init();
  __syncthreads();

  const long long g = gridDim.x;
  auto tile_of = [&](long long k) { return (long long)blockIdx.x + k * g; };
  auto issue = [&](long long k) {  // this warp loads the k-th entry of this CTA
    const long long tile = tile_of(k);
    if (tile >= ntiles) return;
    const int st = (int)(k % S);
    if (lane == 0) mbar_arrive_expect_tx(&full[st], (unsigned)(N * NN * sizeof(T)));
    __syncwarp();
    if (lane < N)
      bulk_g2s(tiles + st * ITEM + lane * PS, p.X + tile * p.sx + (long long)lane * NN, NN * sizeof(T), &full[st]);
  };
  if (warp == 0)
#pragma unroll
    for (int s = 0; s < S; ++s) issue(s);

  const int p1 = 4 * warp + (lane & 3), m1 = lane >> 2;
  const int p2 = 4 * warp + (sizeof(T) == 4 ? ((lane >> 2) & 3) : (lane >> 3));
  const int q2 = sizeof(T) == 4 ? ((lane & 3) + 4 * (lane >> 4)) : (lane & 7);
  const int j3 = tid >> 3, q3 = tid & 7;

  // modes 1 + 2 of this warp's four planes of the k-th entry, then arrive
  auto modes12 = [&](long long k) {
    const int st = (int)(k % S);
    mbar_wait(&full[st], (unsigned)((k / S) & 1));
    T* buf = tiles + st * ITEM;
    {
      T* c0 = buf + p1 * PS + m1 * N;
      T* c1 = c0 + 8 * N;
      T acc0[N], acc1[N];
#pragma unroll
      for (int i = 0; i < N; ++i) acc0[i] = acc1[i] = T(0);
#pragma unroll
      for (int l0 = 0; l0 < N; l0 += VXR) {
        T x0[VXR], x1[VXR];
        lds_vec<VXR>(x0, c0 + l0);
        lds_vec<VXR>(x1, c1 + l0);
#pragma unroll
        for (int ll = 0; ll < VXR; ++ll) {
          axpy_pairs_c(acc0, kc.a + (l0 + ll) * kc.LD, x0[ll], N);
          axpy_pairs_c(acc1, kc.a + (l0 + ll) * kc.LD, x1[ll], N);
        }
      }
#pragma unroll
      for (int i = 0; i < N; i += VXR) {
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(c0 + i) = make_float4(acc0[i], acc0[i + 1], acc0[i + 2], acc0[i + 3]);
          *reinterpret_cast<float4*>(c1 + i) = make_float4(acc1[i], acc1[i + 1], acc1[i + 2], acc1[i + 3]);
        } else {
          *reinterpret_cast<double2*>(c0 + i) = make_double2(acc0[i], acc0[i + 1]);
          *reinterpret_cast<double2*>(c1 + i) = make_double2(acc1[i], acc1[i + 1]);
        }
      }
    }
    __syncwarp();
    {
      T* pl = buf + p2 * PS + q2 * R;
      T acc[N][R];
#pragma unroll
      for (int j = 0; j < N; ++j) acc[j][0] = acc[j][1] = T(0);
#pragma unroll
      for (int m = 0; m < N; ++m) {
        T t[R];
        lds_vec<VR>(t, pl + m * N);
#pragma unroll
        for (int j = 0; j < N; ++j) axpy_rows<R>(acc[j], t, kc.bt[m * kc.LD + j]);
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if constexpr (sizeof(T) == 4)
          *reinterpret_cast<float2*>(pl + j * N) = make_float2(acc[j][0], acc[j][1]);
        else
          *reinterpret_cast<double2*>(pl + j * N) = make_double2(acc[j][0], acc[j][1]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&t2done[st]);
  };

  if (tile_of(0) < ntiles) modes12(0);
  for (long long k = 0; tile_of(k) < ntiles; ++k) {
    if (tile_of(k + 1) < ntiles) modes12(k + 1);
    const int st = (int)(k % S);
    mbar_wait(&t2done[st], (unsigned)((k / S) & 1));
    T* buf = tiles + st * ITEM;
    {
      const T* fb = buf + j3 * N + q3 * R;
      T* yb = p.Y + tile_of(k) * p.sy + (long long)j3 * p.ldy + q3 * R;
      T acc[N][R];
#pragma unroll
      for (int kk = 0; kk < N; ++kk) {
        if (p.beta_mode == kBetaZero) {
          acc[kk][0] = acc[kk][1] = T(0);
        } else {
          T y0[R];
          ldg_n<R, VR>(y0, yb + (long long)kk * p.ldy2);
          acc[kk][0] = beta_init(p.beta_mode, p.beta, y0[0]);
          acc[kk][1] = beta_init(p.beta_mode, p.beta, y0[1]);
        }
      }
#pragma unroll
      for (int n = 0; n < N; ++n) {
        T f[R];
        lds_vec<VR>(f, fb + n * PS);
#pragma unroll
        for (int kk = 0; kk < N; ++kk) axpy_rows<R>(acc[kk], f, kc.ct[n * kc.LD + kk]);
      }
#pragma unroll
      for (int kk = 0; kk < N; ++kk) stg_n<R, VR>(yb + (long long)kk * p.ldy2, acc[kk]);
    }
    fence_proxy_async();
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) {
      last = atom_add_acq_rel_cta(&cnt[st], 1u) == 3u;
      if (last) cnt[st] = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) issue(k + S);
  }
}

}  // namespace kb
