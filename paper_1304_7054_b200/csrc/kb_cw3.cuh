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
#include "kb_oddmaps.h"

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
  static constexpr int MAXT = ES == 4 && V != 2 && V != 7 ? 256 : 128;
  // V7: two independent groups of the V2 tile per CTA sharing a 3-stage ring
  // (1.5 stages per group instead of 2: 8 groups = 32 warps per SM at n = 16
  // fp32, where V2's 2-stage CTAs fit only 6 = 24 warps in shared memory)
  static constexpr int G = V == 7 ? 2 : 1;
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
    if (ES == 4 && V != 2 && V != 3 && V != 7) return MAXT / (N * TPI) > 0 ? MAXT / (N * TPI) : 1;
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
  static constexpr int GT = WP ? (NP + PPW - 1) / PPW * 32 : (NTASK + 31) / 32 * 32;  // threads per group
  static constexpr int THREADS = G * GT;
  static constexpr int NCOL = NP * N;         // mode-1 columns per tile
  static constexpr int CA = WP ? (PPW * N + 31) / 32 : (NCOL + GT - 1) / GT;
  static constexpr int STAGES = V == 1 ? 1 : (V == 7 ? 3 : 2);
  // resident CTAs the register budget targets (~24 warps per SM)
  // threads per SM the register budget targets: ~24 warps, except fp32 n = 10
  // (40 warps at 48 registers, no spills: 35.9 -> 37.3 TFLOP/s; the other
  // sizes gain nothing or spill, profiles/r02_k3_occupancy.txt)
  static constexpr int MINT = ES == 4 && N == 10 ? 1280 : 768;
  static constexpr int MINB_AUTO = MINT / ((IT * N * TPI + 31) / 32 * 32) > 0 ? MINT / ((IT * N * TPI + 31) / 32 * 32) : 1;
  static constexpr int MINB = V == 7 ? 1024 / THREADS
                             : V == 6 ? (768 / THREADS > 0 ? 768 / THREADS : 1)
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
  // mbarriers: one per stage, except V7 -- there a stage alternates between two
  // barriers (tile k uses k % (2 S)), because a parity wait only tells
  // adjacent phases apart and a group can reach tile k before the other
  // group's load of tile k - S (same stage) has landed; with two barriers the
  // previous phase of k's barrier belongs to tile k - 2S, this group's own.
  static constexpr int NBAR = G == 2 ? 2 * STAGES : STAGES;
  // odd n: Y leaves through a per-group shared-memory image of the tile's
  // output span (its own 16-byte misalignment, <= 16/ES - 1 elements, in
  // front) and one bulk store, instead of 2 x N scalar 4/8-byte STGs per task
  // at runtime-strided addresses (p.ystage)
  static constexpr bool YS = !BULK && R == 2;
  static constexpr int YTILE = (IT * N * NN + 16 / ES + 16 / ES - 1) / (16 / ES) * (16 / ES);
  static constexpr size_t YOFF = ((size_t)ES * STAGES * TILE + 8 * NBAR + 8 * STAGES + 15) / 16 * 16;
  static constexpr size_t smem_bytes(bool ystage = false) {
    return ystage ? YOFF + (size_t)ES * G * YTILE : (size_t)ES * STAGES * TILE + 8 * NBAR + 8 * STAGES;
  }
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
  // V7 with a tile counter: the tile each stage holds (-1: none left), written
  // by the issuing lane before its arrive (release) and read after the wait (acquire)
  long long* stage_tile = reinterpret_cast<long long*>(bars + K::NBAR);
  const bool dyn = p.sched != nullptr;
  const bool ys = K::YS && p.ystage;
  // group-local thread index: with G = 2 each group runs the whole tile
  // pipeline on its own tiles, synchronising with a named barrier
  const int grp = K::G == 1 ? 0 : (int)(threadIdx.x / K::GT);
  const int tid = (int)threadIdx.x - grp * K::GT;
  if (threadIdx.x == 0)
    for (int s = 0; s < K::NBAR; ++s) mbar_init(&bars[s], 1);
  mbar_fence_init();
  __syncthreads();
  T* ysm = reinterpret_cast<T*>(smem_raw + K::YOFF) + grp * K::YTILE;  // this group's Y image (ys)
  auto group_sync = [&]() {
    if constexpr (K::G == 1)
      __syncthreads();
    else if (grp == 0)  // compile-time barrier ids: a runtime id reserves all 16 per CTA
      asm volatile("bar.sync 1, %0;" ::"n"(K::GT) : "memory");
    else
      asm volatile("bar.sync 2, %0;" ::"n"(K::GT) : "memory");
  };

  auto issue = [&](long long tile, int stage, int bar = -1) {
    if (tile >= ntiles || tid >= 32) return;
    if (bar < 0) bar = stage;
    T* dst = tiles + stage * K::TILE;
    const long long first = tile * IT;
    const int valid = (int)(p.batch - first < IT ? p.batch - first : IT);
    if constexpr (K::BULK) {
      if (tid == 0) mbar_arrive_expect_tx(&bars[bar], (unsigned)(valid * N * NN * sizeof(T)));
      __syncwarp();
      for (int pl = tid; pl < valid * N; pl += 32) {
        const int e = pl / N, n = pl - e * N;
        bulk_g2s(dst + e * ITEM + n * PS, p.X + (first + e) * p.sx + (long long)n * NN, NN * sizeof(T), &bars[bar]);
      }
    } else if (tid == 0) {
      uintptr_t lo, hi;
      group_span(p.X, p.batch, p.sx, first, valid, lo, hi);
      span_g2s<T>(dst, lo, hi, &bars[bar]);
    }
  };
  // dynamic scheduling (V7 + p.sched): warp 0 of the calling group takes the
  // next tile from the call's counter and loads it into `stage` on barrier
  // `bar`; past the end it publishes -1 with a plain arrive, which releases
  // the consumer so it can stop
  auto claim = [&](int stage, int bar) {
    if (tid >= 32) return;
    long long t = 0;
    if (tid == 0) t = (long long)atomicAdd(p.sched, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t < ntiles) {
      if (tid == 0) stage_tile[stage] = t;
      issue(t, stage, bar);  // lane 0 stores the index before its arrive.expect_tx (release)
    } else if (tid == 0) {
      stage_tile[stage] = -1;
      mbar_arrive(&bars[bar]);
    }
  };

  // per-thread task coordinates (fixed for the kernel)
  const bool task_ok = tid < K::NTASK;
  int q = tid % TPI;
  int j3 = (tid / TPI) % N, e3 = tid / (TPI * N);        // mode-3 fiber column / entry
  const int wid = tid >> 5, lid = tid & 31;
  // mode-2 task: warp-plane (V6) = this warp's planes, else entry-major groups
  const bool m2_ok = K::WP ? (lid < K::PPW * TPI && wid * K::PPW + lid / TPI < NP) : task_ok;
  int P2 = K::WP ? wid * K::PPW + lid / TPI : K::plane_of_group(tid / TPI);
  int q2 = K::WP ? lid % TPI : q;
  // odd n (planes at stride n^2): bank-conflict-aware task maps where the
  // generator found one for this tile shape -- same tasks, other threads
  using OM = OddMap<(int)sizeof(T), N, IT>;
  if constexpr (!K::BULK && R == 2 && OM::M3) {
    if (p.oddmap && task_ok) {
      const unsigned v = OM::m3()[tid];
      e3 = (int)(v >> 7);
      j3 = (int)((v >> 3) & 15);
      q = (int)(v & 7);
    }
  }
  if constexpr (!K::BULK && !K::WP && R == 2 && OM::M2) {
    if (p.oddmap && task_ok) {
      const unsigned v = OM::m2()[tid];
      P2 = (int)(v >> 3);
      q2 = (int)(v & 7);
    }
  }

  pdl_enter();  // no global access before the previous kernel on the stream has completed
  // CTA-local tile counter k: tile(k) = blockIdx.x + k * gridDim.x; group
  // k % G runs it in stage k % S (G = 2: refilled by the group that ran k - 3)
  if constexpr (K::G == 1) {
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
      if (dyn)
        claim(s, s);
      else
        issue(blockIdx.x + (long long)s * gridDim.x, s);
    }
  } else if (grp == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (dyn)
        claim(s, s);
      else
        issue(blockIdx.x + (long long)s * gridDim.x, s, s);
    }
  }
  int stage = 0;
  unsigned phase = 0;
  long long kk = grp;
  for (long long tile = blockIdx.x + kk * gridDim.x; dyn || tile < ntiles; tile += (long long)K::G * gridDim.x) {
    if constexpr (K::G == 1) {
      if (dyn)
        claim(S == 1 ? 0 : (stage + S - 1) % S, S == 1 ? 0 : (stage + S - 1) % S);
      else if constexpr (S == 1)
        issue(tile, 0);
      else
        issue(tile + (long long)(S - 1) * gridDim.x, (stage + S - 1) % S);
    } else {
      stage = (int)(kk % S);
      phase = (unsigned)((kk / (2 * S)) & 1);
    }
    mbar_wait(&bars[K::G == 1 ? stage : (int)(kk % (2 * S))], phase);
    if (dyn) {
      tile = stage_tile[stage];
      if (tile < 0) {  // no tiles left
        // pass the end on: tile kk + S (the other group's next) sits in this
        // same stage, whose stage_tile already reads -1
        if (K::G == 2 && tid == 0) mbar_arrive(&bars[(int)((kk + S) % (2 * S))]);
        break;
      }
    }
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
          const int c = tid + k * K::GT;
          P = c % NP;
          m = c / NP;
          cok[k] = K::CA * K::GT == K::NCOL || c < K::NCOL;
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
      group_sync();

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
    if (ys && tid == 0) bulk_wait_read();  // the previous tile's Y store has read the image
    group_sync();

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
      // ys: the same element's place in the image (tight Y: ldy = N, ldy2 = NN)
      T* yi = ysm + (reinterpret_cast<uintptr_t>(p.Y + first * p.sy) & 15) / sizeof(T) + e3 * N * NN + j3 * N + q * R;
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
      if (ys) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          yi[k * NN] = acc[k][0];
          if (two) yi[k * NN + 1] = acc[k][1];
        }
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          if (K::VRY == 2 || two)
            stg_n<R, K::VRY>(yb + (long long)k * p.ldy2, acc[k]);
          else
            yb[(long long)k * p.ldy2] = acc[k][0];
        }
      }
    }
    fence_proxy_async();  // generic smem writes before the stage's next TMA refill (and the Y bulk store)
    group_sync();
    if (ys && tid < 32) {
      const uintptr_t lo = reinterpret_cast<uintptr_t>(p.Y + first * p.sy);
      span_s2g<T>(lo, lo + (uintptr_t)valid * N * NN * sizeof(T), ysm, tid);
    }
    if constexpr (K::G == 1) {
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    } else {
      if (dyn)
        claim(stage, (int)((kk + S) % (2 * S)));
      else
        issue(blockIdx.x + (kk + S) * (long long)gridDim.x, stage, (int)((kk + S) % (2 * S)));  // the other group's
      kk += K::G;
    }
  }
  if (ys && tid == 0) bulk_wait_all();  // the image stays valid until the last store has read it
  if (dyn) sched_rewind(p.sched);  // the last CTA out rewinds the counters for the next launch on the stream
}

}  // namespace kb
