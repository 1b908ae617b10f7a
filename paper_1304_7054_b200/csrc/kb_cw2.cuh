// kb_cw2.cuh -- "column-wise" square 2-D kernel (kron2, op_x = N, n <= 16).
//
// The 2-D analogue of kb_cw3.cuh, for kron2.hpp:92-107 (tmp = A_r op(X) with
// alpha 1 beta 0, then Y = init + tmp w(B)^T, w = fl(alpha B_r); each
// gemm_axpy_fixed of detail.hpp:38-59 an ascending FMA chain per element):
//
//   mode 1 (column owner): tmp(:, m) = A_r X(:, m); a lane owns whole columns,
//     FFMA2 pairs two rows with the A row pair from the constant bank (uniform
//     register pair) and the X element as the scalar; tmp overwrites X(:, m).
//   mode 2 (row owner, R = 2): Y(I_q, j) = init + sum_m tmp(I_q, m) w(j, m),
//     row pair from smem x uniform scalar w(j, m).
//
// Every warp is independent (no CTA barrier at all): it owns a ring of STAGES
// shared-memory stages, each holding EPW = 32 / ceil(n/2) entries that land
// by one cp.async.bulk per entry (16-byte entries) or one bulk copy of the
// group's aligned span (odd n), and it runs modes 1 and 2 on its own entries
// with only __syncwarp between them. ~60 registers per thread versus ~180-210
// for the row-owner kron2_sq_kernel, so 2-3x the warps (bytes in flight) per SM.
// Y either leaves registers directly as row pairs or is staged into the
// entry's smem slot and copied out with coalesced 16-byte stores.
#pragma once

#include "kb_cw3.cuh"

#ifndef KB_CW2_STAGES
#define KB_CW2_STAGES 0  // ring stages per warp; 0 = per-size default (sweeps build variant libraries with -D)
#endif

namespace kb {

// 2-D column-wise constants: A_r columns at an even stride, so every row pair
// {i, i+1} (i even) is an 8-byte-aligned constant-bank pair (one UR.F32x2
// FFMA2 operand, no UMOVs at odd n); w as in SqConsts2.
template <typename T, int N>
struct SqConstsCw2 {
  static constexpr int LD = N % 2 ? N + 1 : N;
  T a[N * LD];  // a[l*LD + i] = A_r(i, l)
  T w[N * N];   // w[j*N + m] = fl(alpha B_r(j, m))
};

template <typename T, int N>
struct Cw2 {
  static constexpr int ES = sizeof(T);
  static constexpr int R = 2;
  static constexpr int TPI = (N + 1) / 2;          // mode-2 tasks per entry
  static constexpr int NN = N * N;
  // tiny entries (<= 64 B): KE x more entries per group, contiguous in smem,
  // one span copy per group -- amortises the per-group TMA / mbarrier cost
  static constexpr bool TINY = NN * ES <= 64;
  static constexpr int KE = NN * ES <= 16 ? 8 : (TINY ? 2 : 1);
  static constexpr int EPW = KE * (32 / TPI);      // entries per warp group
  static constexpr int NCOL = EPW * N;             // mode-1 columns per group
  static constexpr int CA = (NCOL + 31) / 32;      // columns per lane
  static constexpr int KT = (EPW * TPI + 31) / 32;  // mode-2 tasks per lane
  static constexpr int WARPS = 8;
  // ring depth: 2 stages for fp32 n = 10 and odd n >= 9, fp64 n = 10, 11, 13 (fewer
  // smem bytes per CTA -> more resident warps: fp32 n = 13 27.7 -> 29.3,
  // fp64 n = 13 14.8 -> 17.0, n = 10 13.6 -> 14.9 TFLOP/s), else 3
  // (profiles/r02_k2_families.txt); KB_CW2_STAGES overrides for sweeps
  static constexpr int STAGES = KB_CW2_STAGES > 0 ? KB_CW2_STAGES
                                : (ES == 4 && ((N % 2 && N >= 9) || N == 10)) || (ES == 8 && (N == 10 || N == 11 || N == 13)) ? 2
                                                                                                              : 3;
  static constexpr int VXR = vec_width(N, ES);     // column read width
  static constexpr bool BULK = (NN * ES) % 16 == 0 && !TINY;  // one bulk copy per entry (else per group span)
  static constexpr int VR = BULK || (TINY && (NN * ES) % 16 == 0) ? vec_width(R, ES) : 1;
  static constexpr int VRY = N % 2 == 0 ? vec_width(R, ES) : 1;
  static constexpr int VXC = vec_width(NN, ES);    // copy-out chunk
  // slot stride: mode-1 column reads (lane c -> entry c % EPW, column c / EPW)
  // and mode-2 row-pair reads (lane t -> entry t / TPI, rows 2 (t % TPI))
  __host__ __device__ static constexpr int conflicts(int slot) {
    const int wpe = ES / 4;
    int worst = 1;
    {
      const int lanes = 128 / (VXR * ES) < 32 ? 128 / (VXR * ES) : 32;
      auto off = [&](int k) { return ((k % EPW) * slot + (k / EPW) * N) * wpe; };
      const int c = phase_banks(off, lanes, VXR * wpe);
      worst = c > worst ? c : worst;
    }
    {
      const int lanes = 128 / (VR * ES) < 32 ? 128 / (VR * ES) : 32;
      auto off = [&](int k) { return ((k / TPI) * slot + (k % TPI) * R) * wpe; };
      const int c = phase_banks(off, lanes, VR * wpe);
      worst = c > worst ? c : worst;
    }
    return worst;
  }
  __host__ __device__ static constexpr int slot_stride() {
    if (!BULK) return NN;  // odd n / tiny: entries contiguous as in HBM
    const int align = 16 / ES;
    int best = NN, best_c = 1 << 30;
    for (int s = NN; s <= NN + 32 * align; s += align) {
      const int c = conflicts(s);
      if (c < best_c) {
        best_c = c;
        best = s;
        if (c == 1) break;
      }
    }
    return best;
  }
  static constexpr int SLOT = slot_stride();
  static constexpr int SLACK = BULK ? 0 : 32 / ES;
  static constexpr int RING = (EPW * SLOT + SLACK + 16 / ES - 1) / (16 / ES) * (16 / ES);  // per stage
  static constexpr size_t smem_bytes() { return (size_t)ES * WARPS * STAGES * RING + 8 * WARPS * STAGES; }
};

template <typename T, int N, bool YS>
__global__ void __launch_bounds__(Cw2<T, N>::WARPS * 32)
    kron2_cw_kernel(const Kron2Params<T> p, const __grid_constant__ SqConstsCw2<T, N> kc, const long long ngroups) {
  constexpr bool ystage = YS;  // compile-time: the other store path is not even in the binary
  using K = Cw2<T, N>;
  constexpr int R = K::R, TPI = K::TPI, EPW = K::EPW, NN = K::NN, S = K::STAGES, SLOT = K::SLOT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + K::WARPS * S * K::RING);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wring = ring + warp * S * K::RING;
  unsigned long long* wbar = bars + warp * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&wbar[s], 1);
  mbar_fence_init();
  __syncwarp();

  const long long gw = (long long)blockIdx.x * K::WARPS + warp;
  const long long gstride = (long long)gridDim.x * K::WARPS;

  // ystage with a tight Y whose 16-byte phase matches the stage image: Y
  // leaves by bulk stores (odd n: one span per group; padded slots: one per
  // entry) instead of the copy-out loop; a stage is refilled only after the
  // stores that read it (this lane's bulk groups) have read it
  const bool ybulk = ystage && p.ldy == N &&
                     (K::BULK ? (p.sy * (long long)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.Y) & 15) == 0
                              : p.sy == NN && ((reinterpret_cast<uintptr_t>(p.X) ^ reinterpret_cast<uintptr_t>(p.Y)) & 15) == 0);
  auto issue = [&](long long g, int stage) {
    if (g >= ngroups) return;
    if (ystage) bulk_wait_read();
    T* dst = wring + stage * K::RING;
    const long long first = g * EPW;
    const int valid = (int)(p.batch - first < EPW ? p.batch - first : EPW);
    if constexpr (K::BULK) {
      if (lane == 0) mbar_arrive_expect_tx(&wbar[stage], (unsigned)(valid * NN * sizeof(T)));
      __syncwarp();
      if (lane < valid) bulk_g2s(dst + lane * SLOT, p.X + (first + lane) * p.sx, NN * sizeof(T), &wbar[stage]);
    } else if (lane == 0) {
      uintptr_t lo, hi;
      group_span(p.X, p.batch, (long long)NN, first, valid, lo, hi);
      span_g2s<T>(dst, lo, hi, &wbar[stage]);
    }
  };
  // warm L2 with this warp's first groups while the previous kernel drains (hint only)
  if (p.prefetch) {
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
      const long long g = gw + s * gstride;
      if (g >= ngroups) break;
      const long long first = g * EPW;
      const int valid = (int)(p.batch - first < EPW ? p.batch - first : EPW);
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

  int stage = 0;
  unsigned phase = 0;
  for (long long g = gw; g < ngroups; g += gstride) {
    issue(g + (S - 1) * gstride, (stage + S - 1) % S);
    mbar_wait(&wbar[stage], phase);
    const long long first = g * EPW;
    const int valid = (int)(p.batch - first < EPW ? p.batch - first : EPW);
    T* base = wring + stage * K::RING;
    if constexpr (!K::BULK) base += (reinterpret_cast<uintptr_t>(p.X + first * NN) & 15) / sizeof(T);

    // ---- mode 1: columns c = lane + 32k -- padded slots: entry c % EPW, column
    //      c / EPW (the bank model picked SLOT for this); contiguous entries
    //      (odd n, tiny): column c of the group, i.e. consecutive lanes read
    //      consecutive columns
    {
      T acc[K::CA][N];
      T* col[K::CA];
#pragma unroll
      for (int k = 0; k < K::CA; ++k) {
        const int c = lane + 32 * k;
        col[k] = K::BULK ? base + (c % EPW) * SLOT + (c / EPW) * N : base + c * N;
#pragma unroll
        for (int i = 0; i < N; ++i) acc[k][i] = T(0);
      }
#pragma unroll
      for (int l0 = 0; l0 < N; l0 += K::VXR) {
        T x[K::CA][K::VXR];
#pragma unroll
        for (int k = 0; k < K::CA; ++k)
          if (K::CA * 32 == K::NCOL || lane + 32 * k < K::NCOL) lds_vec<K::VXR>(x[k], col[k] + l0);
#pragma unroll
        for (int ll = 0; ll < K::VXR; ++ll)
#pragma unroll
          for (int k = 0; k < K::CA; ++k) axpy_pairs_c(acc[k], kc.a + (l0 + ll) * kc.LD, x[k][ll], N);
      }
#pragma unroll
      for (int k = 0; k < K::CA; ++k)
        if (K::CA * 32 == K::NCOL || lane + 32 * k < K::NCOL)
#pragma unroll
          for (int i = 0; i < N; i += K::VXR) {
            if constexpr (K::VXR * sizeof(T) == 16 && sizeof(T) == 4)
              *reinterpret_cast<float4*>(col[k] + i) = make_float4(acc[k][i], acc[k][i + 1], acc[k][i + 2], acc[k][i + 3]);
            else if constexpr (K::VXR * sizeof(T) == 16)
              *reinterpret_cast<double2*>(col[k] + i) = make_double2(acc[k][i], acc[k][i + 1]);
            else if constexpr (K::VXR == 2 && sizeof(T) == 4)
              *reinterpret_cast<float2*>(col[k] + i) = make_float2(acc[k][i], acc[k][i + 1]);
            else
#pragma unroll
              for (int u = 0; u < K::VXR; ++u) col[k][i + u] = acc[k][i + u];
          }
    }
    __syncwarp();

    // ---- mode 2: Y(I_q, j) = init + sum_m tmp(I_q, m) w(j, m); task t = lane + 32 kt
    //      -> entry t / TPI, rows 2 (t % TPI) .. +1 (odd n: the last task owns one)
#pragma unroll
    for (int kt = 0; kt < K::KT; ++kt) {
    const int t = lane + 32 * kt;
    const int e2 = t / TPI, q = t % TPI;
    const bool two = N % 2 == 0 || q * R + 1 < N;
    if (e2 < EPW && e2 < valid) {
      T* tr = base + e2 * SLOT + q * R;
      T* yb = p.Y + (first + e2) * p.sy + q * R;
      T acc[N][R];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (p.beta_mode == kBetaZero) {
          acc[j][0] = acc[j][1] = T(0);
        } else {
          T y0[R];
          if (K::VRY == 2 || two) {
            ldg_n<R, K::VRY>(y0, yb + (long long)j * p.ldy);
          } else {
            y0[0] = yb[(long long)j * p.ldy];
            y0[1] = T(0);
          }
          acc[j][0] = beta_init(p.beta_mode, p.beta, y0[0]);
          acc[j][1] = beta_init(p.beta_mode, p.beta, y0[1]);
        }
      }
#pragma unroll
      for (int m = 0; m < N; ++m) {
        T t[R];
        lds_rows<R, K::VR>(t, tr + m * N, two);
#pragma unroll
        for (int j = 0; j < N; ++j) axpy_rows<R>(acc[j], t, kc.w[j * N + m]);
      }
      if constexpr (ystage) {  // Y(I_q, j) over tmp(I_q, m = j): the rows this lane read
#pragma unroll
        for (int j = 0; j < N; ++j) {
          if constexpr (K::VR == 2 && sizeof(T) == 4)
            *reinterpret_cast<float2*>(tr + j * N) = make_float2(acc[j][0], acc[j][1]);
          else if constexpr (K::VR == 2)
            *reinterpret_cast<double2*>(tr + j * N) = make_double2(acc[j][0], acc[j][1]);
          else {
            tr[j * N] = acc[j][0];
            if (two) tr[j * N + 1] = acc[j][1];
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          if (K::VRY == 2 || two)
            stg_n<R, K::VRY>(yb + (long long)j * p.ldy, acc[j]);
          else
            yb[(long long)j * p.ldy] = acc[j][0];
        }
      }
    }
    }
    if constexpr (ystage) {
      if (ybulk) {
        fence_proxy_async();  // staged Y (generic writes) -> the bulk stores (async proxy)
        __syncwarp();
        if constexpr (K::BULK) {
          if (lane < valid) {
            bulk_s2g(p.Y + (first + lane) * p.sy, base + lane * SLOT, NN * sizeof(T));
            bulk_commit();
          }
        } else {
          const uintptr_t lo = reinterpret_cast<uintptr_t>(p.Y + first * NN);
          span_s2g<T>(lo, lo + (uintptr_t)valid * NN * sizeof(T), wring + stage * K::RING, lane);
        }
      } else {
        __syncwarp();
        copy_out<T, NN, (K::BULK || K::TINY ? K::VXC : 1)>(p.Y + first * p.sy, p.sy, base, SLOT, 0, 1, valid, lane, 32);
      }
    }
    fence_proxy_async();  // generic smem writes (tmp, staged Y) before the stage's TMA refill
    __syncwarp();
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (ystage) bulk_wait_all();  // the stages stay valid until the last store has read them
}

}  // namespace kb
