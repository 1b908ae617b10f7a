// kb_cw3_variants.cuh -- n = 16 3-D "warp-plane" column-wise kernels (Cwp3,
// Cwpp3) tried in round 1 (profiles/r01_k3_families.txt: none beat the
// default 128-thread tiles). Development-only: compiled into the library only
// by `make VARIANTS=1` (kb_fast_dispatch.cuh includes this file under
// KB_SWEEP_VARIANTS; KB_K3=4..8 select them); not part of the product build.
#pragma once

#include "../../paper_1304_7054_b200/csrc/kb_cw3.cuh"

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

namespace kb {

// n = 16 warp-plane column-wise kernel (kb_cw3.cuh), S stages.
template <typename T, int S, bool EARLY>
static cudaError_t launch3cwp(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                              cudaStream_t s) {
  constexpr int N = 16;
  using K = Cwp3<T, S, EARLY>;
  if (p.ldx != N || p.ldx2 != (long long)N * N || (p.sx * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T)))
    return cudaErrorNotSupported;
  if (p.ldy % 2 || p.ldy2 % 2 || p.sy % 2 || !aligned<T>(p.Y, 2)) return cudaErrorNotSupported;
  auto kern = p.beta_mode == kBetaZero ? kron3_cwp_kernel<T, S, EARLY, true> : kron3_cwp_kernel<T, S, EARLY, false>;
  const size_t smem = K::smem_bytes();
  const int occ = occupancy_for(kern, K::THREADS, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  const long long ntiles = p.batch;
  const int grid = (int)(ntiles < (long long)sm_count * occ ? ntiles : (long long)sm_count * occ);
  SqConstsCw3<T, N> kc;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      kc.a[i + j * kc.LD] = ha[i + j * N];
      kc.bt[j * kc.LD + i] = hb[i * N + j];
      kc.ct[j * kc.LD + i] = hc[i * N + j];
    }
  kern<<<grid, K::THREADS, smem, s>>>(p, kc, ntiles);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t launch3cwpp(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                               cudaStream_t s) {
  constexpr int N = 16;
  using K = Cwpp3<T>;
  if (p.ldx != N || p.ldx2 != (long long)N * N || (p.sx * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T)))
    return cudaErrorNotSupported;
  if (p.ldy % 2 || p.ldy2 % 2 || p.sy % 2 || !aligned<T>(p.Y, 2)) return cudaErrorNotSupported;
  auto kern = kron3_cwpp_kernel<T>;
  const size_t smem = K::smem_bytes();
  const int occ = occupancy_for(kern, K::THREADS, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  const long long ntiles = p.batch;
  const int grid = (int)(ntiles < (long long)sm_count * occ ? ntiles : (long long)sm_count * occ);
  SqConstsCw3<T, N> kc;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      kc.a[i + j * kc.LD] = ha[i + j * N];
      kc.bt[j * kc.LD + i] = hb[i * N + j];
      kc.ct[j * kc.LD + i] = hc[i * N + j];
    }
  kern<<<grid, K::THREADS, smem, s>>>(p, kc, ntiles);
  return cudaGetLastError();
}

}  // namespace kb
