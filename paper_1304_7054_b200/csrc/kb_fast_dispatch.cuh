// kb_fast_dispatch.cuh -- host-side launch of the square n <= 16 kernels:
// fast-path preconditions, persistent grid sizing (SM count x resident CTAs),
// one-time dynamic-smem attribute per instantiation.
#pragma once

#include <mutex>
#include <cstdlib>
#include <map>
#include <tuple>
#include <utility>

#include "kb_cw2.cuh"
#include "kb_cw3.cuh"
#include "kb_tiny3.cuh"
#include "kb_fast.cuh"
#include "kb_kernels.h"
#include "kb_sizes.h"

namespace kb {

// Resident CTAs per SM for a kernel instantiation; sets its dynamic-smem
// attribute on first use. Keyed by the kernel's address (all instantiations
// of one template share a function-pointer type).
template <typename Kern>
static int occupancy_for(Kern kern, int threads, size_t smem) {
  // a kernel can be launched with more than one dynamic smem size (kb_cw3's
  // Y image is only reserved for tight Y): occupancy is cached per size, and
  // the opt-in limit is only ever RAISED, to the largest size seen, so a
  // launch with a size seen earlier stays valid
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> limit;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), dev, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
  cudaError_t e = cudaSuccess;
  size_t& lim = limit[std::make_pair(reinterpret_cast<const void*>(kern), dev)];
  if (smem > lim) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) lim = smem;
  }
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    occ = 0;
  }
  cache[key] = occ;
  return occ;
}

template <typename T>
static bool aligned(const void* p, int elems) {
  return (reinterpret_cast<uintptr_t>(p) % (sizeof(T) * (size_t)elems)) == 0;
}

// Development-time variant selection (tools/ sweeps, `make VARIANTS=1`): KB_VARIANT2 / KB_VARIANT3.
static int env_variant(const char* name, int dflt = 0) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Launch with programmatic stream serialization (PDL, see pdl_enter in
// kb_device.cuh) for the kernels that call pdl_enter() before touching global
// memory. KB_PDL=0 launches them plainly (A/B sweeps).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int threads, size_t smem, cudaStream_t s,
                              Args&&... args) {
  static const int pdl = env_variant("KB_PDL", 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Stage Y through shared memory (bulk stores when Y is tight, else a
// coalesced copy-out) instead of the direct R-row stores of the row-owner
// kernels. Measured per size on B200 (profiles/r01_sweep_ystage.txt,
// r02_k2_families.txt): it pays for 2-D wherever the row-block stores are
// narrow or scattered (fp32: n = 3, 5-11, 15; fp64: n = 3-8, 10, 11); the
// 3-D row-owner kernel never stages (its column-wise siblings do, kb_cw3.cuh).
// KB_YSTAGE=0 / 1 forces it off / on for sweeps.
template <typename T, int N, int DIMS>
static bool want_ystage(bool legal) {
  static const int force = env_variant("KB_YSTAGE", -1);
  if (!legal) return false;
  if (force >= 0) return force != 0;
  if (DIMS == 3) return false;
  if (sizeof(T) == 4) return (N == 3 || (N >= 5 && N <= 11) || N == 15);
  return (N >= 3 && N <= 8) || N == 10 || N == 11;
}

template <typename T, int N, int OPX, int V>
static cudaError_t launch2v(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s) {
  using C = SqCfg<T, N>;
  using K = Kron2Fast<T, N, V>;
  if (p.ldx != N || p.sx % C::VXC || !aligned<T>(p.X, C::VXC)) return cudaErrorNotSupported;
  if (K::BULK && ((p.sx * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T)))) return cudaErrorNotSupported;
  if (p.ldy % C::VY || p.sy % C::VY || !aligned<T>(p.Y, C::VY)) return cudaErrorNotSupported;
  const bool ys = want_ystage<T, N, 2>(p.ldy == N && p.sy % C::VXC == 0 && aligned<T>(p.Y, C::VXC));
  // (a compile-time beta == 0 specialisation, as the 3-D column-wise kernel
  //  has, made these kernels SLOWER: 2-D n = 16 fp64 5.9 -> 5.0 TB/s)
  auto kern = ys ? kron2_sq_kernel<T, N, OPX, V, true> : kron2_sq_kernel<T, N, OPX, V, false>;
  const int threads = K::WARPS * 32;
  const size_t smem = K::smem_bytes();
  const int occ = occupancy_for(kern, threads, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  const long long ngroups = (p.batch + C::IPW - 1) / C::IPW;
  const long long want = (ngroups + K::WARPS - 1) / K::WARPS;
  const int grid = (int)(want < (long long)sm_count * occ ? want : (long long)sm_count * occ);
  SqConsts2<T, N> kc;
  for (int i = 0; i < N * N; ++i) {
    kc.a[i] = ha[i];
    kc.w[i] = hw[i];
  }
  static const int l2pf = env_variant("KB_L2PF", 1);
  Kron2Params<T> q = p;
  q.prefetch = l2pf;
  return launch_pdl(kern, grid, threads, smem, s, q, kc, ngroups);
}

// Column-wise 2-D kernel (kb_cw2.cuh), op_x = N. ys: Y staged through smem.
template <typename T, int N>
static cudaError_t launch2cw(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s,
                             bool ys) {
  using K = Cw2<T, N>;
  if (p.opx || p.ldx != N) return cudaErrorNotSupported;
  if (K::BULK ? ((p.sx * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T))) : p.sx != (long long)N * N)
    return cudaErrorNotSupported;
  // tiny entries: groups start 16-byte aligned (EPW * entry bytes is a 16-byte multiple), so vector smem
  // accesses stay aligned -- needs X itself 16-byte aligned
  if (K::TINY && ((K::EPW * N * N * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T))))
    return cudaErrorNotSupported;
  if (ys) {
    constexpr int vc = K::BULK || K::TINY ? K::VXC : 1;
    if (p.ldy != N || p.sy % vc || !aligned<T>(p.Y, vc)) ys = false;
  }
  if (!ys && K::VRY == 2 && (p.ldy % 2 || p.sy % 2 || !aligned<T>(p.Y, 2))) return cudaErrorNotSupported;
  auto kern = ys ? kron2_cw_kernel<T, N, true> : kron2_cw_kernel<T, N, false>;
  const int threads = K::WARPS * 32;
  const size_t smem = K::smem_bytes();
  const int occ = occupancy_for(kern, threads, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  const long long ngroups = (p.batch + K::EPW - 1) / K::EPW;
  const long long want = (ngroups + K::WARPS - 1) / K::WARPS;
  const int grid = (int)(want < (long long)sm_count * occ ? want : (long long)sm_count * occ);
  SqConstsCw2<T, N> kc;
  for (int l = 0; l < N; ++l)
    for (int i = 0; i < N; ++i) kc.a[l * kc.LD + i] = ha[l * N + i];
  for (int i = 0; i < N * N; ++i) kc.w[i] = hw[i];
  static const int l2pf = env_variant("KB_L2PF", 1);
  Kron2Params<T> q = p;
  q.prefetch = l2pf;
  return launch_pdl(kern, grid, threads, smem, s, q, kc, ngroups);
}

// 2-D kernel family per size: 0 = row-owner kron2_sq_kernel, 1 = column-wise
// with direct Y stores, 2 = column-wise with Y staged through smem. KB_K2
// overrides the default for sweeps.
template <typename T, int N>
static int k2_family() {
  static const int force = env_variant("KB_K2", -1);
  if (force >= 0) return force;
  // fastest family per size, measured on B200 (round 2, with staged Y leaving
  // by bulk stores: profiles/r02_k2_families.txt; round 1: r01_k2_families.txt)
  if (sizeof(T) == 4) {
    // n = 10 (configs[0]): staged Y + bulk stores on the 2-stage ring, 13.1 -> 12.3 us per
    // 65,536-entry launch (CUDA graph), equal at large batches (tools/gpu/cfg0.sh)
    if (N == 9 || N == 10 || N == 13) return 2;
    return (N <= 2 || N == 4 || N == 6 || N == 12) ? 1 : 0;
  }
  if (N == 3 || N == 5 || N == 10 || N == 12) return 2;
  return (N <= 2 || N == 8 || N == 9 || N == 13) ? 1 : 0;
}

template <typename T, int N, int OPX>
static cudaError_t launch2(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s) {
  if constexpr (OPX == 0) {
    const int fam = k2_family<T, N>();
    if (fam == 1 || fam == 2) {
      const cudaError_t e = launch2cw<T, N>(p, ha, hw, sm_count, s, fam == 2);
      if (e != cudaErrorNotSupported) return e;
    }
  }
#ifdef KB_SWEEP_VARIANTS  // tuning variants: built only with `make VARIANTS=1`
  if constexpr (N == 10 || N == 16) {
    static const int v = env_variant("KB_VARIANT2");
    switch (v) {
      case 1: return launch2v<T, N, OPX, 1>(p, ha, hw, sm_count, s);
      case 2: return launch2v<T, N, OPX, 2>(p, ha, hw, sm_count, s);
      case 3: return launch2v<T, N, OPX, 3>(p, ha, hw, sm_count, s);
      default: break;
    }
  }
#endif
  return launch2v<T, N, OPX, 0>(p, ha, hw, sm_count, s);
}

template <typename T, int N, int V>
static cudaError_t launch3v(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                            cudaStream_t s) {
  using C = SqCfg<T, N>;
  using K = Kron3Fast<T, N, V>;
  if (p.ldx != N || p.ldx2 != (long long)N * N || p.sx % C::VXC || !aligned<T>(p.X, C::VXC))
    return cudaErrorNotSupported;
  if (K::BULK && ((p.sx * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T)))) return cudaErrorNotSupported;
  if (p.ldy % C::VY || p.ldy2 % C::VY || p.sy % C::VY || !aligned<T>(p.Y, C::VY)) return cudaErrorNotSupported;
  const bool ys = want_ystage<T, N, 3>(p.ldy == N && p.ldy2 == (long long)N * N && p.sy % C::VXC == 0 &&
                                    aligned<T>(p.Y, C::VXC));
  auto kern = ys ? kron3_sq_kernel<T, N, V, true> : kron3_sq_kernel<T, N, V, false>;
  const size_t smem = K::smem_bytes();
  const int occ = occupancy_for(kern, K::THREADS, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  const long long ntiles = (p.batch + K::IT - 1) / K::IT;
  const int grid = (int)(ntiles < (long long)sm_count * occ ? ntiles : (long long)sm_count * occ);
  SqConsts3<T, N> kc;
  for (int i = 0; i < N * N; ++i) {
    kc.a[i] = ha[i];
    kc.b[i] = hb[i];
    kc.c[i] = hc[i];
  }
  kern<<<grid, K::THREADS, smem, s>>>(p, kc, ntiles);
  return cudaGetLastError();
}

// Column-wise 3-D kernel (kb_cw3.cuh), even n.
template <typename T, int N, int V>
static cudaError_t launch3cw(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                             cudaStream_t s) {
  using K = Cw3<T, N, V>;
  if (p.ldx != N || p.ldx2 != (long long)N * N) return cudaErrorNotSupported;
  if (K::BULK ? ((p.sx * (long long)sizeof(T)) % 16 || !aligned<T>(p.X, 16 / sizeof(T)))
              : p.sx != (long long)N * N * N)  // odd n: contiguous entries, one span copy per tile
    return cudaErrorNotSupported;
  if (K::VRY == 2 && (p.ldy % 2 || p.ldy2 % 2 || p.sy % 2 || !aligned<T>(p.Y, 2))) return cudaErrorNotSupported;
  auto kern = p.beta_mode == kBetaZero ? kron3_cw_kernel<T, N, V, true> : kron3_cw_kernel<T, N, V, false>;
  // odd n with a tight Y: stage Y through shared memory and store each tile
  // with one bulk copy (KB_YS=0 turns it off for A/B sweeps)
  // (measured: fp32 every odd n +4-23 %; fp64 only n = 7-11 gain, n = 5 / 13 / 15 lose 2-5 %)
  static const int ys_env = env_variant("KB_YS", -1);
  const bool ys_on = ys_env >= 0 ? ys_env != 0 : sizeof(T) == 4 || (N >= 7 && N <= 11);
  Kron3Params<T> q = p;
  q.ystage = K::YS && ys_on && p.ldy == N && p.ldy2 == (long long)N * N && p.sy == (long long)N * N * N;
  static const int om_env = env_variant("KB_OM", 1);  // odd-n task maps (kb_oddmaps.h); 0 = plane-major
  q.oddmap = om_env;
  const size_t smem = K::smem_bytes(q.ystage != 0);
  int occ = occupancy_for(kern, K::THREADS, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  static const int force_ctas = env_variant("KB_CW3_CTAS", 0);  // development sweeps: CTAs per SM
  if (force_ctas > 0 && force_ctas < occ) occ = force_ctas;
  const long long ntiles = (p.batch + K::IT - 1) / K::IT;
  const int grid = (int)(ntiles < (long long)sm_count * occ ? ntiles : (long long)sm_count * occ);
  SqConstsCw3<T, N> kc;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      kc.a[i + j * kc.LD] = ha[i + j * N];
      kc.bt[j * kc.LD + i] = hb[i * N + j];  // bt[m*LD + j] = B_r(j, m)
      kc.ct[j * kc.LD + i] = hc[i * N + j];  // ct[n*LD + k] = Cw(k, n)
    }
  // dynamic tile scheduling (p.sched) pays one L2 atomic per tile on one
  // address: at <= 4 KB of X per tile (> 1.5 G tiles/s at HBM speed; fp32 n = 5
  // 1 KB tiles: 2.2x slower, fp64 n = 8 4 KB one-warp tiles: 2x slower) that
  // atomic rate is the bottleneck, so small tiles keep the static round-robin order
  if ((long long)K::IT * N * N * N * (long long)sizeof(T) <= 4096) q.sched = nullptr;
  return launch_pdl(kern, grid, K::THREADS, smem, s, q, kc, ntiles);
}

#ifdef KB_SWEEP_VARIANTS  // n = 16 warp-plane experiments, kept out of the product tree
}  // namespace kb
#include "../../tools/variants/kb_cw3_variants.cuh"
namespace kb {
#endif

// Tiny-entry 3-D kernel (kb_tiny3.cuh), n <= 4, tight entries.
template <typename T, int N>
static cudaError_t launch3tiny(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                               cudaStream_t s) {
  using K = Tiny3<T, N>;
  constexpr long long E = (long long)N * N * N;
  if (p.ldx != N || p.ldx2 != (long long)N * N || p.sx != E) return cudaErrorNotSupported;
  if (p.ldy != N || p.ldy2 != (long long)N * N || p.sy != E) return cudaErrorNotSupported;
  auto kern = kron3_tiny_kernel<T, N>;
  const int threads = K::WARPS * 32;
  const size_t smem = K::smem_bytes();
  const int occ = occupancy_for(kern, threads, smem);
  if (occ <= 0) return cudaErrorNotSupported;
  const long long ngroups = (p.batch + 31) / 32;
  const long long want = (ngroups + K::WARPS - 1) / K::WARPS;
  const int grid = (int)(want < (long long)sm_count * occ ? want : (long long)sm_count * occ);
  SqConsts3<T, N> kc;
  for (int i = 0; i < N * N; ++i) {
    kc.a[i] = ha[i];
    kc.b[i] = hb[i];
    kc.c[i] = hc[i];
  }
  kern<<<grid, threads, smem, s>>>(p, kc, ngroups);
  return cudaGetLastError();
}

// 3-D kernel family per size: 0 = row-owner (kron3_sq_kernel), 1 = column-wise,
// 2 = column-wise single stage, 3 = column-wise 128-thread tiles (fp32; = 1 for
// fp64), 4 / 5 = n = 16 warp-plane kernel with 2 / 1 stages, 6 = n = 16
// software-pipelined warp-plane kernel (3 stages), 7 / 8 = warp-plane with the
// early stage release (1 / 2 stages); n <= 4 tight entries first try the
// tiny-entry kernel (9 forces it; any other KB_K3 skips it), 10 = column-wise
// with one row per mode-2/3 task (2x threads per entry), 11 = column-wise
// with one entry per CTA, 13 = column-wise warp-plane (each warp owns whole
// planes for modes 1 and 2: no CTA barrier between them). KB_K3 overrides
// the default for sweeps.
template <typename T, int N>
static int k3_family() {
  static const int force = env_variant("KB_K3", -1);
  if (N < 3) return 0;
  if (force >= 0) return N % 2 && force > 3 && force != 11 && force != 13 && force != 14 ? 0 : force;
  // fastest family per size, measured on B200 (profiles/r01_k3_families.txt;
  // odd n run the column-wise kernel with span loads)
  // fp32 n = 16: two 4-warp groups per CTA on a 3-stage ring with dynamic
  // tile scheduling (V7, 32 warps per SM instead of 24): 54.8 -> 60.5 TFLOP/s
  // at 262,144 (profiles/r02_k3_occupancy.txt)
  // odd n with Y staged for bulk stores (p.ystage): fp32 n = 5, 13 256-thread
  // tiles, n = 15 balanced tiles; with dynamic scheduling fp32 n = 14 is
  // fastest on the 256-thread tiles (42.0 vs 37.0 TFLOP/s for V7), fp64 n = 16
  // with one row per task (28.1 vs 26.0), fp64 n = 15 on balanced tiles (+5 %)
  if (sizeof(T) == 4 && N == 16) return 14;
  // n = 6 warp-plane (+4 %); n = 9 on 256-thread tiles once the odd-n task
  // maps remove their bank conflicts (26.4 -> 29.0 TFLOP/s vs warp-plane)
  if (sizeof(T) == 4) return N == 8 ? 0 : N == 6 ? 13 : ((N == 5 || N == 9 || N == 11 || N == 13 || N == 14) ? 1 : 3);
  if (N == 3 || N == 4) return 0;
  if (N == 14) return 14;              // two groups on a 3-stage ring: 22.3 -> 23.5 TFLOP/s
  if (N == 12 || N == 16) return 10;  // one row per task: fp64 n = 12 +15 %
  if (N == 10) return 11;                         // one entry per CTA: +3 %
  if (N == 9 || N == 15) return 3;  // balanced tiles (n = 9 with the task maps: 17.0 -> 17.5)
  return N <= 7 ? 1 : 2;
}

template <typename T, int N>
static cudaError_t launch3(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count,
                           cudaStream_t s) {
  if constexpr (N <= 4) {
    // measured (profiles/r01_k3_families.txt): the tiny-entry kernel wins at
    // fp32 n = 2-4 (n = 2: 1.1 -> 5.6 TB/s) and fp64 n = 2, 3
    static const int force = env_variant("KB_K3", -1);
    constexpr bool tiny_default = N >= 2 && (sizeof(T) == 4 || N <= 3);
    if ((force < 0 && tiny_default) || force == 9) {
      const cudaError_t e = launch3tiny<T, N>(p, ha, hb, hc, sm_count, s);
      if (e != cudaErrorNotSupported) return e;
    }
  }
  if constexpr (N >= 3) {
    const int fam = k3_family<T, N>();
#ifdef KB_SWEEP_VARIANTS  // n = 16 warp-plane experiments (profiles/r01_k3_families.txt): `make VARIANTS=1`
    if constexpr (N == 16) {
      if (fam == 6) {
        const cudaError_t e = launch3cwpp<T>(p, ha, hb, hc, sm_count, s);
        if (e != cudaErrorNotSupported) return e;
      }
      if (fam == 4 || fam == 5 || fam == 7 || fam == 8) {
        const cudaError_t e = fam == 4   ? launch3cwp<T, 2, false>(p, ha, hb, hc, sm_count, s)
                              : fam == 5 ? launch3cwp<T, 1, false>(p, ha, hb, hc, sm_count, s)
                              : fam == 7 ? launch3cwp<T, 1, true>(p, ha, hb, hc, sm_count, s)
                                         : launch3cwp<T, 2, true>(p, ha, hb, hc, sm_count, s);
        if (e != cudaErrorNotSupported) return e;
      }
    }
#endif
    if ((fam >= 1 && fam <= 3) || fam == 10 || fam == 11 || fam == 13 || fam == 14) {
      const cudaError_t e = fam == 1    ? launch3cw<T, N, 0>(p, ha, hb, hc, sm_count, s)
                            : fam == 2  ? launch3cw<T, N, 1>(p, ha, hb, hc, sm_count, s)
                            : fam == 3  ? launch3cw<T, N, 2>(p, ha, hb, hc, sm_count, s)
                            : fam == 10 ? launch3cw<T, N, 3>(p, ha, hb, hc, sm_count, s)
                            : fam == 11 ? launch3cw<T, N, 4>(p, ha, hb, hc, sm_count, s)
                            : fam == 14 ? launch3cw<T, N, 7>(p, ha, hb, hc, sm_count, s)
                                        : launch3cw<T, N, 6>(p, ha, hb, hc, sm_count, s);
      if (e != cudaErrorNotSupported) return e;
    }
  }
#ifdef KB_SWEEP_VARIANTS  // tuning variants: built only with `make VARIANTS=1`
  if constexpr (N == 10 || N == 16) {
    static const int v = env_variant("KB_VARIANT3");
    switch (v) {
      case 1: return launch3v<T, N, 1>(p, ha, hb, hc, sm_count, s);
      case 2: return launch3v<T, N, 2>(p, ha, hb, hc, sm_count, s);
      case 3: return launch3v<T, N, 3>(p, ha, hb, hc, sm_count, s);
      default: break;
    }
  }
#endif
  return launch3v<T, N, 0>(p, ha, hb, hc, sm_count, s);
}

// Per-size entry points (explicitly instantiated in the kb_sz*.cu compile
// units, one group of sizes each, so nvcc builds them in parallel); the
// size switch lives in kb_fast_switch.cu.
template <typename T, int N>
cudaError_t kron2_size(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s) {
  return p.opx ? launch2<T, N, 1>(p, ha, hw, sm_count, s) : launch2<T, N, 0>(p, ha, hw, sm_count, s);
}
template <typename T, int N>
cudaError_t kron3_size(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count, cudaStream_t s) {
  return launch3<T, N>(p, ha, hb, hc, sm_count, s);
}

}  // namespace kb
