// kb_device.cuh -- device-side building blocks shared by the sm_100a kron kernels.
//
// Arithmetic contract (reference detail.hpp:38-117):
// every accumulation step is ONE IEEE fma in round-to-nearest, performed in
// ascending contraction index per output element, starting from the beta
// initialisation (0 / Y / fl(Y*beta)); the right factor is pre-scaled as
// w = fl(alpha * R). `fma.rn.f32x2` (SASS FFMA2) packs two DIFFERENT output
// elements per instruction -- never two terms of one sum -- so it preserves
// the per-element order. Nothing here relies on nvcc's --fmad contraction.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace kb {

// ------------------------------------------------------------ arithmetic --

__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// {d.x, d.y} = {fma(a.x, s, c.x), fma(a.y, s, c.y)} as one FFMA2 with a
// broadcast scalar operand.
__device__ __forceinline__ float2 ffma2_s(float2 a, float s, float2 c) {
  unsigned long long ra, rc, rd, rs;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %1};" : "=l"(rs) : "f"(s));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rs), "l"(rc));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}

// acc[r] = fma(a[r], s, acc[r]) for r < R; pairs go through FFMA2 for float.
template <int R>
__device__ __forceinline__ void axpy_rows(float (&acc)[R], const float (&a)[R], float s) {
#pragma unroll
  for (int r = 0; r + 1 < R; r += 2) {
    float2 d = ffma2_s(make_float2(a[r], a[r + 1]), s, make_float2(acc[r], acc[r + 1]));
    acc[r] = d.x;
    acc[r + 1] = d.y;
  }
  if constexpr (R % 2) acc[R - 1] = __fmaf_rn(a[R - 1], s, acc[R - 1]);
}
template <int R>
__device__ __forceinline__ void axpy_rows(double (&acc)[R], const double (&a)[R], double s) {
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = __fma_rn(a[r], s, acc[r]);
}

// -------------------------------------------------------- shared memory --

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gmem_src, bool valid) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int src_bytes = valid ? BYTES : 0;  // 0 => zero-fill, source not read
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem_src), "r"(src_bytes)
                 : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(dst), "l"(gmem_src), "n"(BYTES),
                 "r"(src_bytes)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------- mbarrier + bulk copy --
// 1-D TMA (cp.async.bulk): one instruction moves a whole entry / plane from
// HBM into shared memory and signals an mbarrier with the byte count.

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order this thread's generic-proxy smem accesses before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// One thread lands global bytes [lo, hi) (element-aligned) in shared memory so
// that global address a goes to dst + (a - (lo & ~15)); dst is 16-byte aligned.
// Only [lo, hi) is read: the 16-byte-aligned interior by one bulk copy that
// completes on `bar` (the arrive carries its byte count), the unaligned head
// and tail (< 16 bytes each: only at the ends of a batch) by plain loads
// stored BEFORE the arrive, whose release / the waiters' acquire publishes them
// together with the bulk bytes.
template <typename T>
__device__ __forceinline__ void span_g2s(void* dst, uintptr_t lo, uintptr_t hi, unsigned long long* bar) {
  const uintptr_t base = lo & ~uintptr_t(15);
  const uintptr_t i0 = (lo + 15) & ~uintptr_t(15), i1 = hi & ~uintptr_t(15);
  char* d = static_cast<char*>(dst);
  if (i0 != lo || i1 != hi) {
    const uintptr_t h1 = i0 < hi ? i0 : hi;
    for (uintptr_t a = lo; a < h1; a += sizeof(T))
      *reinterpret_cast<T*>(d + (a - base)) = *reinterpret_cast<const T*>(a);
    for (uintptr_t a = i1 > h1 ? i1 : h1; a < hi; a += sizeof(T))
      *reinterpret_cast<T*>(d + (a - base)) = *reinterpret_cast<const T*>(a);
    fence_proxy_async();  // these generic writes before later TMA refills of the stage
  }
  const unsigned bulk = i1 > i0 ? static_cast<unsigned>(i1 - i0) : 0u;
  mbar_arrive_expect_tx(bar, bulk);
  if (bulk) bulk_g2s(d + (i0 - base), reinterpret_cast<const void*>(i0), bulk, bar);
}

// Span of a group of contiguous entries [first, first + count) (stride sx) of a
// batch of `batch` entries at X: rounded out to 16 bytes for the bulk copy,
// clamped to the batch's own bytes [X, X + batch*sx) so that nothing before the
// first or after the last entry is read.
template <typename T>
__device__ __forceinline__ void group_span(const T* X, long long batch, long long sx, long long first, long long count,
                                           uintptr_t& lo, uintptr_t& hi) {
  const uintptr_t xb = reinterpret_cast<uintptr_t>(X), xe = reinterpret_cast<uintptr_t>(X + batch * sx);
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(X + first * sx) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(X + (first + count) * sx) + uintptr_t(15)) & ~uintptr_t(15);
  lo = a0 > xb ? a0 : xb;
  hi = a1 < xe ? a1 : xe;
}

// shared -> global bulk copy (TMA engine), tracked by this thread's bulk groups
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// this thread's bulk stores have finished READING shared memory (the source may be rewritten)
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// The store-side twin of span_g2s, run by one warp: global bytes [lo, hi)
// (element-aligned) from their shared-memory image at src (src <-> lo & ~15,
// 16-byte aligned; the generic writes that made it are fenced to the async
// proxy and barrier-ordered before this). Lane 0 stores the 16-byte-aligned
// interior with one bulk copy (own bulk group: wait with bulk_wait_read before
// src is rewritten); lanes 1-15 store the unaligned head / tail elements, so
// nothing outside [lo, hi) -- a neighbouring tile's output -- is written.
template <typename T>
__device__ __forceinline__ void span_s2g(uintptr_t lo, uintptr_t hi, const void* src, int lane) {
  const uintptr_t base = lo & ~uintptr_t(15);
  const uintptr_t i0 = (lo + 15) & ~uintptr_t(15), i1 = hi & ~uintptr_t(15);
  const char* s = static_cast<const char*>(src);
  if (lane == 0) {
    if (i1 > i0) {
      bulk_s2g(reinterpret_cast<void*>(i0), s + (i0 - base), static_cast<unsigned>(i1 - i0));
      bulk_commit();
    }
  } else if (lane < 16) {
    constexpr int E = 16 / sizeof(T);  // elements per 16 bytes
    const uintptr_t h1 = i0 < hi ? i0 : hi;
    const int k = (lane - 1) % E;
    const uintptr_t a = lane <= E ? lo + k * sizeof(T) : (i1 > h1 ? i1 : h1) + k * sizeof(T);
    if (lane <= 2 * E && (lane <= E ? a < h1 : a < hi))
      *reinterpret_cast<T*>(a) = *reinterpret_cast<const T*>(s + (a - base));
  }
}

// L2 prefetch of global bytes [p, p + bytes) (16-byte aligned, multiple of
// 16) by the TMA engine. A hint only: L2 is the GPU's point of coherence, so
// warming it with a buffer the previous kernel on the stream may still be
// writing is safe -- the kernels issue it for their first tiles BEFORE
// pdl_enter(), overlapping the HBM latency of their first loads with the
// previous kernel's tail.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// The aligned interior of the span group_span() returns for a group of
// contiguous entries (head / tail bytes are loaded directly anyway).
__device__ __forceinline__ void prefetch_l2_span(uintptr_t lo, uintptr_t hi) {
  const uintptr_t i0 = (lo + 15) & ~uintptr_t(15), i1 = hi & ~uintptr_t(15);
  if (i1 > i0) prefetch_l2(reinterpret_cast<const void*>(i0), static_cast<unsigned>(i1 - i0));
}

// Programmatic dependent launch: kernels launched with the programmatic
// stream-serialization attribute (kb_fast_dispatch.cuh launch_pdl) may be
// scheduled while the previous kernel on the stream drains its last CTAs, so
// their launch latency and prologue (barrier init, constant staging) overlap
// that tail. griddepcontrol.wait blocks until the previous grid has completed
// and its memory is visible -- every global access of the kernel comes after
// it, so stream order is kept exactly; launch_dependents lets the NEXT kernel
// start its own prologue. Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Dynamic scheduling (Kron3Params::sched): the last CTA to finish rewinds the
// call's counter pair {next tile, CTAs done} for the next launch on the stream.
__device__ __forceinline__ void sched_rewind(unsigned long long* ctr) {
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&ctr[1], 1ull) == gridDim.x - 1) {
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

// Vector load of W consecutive elements (W*sizeof(T) bytes, naturally aligned).
template <int W, typename T>
__device__ __forceinline__ void lds_vec(T* dst, const T* src) {
  if constexpr (W * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      float4 v = *reinterpret_cast<const float4*>(src);
      dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
    } else {
      double2 v = *reinterpret_cast<const double2*>(src);
      dst[0] = v.x; dst[1] = v.y;
    }
  } else if constexpr (W * sizeof(T) == 8 && sizeof(T) == 4) {
    float2 v = *reinterpret_cast<const float2*>(src);
    dst[0] = v.x; dst[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) dst[i] = src[i];
  }
}

// Load n consecutive elements with the widest aligned vector width VW.
template <int n, int VW, typename T>
__device__ __forceinline__ void lds_n(T* dst, const T* src) {
  static_assert(n % VW == 0, "vector width must divide the length");
#pragma unroll
  for (int i = 0; i < n; i += VW) lds_vec<VW>(dst + i, src + i);
}

// R consecutive rows of a row block; odd n: the last block of a column has a
// single row (two == false) and must not touch the next column's first element
// (another thread's, which may be written concurrently in place).
template <int R, int VW, typename T>
__device__ __forceinline__ void lds_rows(T* dst, const T* src, bool two) {
  if constexpr (R == 2 && VW == 1) {
    dst[0] = src[0];
    dst[1] = two ? src[1] : T(0);
  } else {
    lds_n<R, VW>(dst, src);
  }
}

// Store n consecutive elements to global memory with vector width VW.
template <int n, int VW, typename T>
__device__ __forceinline__ void stg_n(T* dst, const T* src) {
#pragma unroll
  for (int i = 0; i < n; i += VW) {
    if constexpr (VW * sizeof(T) == 16) {
      if constexpr (sizeof(T) == 4)
        *reinterpret_cast<float4*>(dst + i) = make_float4(src[i], src[i + 1], src[i + 2], src[i + 3]);
      else
        *reinterpret_cast<double2*>(dst + i) = make_double2(src[i], src[i + 1]);
    } else if constexpr (VW * sizeof(T) == 8 && sizeof(T) == 4) {
      *reinterpret_cast<float2*>(dst + i) = make_float2(src[i], src[i + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < VW; ++k) dst[i + k] = src[i + k];
    }
  }
}

template <int n, int VW, typename T>
__device__ __forceinline__ void ldg_n(T* dst, const T* src) {
#pragma unroll
  for (int i = 0; i < n; i += VW) {
    if constexpr (VW * sizeof(T) == 16) {
      if constexpr (sizeof(T) == 4) {
        float4 v = *reinterpret_cast<const float4*>(src + i);
        dst[i] = v.x; dst[i + 1] = v.y; dst[i + 2] = v.z; dst[i + 3] = v.w;
      } else {
        double2 v = *reinterpret_cast<const double2*>(src + i);
        dst[i] = v.x; dst[i + 1] = v.y;
      }
    } else if constexpr (VW * sizeof(T) == 8 && sizeof(T) == 4) {
      float2 v = *reinterpret_cast<const float2*>(src + i);
      dst[i] = v.x; dst[i + 1] = v.y;
    } else {
#pragma unroll
      for (int k = 0; k < VW; ++k) dst[i + k] = src[i + k];
    }
  }
}

// --------------------------------------------------------- kernel params --

// beta initialisation classes of gemm_axpy (detail.hpp:45-51)
enum BetaMode : int { kBetaZero = 0, kBetaOne = 1, kBetaScale = 2 };

template <typename T>
__device__ __forceinline__ T beta_init(int mode, T beta, T prior) {
  return mode == kBetaZero ? T(0) : (mode == kBetaOne ? prior : mul_rn(prior, beta));
}

template <typename T>
struct Kron2Params {
  const T* A;
  const T* B;
  const T* X;
  T* Y;
  long long lda, ldb, ldx, sx, ldy, sy;
  long long m_a, n_a, m_b, n_b;
  long long batch;   // entries this launch processes (already offset pointers)
  int opa, opb, opx; // 1 = transposed
  int beta_mode;
  T alpha, beta;
  int prefetch = 1;  // warm L2 with the first groups before the PDL wait (launcher: KB_L2PF=0 turns it off)
};

template <typename T>
struct Kron3Params {
  const T* A;
  const T* B;
  const T* C;
  const T* X;
  T* Y;
  long long lda, ldb, ldc, ldx, ldx2, sx, ldy, ldy2, sy;
  long long m_a, n_a, m_b, n_b, m_c, n_c;
  long long batch;
  int opa, opb, opc;
  int beta_mode;
  T alpha, beta;
  // optional per-call tile counter (device, zeroed before the launch): kernels
  // that support it take tiles dynamically instead of round-robin, so SMs that
  // run slower (die / L2-slice distance) do less of the batch
  unsigned long long* sched = nullptr;
  // odd-n column-wise kernels, tight Y: mode 3 writes the tile's Y into a
  // shared-memory image and one bulk copy per tile stores it (set by the launcher)
  int ystage = 0;
  // odd-n column-wise kernels: bank-conflict-aware thread -> task maps
  // (kb_oddmaps.h) where one exists for the tile shape (launcher: KB_OM=0 off)
  int oddmap = 1;
};

// op-resolved element (i, j) of a stored matrix: op(M)(i, j)
template <typename T>
__device__ __forceinline__ T op_at(const T* m, long long ld, int trans, long long i, long long j) {
  return trans ? m[j + i * ld] : m[i + j * ld];
}

}  // namespace kb
