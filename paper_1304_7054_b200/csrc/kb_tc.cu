// kb_tc.cu -- 3-D fp32 n = 16 Kronecker action on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, accumulators in TMEM) with 3xTF32 error
// compensation. Opt-in (KB_EXEC_TF32 / KB_TF32=1): tolerance-level parity
// (1e-5, tests/test_gpu_tc.py), not bit-identical to the reference's FMA chain.
//
// Why: the exact CUDA-core kernel (kb_cw3.cuh) is bound by the FFMA pipe at
// n = 16 (AI = 12 flop/B sits at the FP32 ridge; ncu in profiles/); the
// tensor cores have ~15x the FP32 rate, so three TF32 products per term fit.
//
// Math (the reference's mode order, kron3.hpp:147-163):
//   mode 1:  T1(i,m,n) = sum_l A(i,l) X(l,m,n)
//   mode 2:  T2(i,j,n) = sum_m T1(i,m,n) B(j,m)
//   mode 3:  Y(i,j,k)  = sum_n T2(i,j,n) Cw(k,n) (+ beta Y),  Cw = fl(alpha C_r)
// Each mode is a [256 x 16] x [16 x 16] product per entry (2 M = 128 tiles).
// The data operand v is split v = hi + lo, hi = v rounded to TF32 (integer
// round-to-nearest on the bit pattern: 2 integer ops), lo = v - hi (exact);
// the constants likewise (once per CTA). Per tile, six M128 x N16 x K8 MMAs
// accumulate hi*Ch + lo*Ch + hi*Cl into ONE TMEM accumulator (lo*Cl ~ 2^-22
// dropped): relative error per product ~2^-21.
//
// Layout of the work (one persistent CTA per SM, WGS independent 4-warp
// groups; a group owns 128 TMEM lanes x 128 columns and a 17 KB smem slice):
//   X rows (m, n) of an entry -> registers (LDG, prefetched one entry ahead)
//   -> split -> tcgen05.st A (lanes = rows (m, n), cols = [hi | lo] over l)
//   -> MMA mode 1 (A from TMEM, constants from smem) -> D1 (cols i)
//   -> tcgen05.ld -> 16x16 transpose per plane through the warp's smem slice
//      (rows become (i, n): the SAME TMEM lane) -> split -> A -> MMA mode 2
//   -> tcgen05.ld D2 -> exchange (n <-> j) through the group's smem slice
//      -> split -> A (rows (i, j), cols n) -> MMA mode 3
//   -> tcgen05.ld D3 (cols k) -> Y(i, j, k), coalesced 128 B per warp store.
// One elected thread per group issues the MMAs and commits them to the
// group's mbarrier; the other groups' data movement overlaps its MMA latency.
// Nothing but X and Y touches HBM (no workspace, no intermediate round trip).
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "kb_device.cuh"
#include "kb_kernels.h"

namespace kb {
namespace tc {

constexpr int N = 16;
constexpr int WGS_DEFAULT = 4;          // independent 4-warp groups per CTA (KB_TC_WGS: 2..5)
constexpr uint32_t TMEM_COLS = 512;
constexpr int WG_COLS = 96;             // per group: A [0, 64) (2 tiles x [hi|lo]), D [64, 96) (2 tiles x 16)
// instruction descriptor: D f32, A/B tf32, both K-major, N = 16, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
// constant operand tile: 16 (n) x 16 (k), canonical no-swizzle K-major layout,
// core matrices 8 rows x 16 B; SBO = 128 B between the two 8-row groups,
// LBO = 256 B between K chunks of 4; one K = 8 MMA step spans 512 B.
constexpr int CT_BYTES = 1024;
// per-group smem slice (floats): mode-2 transposes (4 warps x 2 tiles x 2 planes x 336)
// and the mode-3 exchange (256 rows (j, i) x 17) share it
constexpr int TP_RS = 20, TP_PS = 336;  // conflict-free 16x16 transposes (see transpose_planes)
constexpr int EX_IS = 17;               // exchange: element (j, i, n) at (j * 16 + i) * 17 + n
constexpr int SLICE = 4 * 4 * TP_PS;    // 5376 floats: 4 warps x 4 planes of transposes >= 256 * 17 exchange

template <int WGS>
struct Smem {
  alignas(128) unsigned char ct[3][2][CT_BYTES];  // [mode][hi, lo] (no-swizzle operands: 16-byte alignment suffices)
  alignas(16) float slice[WGS][SLICE];
  alignas(128) float ystage[WGS][N * N * N];  // Y staging for the bulk store (tight Y, beta = 0)
  unsigned long long dbar[WGS];
  unsigned tmem_base;
};

#ifdef KB_TC_TRACE  // development: per-phase clock stamps of group 0 of CTA 0 (tools/microbench/tc_trace.cu)
__device__ long long g_tc_trace[64][16];
#define TC_STAMP(k)                                                                   \
  do {                                                                                \
    if (blockIdx.x == 0 && g == 0 && (tid & 127) == 0 && it < 64) g_tc_trace[it][k] = clock64(); \
  } while (0)
#else
#define TC_STAMP(k) \
  do {              \
  } while (0)
#endif

struct Consts {
  float a[N * N];  // A_r col-major: a[i + l*N]
  float b[N * N];  // B_r row-major: b[j*N + m]
  float c[N * N];  // fl(alpha*C_r) row-major: c[k*N + n]
};

// ---------------------------------------------------------------- PTX ---

__device__ __forceinline__ float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// v = hi + lo, hi = v rounded to 10 explicit mantissa bits (ties away from
// zero, on the bit pattern), lo = v - hi exactly (Sterbenz). Finite inputs.
__device__ __forceinline__ void split_fast(float v, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u);
  lo = v - hi;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(unsigned taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_ts(unsigned d, unsigned a, unsigned long long bdesc, bool acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(IDESC), "r"((unsigned)acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ unsigned long long smem_desc(const void* p, unsigned lbo, unsigned sbo) {
  const unsigned long long addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// element (n, k) of a 16 x 16 constant operand tile
__device__ __forceinline__ float* ct_at(unsigned char* t, int n, int k) {
  return reinterpret_cast<float*>(t + (k / 4) * 256 + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4);
}

// ------------------------------------------------------------------ kernel --

template <int WGS>
__global__ void __launch_bounds__(WGS * 128, 1)
    kron3_tc_kernel(const float* __restrict__ X, long long sx, const __grid_constant__ Consts kc,
                    float* __restrict__ Y, long long ldy, long long ldy2, long long sy, long long batch, int beta_mode,
                    float beta) {
  // used in place (no integer re-alignment of the pointer: that would drop the
  // shared address space and turn every LDS/STS into a generic LD/ST)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int THREADS = WGS * 128;
  Smem<WGS>& sm = *reinterpret_cast<Smem<WGS>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp >> 2;               // group
  const int wq = warp & 3;               // warp within the group = TMEM lane quarter
  const int L = (wq << 5) | lane;        // TMEM lane == tile row
  const bool leader = (tid & 127) == 0;

  // ---- setup: constant operand tiles (hi / lo), barriers, TMEM
  for (int t = tid; t < 3 * N * N; t += THREADS) {
    const int md = t / (N * N), r = (t / N) % N, k = t % N;
    // B operand element (n = output index r, k = contraction index)
    const float v = md == 0 ? kc.a[r + k * N] : (md == 1 ? kc.b[r * N + k] : kc.c[r * N + k]);
    const float hi = tf32_rna(v);
    *ct_at(sm.ct[md][0], r, k) = hi;
    *ct_at(sm.ct[md][1], r, k) = tf32_rna(v - hi);
  }
  if (tid == 0) {
    for (int gg = 0; gg < WGS; ++gg) mbar_init(&sm.dbar[gg], 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();  // constant tiles (generic writes) -> visible to the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tbase = sm.tmem_base + (unsigned)(g * WG_COLS) + ((unsigned)(wq * 32) << 16);
  const unsigned a_col = sm.tmem_base + (unsigned)(g * WG_COLS);  // MMA operands: lane 0 of the group's columns
  const unsigned d_col = a_col + 64;
  unsigned long long bd[3][2];
#pragma unroll
  for (int md = 0; md < 3; ++md)
#pragma unroll
    for (int h = 0; h < 2; ++h) bd[md][h] = smem_desc(sm.ct[md][h], 256, 128);
  float* slice = sm.slice[g];
  const int bar_id = 1 + g;
  const bool ybulk = beta_mode == kBetaZero && ldy == N && ldy2 == N * N && sy % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(Y) & 15) == 0;

  // entries of this group: e = first + k * stride
  const long long stride = (long long)gridDim.x * WGS;
  const long long first = (long long)blockIdx.x * WGS + g;
  unsigned dphase = 0;

  // one mode: per tile, hi*Ch (2 K-steps), lo*Ch (2), hi*Cl (2) into D (N = 16)
  auto issue_mode = [&](int md) {
    if (leader) {
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const unsigned d = d_col + t * 16, a = a_col + t * 32;
        mma_ts(d, a + 0, bd[md][0], false);
        mma_ts(d, a + 8, bd[md][0] + (512 >> 4), true);
        mma_ts(d, a + 16, bd[md][0], true);
        mma_ts(d, a + 24, bd[md][0] + (512 >> 4), true);
        mma_ts(d, a + 0, bd[md][1], true);
        mma_ts(d, a + 8, bd[md][1] + (512 >> 4), true);
      }
      mma_commit(&sm.dbar[g]);
    }
  };
  auto sync_group = [&]() {  // all A stores of the group done -> one thread issues
    tmem_st_wait();
    tc_fence_before();
    named_bar(bar_id, 128);
  };
  auto wait_d = [&]() {
    mbar_wait(&sm.dbar[g], dphase);
    dphase ^= 1;
    tc_fence_after();
  };
  auto split_store = [&](const float (&v)[16], int t) {  // A tile t = [hi | lo] over K
    float a[32];
#pragma unroll
    for (int k = 0; k < 16; ++k) split_fast(v[k], a[k], a[16 + k]);
    tmem_st32(tbase + t * 32, a);
  };

  // X row (m, n) = tile t row L -> 16 floats at X + e*sx + (128 t + L) * 16
  float4 xn[2][4];
  auto load_x = [&](long long e) {
    if (e < batch) {
      const float4* src = reinterpret_cast<const float4*>(X + e * sx) + L * 4;
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int c = 0; c < 4; ++c) xn[t][c] = __ldcs(src + t * 512 + c);
    }
  };
  load_x(first);

  int it = 0;
  (void)it;
  for (long long e = first; e < batch; e += stride, ++it) {
    TC_STAMP(0);
    // ---- mode 1: A = X rows (m, n) x l
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const float v[16] = {xn[t][0].x, xn[t][0].y, xn[t][0].z, xn[t][0].w, xn[t][1].x, xn[t][1].y,
                           xn[t][1].z, xn[t][1].w, xn[t][2].x, xn[t][2].y, xn[t][2].z, xn[t][2].w,
                           xn[t][3].x, xn[t][3].y, xn[t][3].z, xn[t][3].w};
      split_store(v, t);
    }
    load_x(e + stride);  // the next entry's X streams in under the three modes below
    sync_group();
    TC_STAMP(1);
    issue_mode(0);
    wait_d();
    TC_STAMP(2);

    // ---- mode 2: D1 (lanes (m, n), cols i) -> transpose per plane -> lanes (i, n), cols m
    {
      float d[2][16];
      tmem_ld16(tbase + 64, d[0]);
      tmem_ld16(tbase + 80, d[1]);
      tmem_ld_wait();
      TC_STAMP(8);
      const int r16 = lane & 15;
      float* tp = slice + (wq * 4 + (lane >> 4)) * TP_PS;  // this lane's plane in tile 0 (tile 1: +2 planes)
#ifdef KB_TC_EXP_NO_T2  // timing experiment only: skip the transposes' stores
      if (d[0][0] == 12345.f)
#endif
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int i = 0; i < 16; ++i) tp[t * 2 * TP_PS + i * TP_RS + r16] = d[t][i];  // 32 consecutive banks per i
      __syncwarp();
      TC_STAMP(9);
      float v[2][16];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 q = *reinterpret_cast<const float4*>(tp + t * 2 * TP_PS + r16 * TP_RS + 4 * c);  // row i = r16
          v[t][4 * c] = q.x, v[t][4 * c + 1] = q.y, v[t][4 * c + 2] = q.z, v[t][4 * c + 3] = q.w;
        }
      split_store(v[0], 0);
      split_store(v[1], 1);
      TC_STAMP(10);
      tmem_st_wait();
      TC_STAMP(11);
    }
    sync_group();  // (also orders the transposes' reads before the slice's reuse by the exchange)
    TC_STAMP(3);
    issue_mode(1);
    wait_d();
    TC_STAMP(4);

    // ---- mode 3: D2 (lanes (i, n), cols j) -> exchange -> lanes (i, j), cols n
    {
      const int i = L & 15;
      float d[2][16];
      tmem_ld16(tbase + 64, d[0]);
      tmem_ld16(tbase + 80, d[1]);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        float* dst = slice + i * EX_IS + 8 * t + (L >> 4);  // (j, i, n = 8t + L/16) at (j*16 + i)*17 + n
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[j * 16 * EX_IS] = d[t][j];
      }
      named_bar(bar_id, 128);
      float v[2][16];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float* src = slice + ((8 * t + (L >> 4)) * 16 + i) * EX_IS;  // row (i, j = 8t + L/16)
#pragma unroll
        for (int n = 0; n < 16; ++n) v[t][n] = src[n];
      }
      split_store(v[0], 0);
      split_store(v[1], 1);
    }
    if (ybulk && leader) bulk_wait_read();  // the previous entry's Y has left the staging buffer
    sync_group();  // (also: every exchange read is done before the slice is reused)
    TC_STAMP(5);
    issue_mode(2);
    wait_d();
    TC_STAMP(6);

    // ---- D3 (lanes (i, j), cols k) -> Y(i, j, k): per k, a warp stores 128 contiguous bytes
    {
      float d[2][16];
      tmem_ld16(tbase + 64, d[0]);
      tmem_ld16(tbase + 80, d[1]);
      tmem_ld_wait();
      TC_STAMP(12);
      if (ybulk) {
        // tight Y, beta = 0: stage the entry in the group's slice in Y's own
        // layout (k*256 + 16 j + i: per k a warp writes 32 consecutive words)
        // and let one thread's bulk copy (TMA engine) write the 16 KB to HBM
        float* st = sm.ystage[g] + 16 * (L >> 4) + (L & 15);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int k = 0; k < 16; ++k) st[t * 128 + k * 256] = d[t][k];
        fence_proxy_async();
        named_bar(bar_id, 128);
        if (leader) {
          bulk_s2g(Y + e * sy, sm.ystage[g], N * N * N * 4);
          bulk_commit();
        }
      } else {
        float* yp = Y + e * sy + (long long)(L >> 4) * ldy + (L & 15);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          float* yt = yp + (long long)(8 * t) * ldy;
          if (beta_mode == kBetaZero) {
#pragma unroll
            for (int k = 0; k < 16; ++k) __stcs(yt + k * ldy2, d[t][k]);
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const float y0 = yt[k * ldy2];
              yt[k * ldy2] = d[t][k] + (beta_mode == kBetaOne ? y0 : beta * y0);
            }
          }
        }
      }
    }
    TC_STAMP(7);
    tc_fence_before();  // D reads done before the next entry's MMAs overwrite it (ordered by sync_group)
  }

  if (ybulk && leader) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_base), "r"(TMEM_COLS)
                 : "memory");
}

template <int WGS>
cudaError_t launch_tc(const Kron3Params<float>& p, const Consts& kc, int sm_count, cudaStream_t s) {
  // >= 114 KB: exactly one CTA per SM (each CTA allocates all 512 TMEM columns)
  const size_t smem = sizeof(Smem<WGS>) > (size_t)(120 << 10) ? sizeof(Smem<WGS>) : (size_t)(120 << 10);
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] {
    attr = cudaFuncSetAttribute(kron3_tc_kernel<WGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr != cudaSuccess) return attr;
  const long long groups_needed = (p.batch + WGS - 1) / WGS;
  const int grid = (int)(groups_needed < sm_count ? groups_needed : sm_count);
  kron3_tc_kernel<WGS><<<grid, WGS * 128, smem, s>>>(p.X, p.sx, kc, p.Y, p.ldy, p.ldy2, p.sy, p.batch, p.beta_mode,
                                                      p.beta);
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t launch_kron3_tc(const Kron3Params<float>& p, const float* ha, const float* hb, const float* hc,
                            int sm_count, cudaStream_t s) {
  using namespace tc;
  if (p.m_a != N || p.n_a != N || p.m_b != N || p.n_b != N || p.m_c != N || p.n_c != N) return cudaErrorNotSupported;
  if (p.ldx != N || p.ldx2 != N * N || p.sx % 4 || (reinterpret_cast<uintptr_t>(p.X) % 16)) return cudaErrorNotSupported;
  Consts kc;
  for (int i = 0; i < N * N; ++i) {
    kc.a[i] = ha[i];
    kc.b[i] = hb[i];
    kc.c[i] = hc[i];
  }
  static const int wgs = [] {
    const char* v = std::getenv("KB_TC_WGS");  // development sweeps
    const int w = v ? std::atoi(v) : WGS_DEFAULT;
    return w < 2 ? 2 : (w > 5 ? 5 : w);
  }();
  switch (wgs) {
    case 2: return launch_tc<2>(p, kc, sm_count, s);
    case 3: return launch_tc<3>(p, kc, sm_count, s);
    case 5: return launch_tc<5>(p, kc, sm_count, s);
    default: return launch_tc<4>(p, kc, sm_count, s);
  }
}

}  // namespace kb
