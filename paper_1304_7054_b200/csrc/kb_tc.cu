// kb_tc.cu -- 3-D fp32 n = 16 Kronecker action on the 5th-generation tensor
// cores (tcgen05, kind::tf32) with 3xTF32 error compensation.
//
// Why: the exact CUDA-core kernel (kb_fast.cuh) is bound by the FFMA pipe and
// the shared-memory crossbar at ~60-65 % of the HBM roofline for this case
// (AI = 12 flop/B sits at the FP32 ridge; ncu in profiles/). The tensor cores
// have ~15x the FP32 throughput, so three TF32 products per term fit easily.
//
// Math (same mode order as the reference, kron3.hpp:147-163):
//   mode 1:  T1(i,m,n) = sum_l A(i,l) X(l,m,n)
//   mode 2:  T2(i,j,n) = sum_m T1(i,m,n) B(j,m)
//   mode 3:  Y(i,j,k)  = sum_n T2(i,j,n) Cw(k,n) (+ beta Y),  Cw = fl(alpha C_r)
// Every operand v is split v = hi + lo with hi = rna_tf32(v),
// lo = rna_tf32(v - hi); each mode is ONE chain of MMAs with the data operand
// stacked on K ([hi | lo], K = 32) and the constant stacked on N:
//   D[:, 0:16]  = hi*Ch + lo*Ch      D[:, 16:32] = hi*Cl       (lo*Cl ~ 2^-22 dropped)
// and the mode result is D[:, 0:16] + D[:, 16:32]. Relative error per product
// is ~2^-21, well inside the 1e-5 (fp32) tolerance; results are NOT bit-equal
// to the CPU path (use the default exact kernels for that).
//
// Per SM: one persistent CTA of GROUPS independent 4-warp groups. A group owns
// 128 TMEM lanes x 64 columns (A operand, 2 tiles x [hi|lo]) + 64 columns (D,
// 2 tiles x N = 32) and processes whole entries:
//   TMA (3-D tensor map, 64B swizzle) -> X tile in smem
//   X -> split -> tcgen05.st A1 -> MMA mode 1 (TS) -> D1
//   D1 -> sum -> 16x16 in-warp transpose (shuffles) -> split -> A2 -> MMA -> D2
//   D2 -> sum -> smem exchange (n <-> j) -> split -> A3 -> MMA -> D3
//   D3 -> sum (+ beta Y) -> Y in HBM
// The constant operands (32 x 32, [hi;lo] blocks) sit in shared memory in the
// canonical no-swizzle K-major UMMA layout. One elected thread per group issues
// the MMAs and commits them to the group's mbarrier.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "kb_device.cuh"
#include "kb_kernels.h"

namespace kb {
namespace tc {

constexpr int N = 16;
constexpr int GROUPS = 3;                 // 4-warp groups per CTA
constexpr int THREADS = GROUPS * 128;
constexpr int XSLOTS = 2;                 // X entry buffers per group
constexpr int XBYTES = N * N * N * 4;     // 16 KiB per entry
constexpr int BBYTES = 32 * 32 * 4;       // one constant operand tile
constexpr int EPAD = 20;                  // exchange row pitch (floats)
constexpr uint32_t TMEM_COLS = 512;
constexpr int GCOLS = 128;                // TMEM columns per group
// idesc: f32 accumulate, tf32 A/B, K-major A/B, N = 32, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

struct Smem {
  // X slots first: 1 KiB alignment for the swizzled TMA destination
  alignas(1024) unsigned char x[GROUPS][XSLOTS][XBYTES];
  alignas(1024) unsigned char b[3][BBYTES];  // mode 1/2/3 constant operands
  alignas(16) float e[GROUPS][N * N * EPAD];
  unsigned long long xbar[GROUPS][XSLOTS];
  unsigned long long dbar[GROUPS];
  unsigned tmem_base;
};

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

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
  unsigned r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

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

// canonical no-swizzle K-major descriptor: core matrices of 8 rows x 16 B,
// LBO = distance between the two K chunks of one MMA, SBO = between 8-row groups
__device__ __forceinline__ unsigned long long smem_desc(const void* p, unsigned lbo, unsigned sbo) {
  const unsigned long long addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------- operand construction --

// Constant operand tile (32 rows x K = 32) in the no-swizzle K-major layout:
// element (row, k) at ((k/4)*4 + row/8)*128 + (row%8)*16 + (k%4)*4 bytes
// (LBO = 512 B between K chunks, SBO = 128 B between 8-row groups).
//   rows 0..15: [ Mh(row, :) | Mh(row, :) ],  rows 16..31: [ Ml(row-16, :) | 0 ]
// where M(r, k) = the constant indexed (output row r, contraction k).
__device__ __forceinline__ void build_const_tile(unsigned char* dst, int row, int k, float v) {
  float* f = reinterpret_cast<float*>(dst + ((k / 4) * 4 + row / 8) * 128 + (row % 8) * 16 + (k % 4) * 4);
  *f = v;
}

__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - hi);
}

// 16x16 transpose inside each half-warp: lane l holds v[0..16) = row l of a
// 16x16 block; afterwards lane l holds column l (v[k] = old row k, entry l).
__device__ __forceinline__ void transpose16(float (&v)[16]) {
  const int lane = threadIdx.x & 15;
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool upper = lane & s;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if ((k & s) == 0) {
        const float send = upper ? v[k] : v[k + s];
        const float recv = __shfl_xor_sync(0xffffffffu, send, s);
        if (upper)
          v[k] = recv;
        else
          v[k + s] = recv;
      }
    }
  }
}

// ------------------------------------------------------------------ kernel --

__global__ void __launch_bounds__(THREADS, 1)
    kron3_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ Consts kc, float* __restrict__ Y,
                    long long ldy, long long ldy2, long long sy, long long batch, int beta_mode, float beta) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp >> 2;                 // group
  const int gt = tid & 127;                // thread within group
  const int lrow = ((warp & 3) << 5) | lane;  // TMEM lane == tile row
  const bool leader = gt == 0;

  // ---- setup: constant operand tiles, barriers, TMEM
  for (int t = tid; t < 32 * 32; t += THREADS) {
    const int row = t / 32, k = t % 32;
    const int r = row % 16, kk = k % 16;
    // mode 1: row = i (output), k = l ; M(i, l) = A_r(i, l)
    // mode 2: row = j,          k = m ; M(j, m) = B_r(j, m)
    // mode 3: row = k_out,      k = n ; M(k, n) = fl(alpha C_r(k, n))
    const float mv[3] = {kc.a[r + kk * N], kc.b[r * N + kk], kc.c[r * N + kk]};
#pragma unroll
    for (int md = 0; md < 3; ++md) {
      float hi, lo;
      split(mv[md], hi, lo);
      const float v = row < 16 ? hi : (k < 16 ? lo : 0.f);
      build_const_tile(sm.b[md], row, k, v);
    }
  }
  if (tid == 0) {
    for (int gg = 0; gg < GROUPS; ++gg) {
      for (int s = 0; s < XSLOTS; ++s) mbar_init(&sm.xbar[gg][s], 1);
      mbar_init(&sm.dbar[gg], 1);
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
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
  const unsigned tmem = sm.tmem_base + (unsigned)(g * GCOLS);
  const unsigned lane_off = (unsigned)((warp & 3) * 32) << 16;
  const unsigned a_col = tmem + 0, d_col = tmem + 64;  // [0,64): A tiles, [64,128): D tiles
  const unsigned long long bdesc0[3] = {smem_desc(sm.b[0], 512, 128), smem_desc(sm.b[1], 512, 128),
                                        smem_desc(sm.b[2], 512, 128)};

  // entries of this group: e = (blockIdx.x * GROUPS + g) + k * gridDim.x * GROUPS
  const long long stride = (long long)gridDim.x * GROUPS;
  const long long first = (long long)blockIdx.x * GROUPS + g;
  if (leader) {
    for (int s = 0; s < XSLOTS; ++s) {
      const long long e = first + s * stride;
      if (e < batch) {
        mbar_arrive_expect_tx(&sm.xbar[g][s], XBYTES);
        tma_load_3d(sm.x[g][s], &xmap, 0, 0, (int)e, &sm.xbar[g][s]);
      }
    }
  }
  unsigned xphase[XSLOTS] = {0, 0};
  unsigned dphase = 0;
  const int bar_id = 1 + g;  // named barrier per group

  // MMA chain for one mode: per tile, 4 K-steps of K = 8 (A cols 8s, B chunks 2s)
  auto issue_mode = [&](int md) {
    if (leader) {
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int s = 0; s < 4; ++s)
          mma_ts(d_col + t * 32, a_col + t * 32 + s * 8, bdesc0[md] + ((unsigned long long)((s * 2 * 512) >> 4)), s > 0);
      mma_commit(&sm.dbar[g]);
    }
  };
  auto wait_d = [&]() {
    mbar_wait(&sm.dbar[g], dphase);
    dphase ^= 1;
    tc_fence_after();
  };

  int slot = 0;
  for (long long e = first; e < batch; e += stride) {
    // ---- X (TMA, swizzled 64B rows) -> split -> A1 = [X_hi | X_lo] per tile
    mbar_wait(&sm.xbar[g][slot], xphase[slot]);
    xphase[slot] ^= 1;
    const unsigned char* xs = sm.x[g][slot];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int r = lrow + 128 * t;  // X row (m, n) = (r % 16, r / 16)
      float v[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 q = *reinterpret_cast<const float4*>(xs + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
        const float xv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) split(xv[u], v[c * 4 + u], v[16 + c * 4 + u]);
      }
      tmem_st32(a_col + t * 32 + lane_off, v);
    }
    tmem_st_wait();
    fence_proxy_async();  // X slot reads done before the TMA refill (async proxy)
    tc_fence_before();
    named_bar(bar_id, 128);
    if (leader) {
      const long long nx = e + XSLOTS * stride;
      if (nx < batch) {
        mbar_arrive_expect_tx(&sm.xbar[g][slot], XBYTES);
        tma_load_3d(sm.x[g][slot], &xmap, 0, 0, (int)nx, &sm.xbar[g][slot]);
      }
    }
    issue_mode(0);
    wait_d();

    // ---- D1 (rows (m, n), cols i) -> T1 -> transpose (lanes i) -> A2 = [hi | lo] over m
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      float d[32];
      tmem_ld32(d_col + t * 32 + lane_off, d);
      float v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = d[k] + d[16 + k];
      transpose16(v);  // lane (i = lrow%16): v[m] = T1(i, m, n)
      float a[32];
#pragma unroll
      for (int k = 0; k < 16; ++k) split(v[k], a[k], a[16 + k]);
      tmem_st32(a_col + t * 32 + lane_off, a);
    }
    tmem_st_wait();
    tc_fence_before();
    named_bar(bar_id, 128);
    issue_mode(1);
    wait_d();

    // ---- D2 (rows (i, n), cols j) -> T2 -> smem exchange -> rows (i, j), K = n
    float* ex = sm.e[g];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      float d[32];
      tmem_ld32(d_col + t * 32 + lane_off, d);
      const int i = lrow & 15, n = 8 * t + (lrow >> 4);
#pragma unroll
      for (int j = 0; j < 16; ++j) ex[(j * N + i) * EPAD + n] = d[j] + d[16 + j];
    }
    tc_fence_before();
    named_bar(bar_id, 128);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int i = lrow & 15, j = 8 * t + (lrow >> 4);  // mode-3 row (i, j) of tile t
      const float* src = ex + (j * N + i) * EPAD;
      float a[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 q = *reinterpret_cast<const float4*>(src + 4 * c);
        const float xv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) split(xv[u], a[c * 4 + u], a[16 + c * 4 + u]);
      }
      tmem_st32(a_col + t * 32 + lane_off, a);
    }
    tmem_st_wait();
    tc_fence_before();
    named_bar(bar_id, 128);
    issue_mode(2);
    wait_d();

    // ---- D3 (rows (i, j), cols k) -> Y(i, j, k)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      float d[32];
      tmem_ld32(d_col + t * 32 + lane_off, d);
      const int i = lrow & 15, j = 8 * t + (lrow >> 4);
      float* yp = Y + e * sy + (long long)j * ldy + i;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float r = d[k] + d[16 + k];
        if (beta_mode != kBetaZero) r += (beta_mode == kBetaOne) ? yp[k * ldy2] : beta * yp[k * ldy2];
        yp[k * ldy2] = r;
      }
    }
    tc_fence_before();
    named_bar(bar_id, 128);  // D / exchange buffers free for the next entry
    slot = (slot + 1) % XSLOTS;
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem_base), "r"(TMEM_COLS)
                 : "memory");
}

// ------------------------------------------------------------------ launch --

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

}  // namespace tc

cudaError_t launch_kron3_tc(const Kron3Params<float>& p, const float* ha, const float* hb, const float* hc,
                            int sm_count, cudaStream_t s) {
  using namespace tc;
  if (p.m_a != N || p.n_a != N || p.m_b != N || p.n_b != N || p.m_c != N || p.n_c != N) return cudaErrorNotSupported;
  if (p.ldx != N || p.ldx2 != N * N || (p.sx * 4) % 16 || (reinterpret_cast<uintptr_t>(p.X) % 16))
    return cudaErrorNotSupported;
  if (p.batch > 0x7fffffffLL) return cudaErrorNotSupported;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[3] = {16, 256, (cuuint64_t)p.batch};
  const cuuint64_t strides[2] = {64, (cuuint64_t)p.sx * 4};
  const cuuint32_t box[3] = {16, 256, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p.X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  Consts kc;
  for (int i = 0; i < N * N; ++i) {
    kc.a[i] = ha[i];
    kc.b[i] = hb[i];
    kc.c[i] = hc[i];
  }
  const size_t smem = sizeof(Smem) + 1024;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] {
    attr = cudaFuncSetAttribute(kron3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr != cudaSuccess) return attr;
  const long long groups_needed = (p.batch + GROUPS - 1) / GROUPS;
  const int grid = (int)(groups_needed < sm_count ? groups_needed : sm_count);
  kron3_tc_kernel<<<grid, THREADS, smem, s>>>(map, kc, p.Y, p.ldy, p.ldy2, p.sy, p.batch, p.beta_mode, p.beta);
  return cudaGetLastError();
}

}  // namespace kb
