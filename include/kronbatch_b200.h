/*
 * kronbatch_b200.h -- C ABI of the B200 (sm_100a) batched Kronecker-product
 * action library (libkronbatch_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (/root/reference/proj) is a header-only C++ template library whose
 * operator API *is* the template signatures; it has no FFI. The entry points
 * below are what a foreign-language binding of that API would bind, with the
 * paper's BLAS-style parameter lists (TKRON2/TKRON3) plus
 * the reference's additions (independent X/Y batch strides, kron3 workspace,
 * SPEC.md:292). Each one replaces, one-for-one:
 *
 *   kb_skron2 / kb_dkron2  <- kronbatch::kron2<float|double>
 *                             proj/include/kronbatch/kron2.hpp:37-110
 *   kb_skron3 / kb_dkron3  <- kronbatch::kron3<float|double>
 *                             proj/include/kronbatch/kron3.hpp:72-166
 *   kb_kron3_workspace_size <- kronbatch::kron3_workspace_size
 *                             proj/include/kronbatch/kron3.hpp:43-53
 *   kb_skron1 / kb_dkron1  <- kronbatch::kron1<float|double>
 *                             proj/include/kronbatch/kron1.hpp:17-62
 *   kb_sgemm_a / kb_dgemm_a <- kronbatch::gemm_a<float|double>
 *                             proj/include/kronbatch/gemm_a.hpp:18-76
 *
 * The C++ header include/kronbatch/kronbatch.hpp re-exposes the reference's
 * template API unchanged on top of these.
 *
 * Conventions (same as the reference):
 *  - column-major; sizes, leading dimensions, strides and lengths in ELEMENTS;
 *  - trans* in {'N','T','C'} ('C' == 'T' for real types, types.hpp:27-29);
 *  - A is stored m_a x n_a when transa == 'N', n_a x m_a otherwise (same for
 *    B, C, and X with transx in 2-D: stored n_a x n_b or n_b x n_a);
 *  - len* = addressable elements from the pointer (the span length the
 *    reference views carry, views.hpp:14-20), used only for validation;
 *  - entry p of X starts at X + p*ldxp (ldxp = the reference's batch_stride);
 *  - beta == 0 never reads Y; alpha == 0 (or an empty sum) never reads
 *    A/B/C/X and sets Y <- beta*Y (README.md:71-72);
 *  - synchronous: Y is complete on return, unless exec->flags has
 *    KB_EXEC_ASYNC (device buffers only);
 *  - pointers may be device (cudaMalloc), managed, pinned host or pageable
 *    host memory; host buffers are staged through pooled device memory in
 *    chunks whose copies overlap the kernels (pageable ones through pooled
 *    pinned bounce buffers filled by several host threads).
 *
 * Return value: KB_OK or an error status; on error a NUL-terminated message
 * is written to err (if non-NULL) with the reference's exact wording, e.g.
 * "kron2: X: batch_stride (3) < (4), batch_stride < entry footprint".
 * KB_EINVAL maps to std::invalid_argument, KB_EOVERFLOW to std::overflow_error,
 * everything else to std::runtime_error.
 */
#ifndef KRONBATCH_B200_H
#define KRONBATCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  KB_OK = 0,
  KB_EINVAL = 1,    /* layout / dimension / workspace error (invalid_argument) */
  KB_EOVERFLOW = 2, /* index_t overflow (overflow_error) */
  KB_ECUDA = 3,     /* CUDA runtime / launch failure */
  KB_ENOMEM = 4,    /* device or pinned allocation failure */
  KB_EINTERNAL = 5
};

#define KB_EXEC_ASYNC 0x1u /* do not synchronize before returning */
#define KB_EXEC_TF32 0x2u  /* allow the tcgen05 3xTF32 tensor-core kernel for fp32 kron3 at n = 16
                              (|err| ~1e-6 relative, within the 1e-5 contract, not bit-exact);
                              also enabled process-wide by the environment variable KB_TF32=1 */

/* Execution options; pass NULL for the defaults (current device, library
 * stream, synchronous).
 *
 * Ordering: the library streams are blocking streams, so a call is ordered
 * after work the caller queued on the legacy default stream (stream 0) of the
 * buffers' device; with an explicit `stream` it is ordered on that stream.
 * Device-resident X/Y always run on the device they live on (a batch that is
 * already split over several GPUs goes through kb_*_parts below). */
typedef struct kb_exec {
  int32_t ndevices;       /* >1: shard a HOST-resident batch over devices[] by
                             contiguous slices [g*ceil(B/G), ...), one host
                             worker per slice, joined before return (host
                             barrier, no collective); 0/1: single device */
  const int32_t* devices; /* CUDA ordinals; NULL => current device */
  void* stream;           /* cudaStream_t for single-device calls; NULL => library stream */
  uint32_t flags;         /* KB_EXEC_* */
} kb_exec;

/* One part of a batch that is split over several GPUs (kb_*_parts). */
typedef struct kb_part {
  int32_t device;      /* GPU that runs the part: must be where X / Y live when
                          they are device memory; host-resident parts are staged
                          through this device */
  int64_t batch_count; /* entries in this part */
  const void* X;       /* entry 0 of the part (float* / double* per entry point) */
  int64_t lenx;        /* addressable elements from X */
  void* Y;
  int64_t leny;
  void* stream;        /* cudaStream_t on `device`; NULL => library stream */
} kb_part;

/* Y^p <- alpha * op(A) * op(X^p) * op(B)^T + beta * Y^p,  p < batch_count
 * (kron2.hpp:23-36). */
int kb_skron2(char transa, char transb, char transx, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
              int64_t batch_count, float alpha, const float* A, int64_t lda, int64_t lena, const float* B,
              int64_t ldb, int64_t lenb, const float* X, int64_t ldx, int64_t ldxp, int64_t lenx, float beta,
              float* Y, int64_t ldy, int64_t ldyp, int64_t leny, const kb_exec* exec, char* err, size_t errlen);
int kb_dkron2(char transa, char transb, char transx, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
              int64_t batch_count, double alpha, const double* A, int64_t lda, int64_t lena, const double* B,
              int64_t ldb, int64_t lenb, const double* X, int64_t ldx, int64_t ldxp, int64_t lenx, double beta,
              double* Y, int64_t ldy, int64_t ldyp, int64_t leny, const kb_exec* exec, char* err, size_t errlen);

/* vec(Y^p) <- alpha * (op(C) (x) op(B) (x) op(A)) vec(X^p) + beta * vec(Y^p)
 * (kron3.hpp:55-71). X^p is n_a x n_b x n_c with (ldx, ldx2), Y^p is
 * m_a x m_b x m_c with (ldy, ldy2). The workspace is only checked for
 * capacity (kron3.hpp:104-109): the sm_100a path keeps the intermediate
 * on chip and never touches it. work may be NULL when work_capacity suffices. */
int kb_skron3(char transa, char transb, char transc, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
              int64_t m_c, int64_t n_c, int64_t batch_count, float alpha, const float* A, int64_t lda,
              int64_t lena, const float* B, int64_t ldb, int64_t lenb, const float* C, int64_t ldc, int64_t lenc,
              const float* X, int64_t ldx, int64_t ldx2, int64_t ldxp, int64_t lenx, float beta, float* Y,
              int64_t ldy, int64_t ldy2, int64_t ldyp, int64_t leny, float* work, int64_t work_capacity,
              const kb_exec* exec, char* err, size_t errlen);
int kb_dkron3(char transa, char transb, char transc, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
              int64_t m_c, int64_t n_c, int64_t batch_count, double alpha, const double* A, int64_t lda,
              int64_t lena, const double* B, int64_t ldb, int64_t lenb, const double* C, int64_t ldc,
              int64_t lenc, const double* X, int64_t ldx, int64_t ldx2, int64_t ldxp, int64_t lenx, double beta,
              double* Y, int64_t ldy, int64_t ldy2, int64_t ldyp, int64_t leny, double* work,
              int64_t work_capacity, const kb_exec* exec, char* err, size_t errlen);

/* Multi-GPU form of kb_?kron2 / kb_?kron3 for batches that are already split
 * over devices (one device-resident slice per GPU, as a data-parallel caller
 * holds them). Same problem arguments as the single-call entry points; the
 * per-part X / Y / batch_count / device / stream come from parts[]. Every part
 * is validated before anything runs (errors are prefixed "part <i>: "), the
 * parts run concurrently, one per device, and the call returns when all are
 * done -- or, with KB_EXEC_ASYNC in flags and device-resident parts, once
 * all are queued on their streams. No collective, no peer traffic. kron3 takes
 * no workspace here (the sm_100a path never uses one). Bit-identical to one
 * call over the concatenated batch. */
int kb_skron2_parts(char transa, char transb, char transx, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
                    float alpha, const float* A, int64_t lda, int64_t lena, const float* B, int64_t ldb,
                    int64_t lenb, int64_t ldx, int64_t ldxp, float beta, int64_t ldy, int64_t ldyp, int32_t nparts,
                    const kb_part* parts, uint32_t flags, char* err, size_t errlen);
int kb_dkron2_parts(char transa, char transb, char transx, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
                    double alpha, const double* A, int64_t lda, int64_t lena, const double* B, int64_t ldb,
                    int64_t lenb, int64_t ldx, int64_t ldxp, double beta, int64_t ldy, int64_t ldyp, int32_t nparts,
                    const kb_part* parts, uint32_t flags, char* err, size_t errlen);
int kb_skron3_parts(char transa, char transb, char transc, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
                    int64_t m_c, int64_t n_c, float alpha, const float* A, int64_t lda, int64_t lena, const float* B,
                    int64_t ldb, int64_t lenb, const float* C, int64_t ldc, int64_t lenc, int64_t ldx, int64_t ldx2,
                    int64_t ldxp, float beta, int64_t ldy, int64_t ldy2, int64_t ldyp, int32_t nparts,
                    const kb_part* parts, uint32_t flags, char* err, size_t errlen);
int kb_dkron3_parts(char transa, char transb, char transc, int64_t m_a, int64_t n_a, int64_t m_b, int64_t n_b,
                    int64_t m_c, int64_t n_c, double alpha, const double* A, int64_t lda, int64_t lena,
                    const double* B, int64_t ldb, int64_t lenb, const double* C, int64_t ldc, int64_t lenc,
                    int64_t ldx, int64_t ldx2, int64_t ldxp, double beta, int64_t ldy, int64_t ldy2, int64_t ldyp,
                    int32_t nparts, const kb_part* parts, uint32_t flags, char* err, size_t errlen);

/* y^p <- alpha * op(A) * x^p + beta * y^p,  p < batch_count (kron1.hpp:9-16),
 * replaces kronbatch::kron1<float|double> (proj/include/kronbatch/kron1.hpp:17-62).
 * A is stored m_a x n_a (transa 'N') or n_a x m_a; x^p is n_a contiguous
 * elements at X + p*ldxp, y^p m_a contiguous elements at Y + p*ldyp. */
int kb_skron1(char transa, int64_t m_a, int64_t n_a, int64_t batch_count, float alpha, const float* A, int64_t lda,
              int64_t lena, const float* X, int64_t ldxp, int64_t lenx, float beta, float* Y, int64_t ldyp,
              int64_t leny, const kb_exec* exec, char* err, size_t errlen);
int kb_dkron1(char transa, int64_t m_a, int64_t n_a, int64_t batch_count, double alpha, const double* A, int64_t lda,
              int64_t lena, const double* X, int64_t ldxp, int64_t lenx, double beta, double* Y, int64_t ldyp,
              int64_t leny, const kb_exec* exec, char* err, size_t errlen);

/* C^p <- alpha * op(A^p) * op(B) + beta * C^p,  p < batch_count (gemm_a.hpp:9-17),
 * replaces kronbatch::gemm_a<float|double> (proj/include/kronbatch/gemm_a.hpp:18-76).
 * op(A^p) is m x k (A^p stored m x k or k x m with lda, at A + p*ldap), op(B)
 * is k x n (B stored k x n or n x k with ldb), C^p is m x n with ldc at
 * C + p*ldcp. parallel_hint is accepted and ignored (it only chunks the CPU
 * worker loop in the reference). */
int kb_sgemm_a(char transa, char transb, int64_t m, int64_t n, int64_t k, int64_t batch_count, float alpha,
               const float* A, int64_t lda, int64_t ldap, int64_t lena, const float* B, int64_t ldb, int64_t lenb,
               float beta, float* C, int64_t ldc, int64_t ldcp, int64_t lenc, const kb_exec* exec, char* err,
               size_t errlen);
int kb_dgemm_a(char transa, char transb, int64_t m, int64_t n, int64_t k, int64_t batch_count, double alpha,
               const double* A, int64_t lda, int64_t ldap, int64_t lena, const double* B, int64_t ldb, int64_t lenb,
               double beta, double* C, int64_t ldc, int64_t ldcp, int64_t lenc, const kb_exec* exec, char* err,
               size_t errlen);

/* Elements of workspace kron3 needs: m_a*m_b*n_c*batch_count. KB_EINVAL on
 * a negative dimension, KB_EOVERFLOW if the product overflows int64. */
int kb_kron3_workspace_size(int64_t m_a, int64_t m_b, int64_t n_c, int64_t batch_count, int64_t* out, char* err,
                            size_t errlen);

/* ---- library introspection (bench / tests) ---- */
const char* kb_version(void);
/* kernels this process has launched through the library (all devices) */
uint64_t kb_launch_count(void);
/* name of the kernel the last call on this thread launched ("" if none):
 * "kron2_fast", "kron2_generic", "kron3_fast", "kron3_generic", "kron1", "gemm_a", "scale" */
const char* kb_last_path(void);
/* release the pooled device / pinned buffers and streams of every idle lane
 * (all devices; lanes of calls in flight are kept) */
void kb_release_buffers(void);
/* device bytes currently held by the pool on `device` (-1: all devices) */
uint64_t kb_pooled_bytes(int device);

#ifdef __cplusplus
}
#endif

#endif /* KRONBATCH_B200_H */
