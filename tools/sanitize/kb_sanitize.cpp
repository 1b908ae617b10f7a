// kb_sanitize.cpp -- one small call of every kernel family of
// libkronbatch_b200.so through the C ABI, on exactly-sized device buffers,
// for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
//
//   compute-sanitizer --tool memcheck --error-exitcode 1 build/sanitize/kb_sanitize [quick]
//
// Covers the square fast paths (every n = 1..16, fp32/fp64, 2-D op_x N and T,
// 3-D; ragged last groups: batch 37), the generic kernels (rectangular,
// padded), the beta-scale path, kron1 / gemm_a (square fast and generic) and
// the 3xTF32 tensor-core kron3. Batches are odd and buffers exactly sized, so
// a read past the last entry (e.g. a 16-byte-rounded span copy) is reported.
// No torch; exits non-zero if any call returns an error status.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <kronbatch_b200.h>

namespace {

int g_fail = 0;

void check(int rc, const char* what, const char* err) {
  if (rc != KB_OK) {
    std::fprintf(stderr, "FAIL %s: rc=%d %s\n", what, rc, err);
    ++g_fail;
  }
}

template <typename T>
T* dev_fill(size_t n, unsigned seed) {
  std::vector<T> h(n);
  for (size_t i = 0; i < n; ++i) {
    seed = seed * 1664525u + 1013904223u;
    h[i] = static_cast<T>((seed >> 8) * (1.0 / 16777216.0) * 2 - 1);
  }
  T* d = nullptr;
  if (cudaMalloc(&d, sizeof(T) * (n ? n : 1)) != cudaSuccess) {
    std::fprintf(stderr, "cudaMalloc failed\n");
    std::exit(2);
  }
  if (n) cudaMemcpy(d, h.data(), sizeof(T) * n, cudaMemcpyHostToDevice);
  return d;
}

template <typename T>
struct Abi;
template <>
struct Abi<float> {
  static constexpr auto k2 = kb_skron2;
  static constexpr auto k3 = kb_skron3;
  static constexpr auto k1 = kb_skron1;
  static constexpr auto ga = kb_sgemm_a;
  static constexpr const char* name = "f32";
};
template <>
struct Abi<double> {
  static constexpr auto k2 = kb_dkron2;
  static constexpr auto k3 = kb_dkron3;
  static constexpr auto k1 = kb_dkron1;
  static constexpr auto ga = kb_dgemm_a;
  static constexpr const char* name = "f64";
};

template <typename T>
void square2(int n, long long batch, char tx, T beta) {
  const long long e = (long long)n * n;
  T *A = dev_fill<T>(e, 1), *B = dev_fill<T>(e, 2), *X = dev_fill<T>(e * batch, 3), *Y = dev_fill<T>(e * batch, 4);
  char err[512] = {0};
  const int rc = Abi<T>::k2('N', 'T', tx, n, n, n, n, batch, T(0.5), A, n, e, B, n, e, X, n, e, e * batch, beta, Y, n,
                            e, e * batch, nullptr, err, sizeof err);
  std::string w = std::string("kron2 ") + Abi<T>::name + " n=" + std::to_string(n) + " opx=" + tx;
  check(rc, w.c_str(), err);
  cudaFree(A), cudaFree(B), cudaFree(X), cudaFree(Y);
}

template <typename T>
void square3(int n, long long batch, T beta, unsigned flags = 0) {
  const long long nn = (long long)n * n, e = nn * n;
  T *A = dev_fill<T>(nn, 1), *B = dev_fill<T>(nn, 2), *C = dev_fill<T>(nn, 3);
  T *X = dev_fill<T>(e * batch, 4), *Y = dev_fill<T>(e * batch, 5);
  char err[512] = {0};
  kb_exec ex{0, nullptr, nullptr, flags};
  const int rc = Abi<T>::k3('N', 'T', 'N', n, n, n, n, n, n, batch, T(0.75), A, n, nn, B, n, nn, C, n, nn, X, n, nn, e,
                            e * batch, beta, Y, n, nn, e, e * batch, nullptr, nn * n * batch, &ex, err, sizeof err);
  std::string w = std::string("kron3 ") + Abi<T>::name + " n=" + std::to_string(n) + (flags ? " tf32" : "");
  check(rc, w.c_str(), err);
  cudaFree(A), cudaFree(B), cudaFree(C), cudaFree(X), cudaFree(Y);
}

template <typename T>
void generic_shapes() {
  char err[512] = {0};
  {  // kron2 rectangular, padded X / Y
    const long long ma = 5, na = 7, mb = 6, nb = 3, batch = 33, ldx = na + 3, sx = ldx * nb + 5, ldy = ma + 2,
                    sy = ldy * mb + 1;
    T *A = dev_fill<T>(ma * na, 1), *B = dev_fill<T>(mb * nb, 2);
    T *X = dev_fill<T>(sx * (batch - 1) + ldx * nb, 3), *Y = dev_fill<T>(sy * (batch - 1) + ldy * mb, 4);
    const int rc = Abi<T>::k2('N', 'N', 'N', ma, na, mb, nb, batch, T(1.25), A, ma, ma * na, B, mb, mb * nb, X, ldx,
                              sx, sx * (batch - 1) + ldx * nb, T(0.5), Y, ldy, sy, sy * (batch - 1) + ldy * mb, nullptr,
                              err, sizeof err);
    check(rc, "kron2 generic", err);
    // alpha = 0: Y <- beta Y (scale kernel)
    const int rc2 = Abi<T>::k2('N', 'N', 'N', ma, na, mb, nb, batch, T(0), A, ma, ma * na, B, mb, mb * nb, X, ldx, sx,
                               sx * (batch - 1) + ldx * nb, T(-2), Y, ldy, sy, sy * (batch - 1) + ldy * mb, nullptr,
                               err, sizeof err);
    check(rc2, "kron2 scale", err);
    cudaFree(A), cudaFree(B), cudaFree(X), cudaFree(Y);
  }
  {  // kron3 rectangular with padding; n = 20 (> 16) square
    const long long ma = 4, na = 3, mb = 5, nb = 2, mc = 3, nc = 6, batch = 21;
    const long long ldx = na + 1, ldx2 = ldx * nb + 2, sx = ldx2 * nc + 3;
    const long long ldy = ma, ldy2 = ldy * mb, sy = ldy2 * mc;
    T *A = dev_fill<T>(ma * na, 1), *B = dev_fill<T>(mb * nb, 2), *C = dev_fill<T>(mc * nc, 3);
    const long long lx = sx * (batch - 1) + ldx2 * nc, ly = sy * batch;
    T *X = dev_fill<T>(lx, 4), *Y = dev_fill<T>(ly, 5);
    const int rc = Abi<T>::k3('T', 'N', 'T', ma, na, mb, nb, mc, nc, batch, T(1), A, na, ma * na, B, mb, mb * nb, C, nc,
                              mc * nc, X, ldx, ldx2, sx, lx, T(0), Y, ldy, ldy2, sy, ly, nullptr, ma * mb * nc * batch,
                              nullptr, err, sizeof err);
    check(rc, "kron3 generic", err);
    cudaFree(A), cudaFree(B), cudaFree(C), cudaFree(X), cudaFree(Y);
    const long long n = 20, e = n * n * n, b2 = 3;
    T *A2 = dev_fill<T>(n * n, 6), *B2 = dev_fill<T>(n * n, 7), *C2 = dev_fill<T>(n * n, 8);
    T *X2 = dev_fill<T>(e * b2, 9), *Y2 = dev_fill<T>(e * b2, 10);
    const int rc3 = Abi<T>::k3('N', 'N', 'N', n, n, n, n, n, n, b2, T(1), A2, n, n * n, B2, n, n * n, C2, n, n * n, X2,
                               n, n * n, e, e * b2, T(1), Y2, n, n * n, e, e * b2, nullptr, n * n * n * b2, nullptr,
                               err, sizeof err);
    check(rc3, "kron3 generic n=20 (scratch)", err);
    cudaFree(A2), cudaFree(B2), cudaFree(C2), cudaFree(X2), cudaFree(Y2);
  }
  for (int n : {3, 9, 16}) {  // kron1 square fast + generic
    const long long batch = 41;
    T *A = dev_fill<T>(n * n, 1), *X = dev_fill<T>(n * batch, 2), *Y = dev_fill<T>(n * batch, 3);
    int rc = Abi<T>::k1('T', n, n, batch, T(1), A, n, n * n, X, n, n * batch, T(0.5), Y, n, n * batch, nullptr, err,
                        sizeof err);
    check(rc, "kron1 square", err);
    rc = Abi<T>::k1('N', n - 1, n, batch, T(1), A, n, n * n, X, n, n * batch, T(0), Y, n, n * batch, nullptr, err,
                    sizeof err);
    check(rc, "kron1 generic", err);
    cudaFree(A), cudaFree(X), cudaFree(Y);
    T *Am = dev_fill<T>((long long)n * n * batch, 4), *Bm = dev_fill<T>(n * n, 5), *Cm = dev_fill<T>(n * n * batch, 6);
    rc = Abi<T>::ga('N', 'T', n, n, n, batch, T(1), Am, n, n * n, n * n * batch, Bm, n, n * n, T(0), Cm, n, n * n,
                    n * n * batch, nullptr, err, sizeof err);
    check(rc, "gemm_a square", err);
    rc = Abi<T>::ga('T', 'N', n, n - 1, n, batch, T(1), Am, n, n * n, n * n * batch, Bm, n, n * n, T(1), Cm, n, n * n,
                    n * n * batch, nullptr, err, sizeof err);
    check(rc, "gemm_a generic", err);
    cudaFree(Am), cudaFree(Bm), cudaFree(Cm);
  }
}

template <typename T>
void all(bool quick) {
  for (int n = 1; n <= 16; ++n) {
    if (quick && n != 3 && n != 9 && n != 10 && n != 16) continue;
    square2<T>(n, 37, 'N', T(0));
    square2<T>(n, 37, 'T', T(1.5));
    square3<T>(n, 37, T(0));
    if (!quick) square3<T>(n, 5, T(2));
  }
  generic_shapes<T>();
}

}  // namespace

int main(int argc, char** argv) {
  const bool quick = argc > 1 && std::strcmp(argv[1], "quick") == 0;
  all<float>(quick);
  all<double>(quick);
  square3<float>(16, 37, 0.0f, KB_EXEC_TF32);  // tcgen05 3xTF32
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::fprintf(stderr, "device error: %s\n", cudaGetErrorString(e));
    ++g_fail;
  }
  std::printf("kb_sanitize: %s, %llu kernel launches, %d failures\n", quick ? "quick" : "full",
              (unsigned long long)kb_launch_count(), g_fail);
  return g_fail ? 1 : 0;
}
