// Host cost of one library call through the C ABI (development aid): kb_skron2
// on device-resident X/Y (2-D fp32 n = 10), asynchronous on a caller stream,
// repeated; prints wall-clock microseconds per call for tiny batches (host-bound)
// and the configs[0] batch, plus the device time per call for reference.
//   build/microbench/call_overhead
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "kronbatch_b200.h"

int main() {
  const int n = 10, e = n * n;
  std::vector<float> a(e, 0.5f), b(e, 0.25f);
  float *A, *B, *X, *Y;
  const long long maxb = 65536;
  cudaMalloc(&A, e * 4);
  cudaMalloc(&B, e * 4);
  cudaMalloc(&X, e * 4 * maxb);
  cudaMalloc(&Y, e * 4 * maxb);
  cudaMemcpy(A, a.data(), e * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, b.data(), e * 4, cudaMemcpyHostToDevice);
  cudaMemset(X, 0, e * 4 * maxb);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  char err[256];
  for (int host_consts = 0; host_consts < 2; ++host_consts)
    for (long long batch : {1LL, 64LL, 65536LL}) {
      kb_exec ex{0, nullptr, s, KB_EXEC_ASYNC};
      const float* pa = host_consts ? a.data() : A;
      const float* pb = host_consts ? b.data() : B;
      auto call = [&]() {
        int rc = kb_skron2('N', 'N', 'N', n, n, n, n, batch, 1.0f, pa, n, e, pb, n, e, X, n, e, e * batch, 0.0f, Y, n,
                           e, e * batch, &ex, err, sizeof err);
        if (rc) std::printf("error %d: %s\n", rc, err);
      };
      for (int i = 0; i < 50; ++i) call();
      cudaStreamSynchronize(s);
      const int reps = 2000;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      const auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < reps; ++i) call();
      const auto t1 = std::chrono::steady_clock::now();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float dev_ms = 0;
      cudaEventElapsedTime(&dev_ms, e0, e1);
      std::printf("constants %-6s batch %6lld: host %.2f us/call (enqueue), stream %.2f us/call\n",
                  host_consts ? "host" : "device", batch,
                  std::chrono::duration<double, std::micro>(t1 - t0).count() / reps, dev_ms * 1e3 / reps);
    }
  return 0;
}
