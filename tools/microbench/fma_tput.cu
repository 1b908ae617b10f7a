// Microbenchmark: FP32 FFMA / FFMA2 (fma.rn.f32x2) / FP64 DFMA issue throughput
// on sm_100a, to size the CUDA-core kron kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int CH>
__global__ void k_ffma(float* out, float s, int iters) {
  float acc[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) acc[i] = threadIdx.x * 1e-3f + i;
  float b = s * 0.5f, c = s;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) acc[i] = __fmaf_rn(acc[i], b, c);
#pragma unroll
    for (int i = 0; i < CH; i++) acc[i] = __fmaf_rn(acc[i], c, b);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// FFMA2 with a scalar broadcast operand, as used by the kron kernels
template <int CH>
__global__ void k_ffma2(float* out, float s, int iters) {
  unsigned long long acc[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    float2 f = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    acc[i] = *reinterpret_cast<unsigned long long*>(&f);
  }
  float2 bb = make_float2(s * 0.5f, s * 0.25f);
  unsigned long long b = *reinterpret_cast<unsigned long long*>(&bb);
  float c = s;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      float2 cc = make_float2(c, c);
      acc[i] = ffma2(b, acc[i], *reinterpret_cast<unsigned long long*>(&cc));
    }
#pragma unroll
    for (int i = 0; i < CH; i++) {
      float2 cc = make_float2(c, c);
      acc[i] = ffma2(acc[i], *reinterpret_cast<unsigned long long*>(&cc), b);
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) {
    float2 f = *reinterpret_cast<float2*>(&acc[i]);
    r += f.x + f.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int CH>
__global__ void k_dfma(double* out, double s, int iters) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) acc[i] = threadIdx.x * 1e-3 + i;
  double b = s * 0.5, c = s;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) acc[i] = __fma_rn(acc[i], b, c);
#pragma unroll
    for (int i = 0; i < CH; i++) acc[i] = __fma_rn(acc[i], c, b);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d l2 %d MB clockRate(kHz) %d smemPerBlockOptin %zu regsPerSM %d\n", p.name,
         p.multiProcessorCount, p.l2CacheSize >> 20, clk, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  const int sms = p.multiProcessorCount;
  float* out;
  cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 20000;
  auto run = [&](const char* name, auto kern, int threads, int blocks_per_sm, double flops_per_thread_iter) {
    kern<<<sms * blocks_per_sm, threads>>>(out, 1.0001f, 100);
    cudaEventRecord(e0);
    kern<<<sms * blocks_per_sm, threads>>>(out, 1.0001f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = flops_per_thread_iter * iters * threads * (double)sms * blocks_per_sm;
    printf("%-28s threads %4d blk/SM %d: %8.3f ms  %8.2f TFLOP/s\n", name, threads, blocks_per_sm, ms, fl / ms / 1e9);
  };
  for (int bps : {1, 2, 4}) {
    run("ffma CH=8", k_ffma<8>, 256, bps, 2.0 * 16);
    run("ffma CH=16", k_ffma<16>, 256, bps, 2.0 * 32);
    run("ffma2 CH=8", k_ffma2<8>, 256, bps, 4.0 * 16);
    run("ffma2 CH=16", k_ffma2<16>, 256, bps, 4.0 * 32);
  }
  auto rund = [&](const char* name, auto kern, int threads, int blocks_per_sm, double flops_per_thread_iter) {
    kern<<<sms * blocks_per_sm, threads>>>((double*)out, 1.0001, 100);
    cudaEventRecord(e0);
    kern<<<sms * blocks_per_sm, threads>>>((double*)out, 1.0001, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = flops_per_thread_iter * iters * threads * (double)sms * blocks_per_sm;
    printf("%-28s threads %4d blk/SM %d: %8.3f ms  %8.2f TFLOP/s\n", name, threads, blocks_per_sm, ms, fl / ms / 1e9);
  };
  for (int bps : {1, 2, 4}) {
    rund("dfma CH=8", k_dfma<8>, 256, bps, 2.0 * 16);
    rund("dfma CH=16", k_dfma<16>, 256, bps, 2.0 * 32);
  }
  size_t bytes = size_t(4) << 30;
  float4 *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 0, bytes);
  for (int g : {sms * 4, sms * 8, sms * 16}) {
    k_copy<<<g, 512>>>(a, b, bytes / 16);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k_copy<<<g, 512>>>(a, b, bytes / 16);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid %d: %.1f GB/s\n", g, 2.0 * bytes * 5 / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
