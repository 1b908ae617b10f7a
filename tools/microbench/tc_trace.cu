// tc_trace.cu -- per-phase clock breakdown of the tcgen05 kron3 kernel
// (kb_tc.cu built with KB_TC_TRACE): group 0 of CTA 0, entries 8..63.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DKB_TC_TRACE \
//        -Ipaper_1304_7054_b200/csrc tools/microbench/tc_trace.cu -o /tmp/tc_trace
#include "../../paper_1304_7054_b200/csrc/kb_tc.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const long long batch = 262144;
  const int wgs = argc > 1 ? std::atoi(argv[1]) : 4;
  float *X, *Y;
  cudaMalloc(&X, sizeof(float) * 4096 * batch);
  cudaMalloc(&Y, sizeof(float) * 4096 * batch);
  cudaMemset(X, 0, sizeof(float) * 4096 * batch);
  std::vector<float> h(256, 0.01f);
  kb::Kron3Params<float> p{};
  p.X = X, p.Y = Y, p.ldx = 16, p.ldx2 = 256, p.sx = 4096, p.ldy = 16, p.ldy2 = 256, p.sy = 4096;
  p.m_a = p.n_a = p.m_b = p.n_b = p.m_c = p.n_c = 16;
  p.batch = batch;
  p.beta_mode = kb::kBetaZero;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  setenv("KB_TC_WGS", argv[1] ? argv[1] : "4", 1);
  for (int r = 0; r < 3; ++r) kb::launch_kron3_tc(p, h.data(), h.data(), h.data(), sms, nullptr);
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  cudaEventRecord(a);
  kb::launch_kron3_tc(p, h.data(), h.data(), h.data(), sms, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long tr[64][16];
  cudaMemcpyFromSymbol(tr, kb::tc::g_tc_trace, sizeof tr);
  const char* names[7] = {"mode1 prep", "MMA1 wait", "mode2 prep", "MMA2 wait", "mode3 prep", "MMA3 wait", "Y store"};
  double sum[8] = {0}, tot = 0;
  int n = 0;
  for (int e = 8; e < 63; ++e, ++n) {
    for (int k = 0; k < 7; ++k) sum[k] += tr[e][k + 1] - tr[e][k];
    tot += tr[e + 1][0] - tr[e][0];
  }
  std::printf("WGS=%d  %.3f ms  (%.1f TF/s)\n", wgs, ms, 6.0 * 65536 * batch / (ms * 1e-3) / 1e12);
  for (int k = 0; k < 7; ++k) std::printf("  %-11s %7.0f clk\n", names[k], sum[k] / n);
  std::printf("  entry total %7.0f clk (group 0 of CTA 0)\n", tot / n);
  double f[6] = {0};
  for (int e = 8; e < 63; ++e) {
    f[0] += tr[e][8] - tr[e][2];   // mode 2: LDTM x2 + wait
    f[1] += tr[e][9] - tr[e][8];   // transposes' STS + syncwarp
    f[2] += tr[e][10] - tr[e][9];  // LDS + split + STTM issue
    f[3] += tr[e][11] - tr[e][10]; // tcgen05.wait::st
    f[4] += tr[e][3] - tr[e][11];  // group barrier
    f[5] += tr[e][12] - tr[e][6];  // Y: LDTM x2 + wait
  }
  const char* fn[6] = {"m2 ldtm+wait", "m2 sts", "m2 lds+split+sttm", "m2 wait::st", "m2 barrier", "Y ldtm+wait"};
  for (int k = 0; k < 6; ++k) std::printf("    %-18s %6.0f clk\n", fn[k], f[k] / n);
  return 0;
}
