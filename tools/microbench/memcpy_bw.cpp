// memcpy_bw.cpp -- host copy bandwidth of the box (development aid for the
// pageable staging pipeline): glibc memcpy vs an AVX-512 non-temporal-store
// copy, T threads, 4 MiB pieces, 2 GiB source -> 2 GiB destination (both
// touched first).  g++ -O3 -march=native -pthread memcpy_bw.cpp -o memcpy_bw
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static void nt_copy(char* d, const char* s, size_t n) {
  size_t i = 0;
  for (; i + 256 <= n; i += 256) {
    __m512i a = _mm512_loadu_si512(s + i), b = _mm512_loadu_si512(s + i + 64);
    __m512i c = _mm512_loadu_si512(s + i + 128), e = _mm512_loadu_si512(s + i + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), a);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 192), e);
  }
  std::memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

int main(int argc, char** argv) {
  const size_t bytes = size_t(2) << 30, piece = size_t(4) << 20;
  char* src = static_cast<char*>(std::aligned_alloc(4096, bytes));
  char* dst = static_cast<char*>(std::aligned_alloc(4096, bytes));
  std::memset(src, 1, bytes);
  std::memset(dst, 2, bytes);
  for (int mode = 0; mode < 2; ++mode)
    for (int T : {1, 2, 4, 8, 12, 16}) {
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        std::atomic<size_t> next{0};
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([&] {
            for (size_t k; (k = next.fetch_add(1)) < bytes / piece;) {
              if (mode == 0)
                std::memcpy(dst + k * piece, src + k * piece, piece);
              else
                nt_copy(dst + k * piece, src + k * piece, piece);
            }
          });
        for (auto& x : th) x.join();
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      }
      std::printf("%-9s threads %2d: %6.1f GB/s copied\n", mode ? "nt-store" : "memcpy", T, bytes / best / 1e9);
    }
  return 0;
}
