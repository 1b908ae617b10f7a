// tests/cpp/test_dropin.cpp -- the drop-in C++ API (include/kronbatch) used
// exactly as reference code uses it (std::vector host buffers, views, the
// KronProblem structs, exceptions), running on the B200 library. Exit status
// 0 = all checks passed. Run by tests/test_gpu_cpp.py (-m gpu).
#include <cmath>
#include <cstring>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <kronbatch/b200_parts.hpp>
#include <kronbatch/kronbatch.hpp>

using namespace kronbatch;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      ++failures;                                                     \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                 \
  } while (0)

template <typename T>
std::vector<T> rnd(std::size_t n, std::mt19937_64& g) {
  std::vector<T> v(n);
  for (auto& e : v) e = static_cast<T>(static_cast<double>(g() >> 11) * (2.0 / 9007199254740992.0) - 1.0);
  return v;
}

// double brute force Y(i,j) = sum_m sum_l A(i,l) X(l,m) B(j,m) (tight, no ops)
static double err2(const std::vector<double>& a, const std::vector<double>& b, const double* x, const float* y,
                   int m) {
  double e = 0, s = 1;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) {
      double acc = 0;
      for (int mm = 0; mm < m; ++mm)
        for (int l = 0; l < m; ++l) acc += a[i + l * m] * x[l + mm * m] * b[j + mm * m];
      e = std::max(e, std::abs(acc - y[i + j * m]));
      s = std::max(s, std::abs(acc));
    }
  return e / s;
}

template <typename T>
void test_kron2(int m, int batch) {
  std::mt19937_64 g(1234 + m);
  auto a = rnd<T>(m * m, g), b = rnd<T>(m * m, g), x = rnd<T>(m * m * batch, g);
  std::vector<T> y(m * m * batch, T(std::nan("")));
  KronProblem2D<T> pr;
  pr.m_a = pr.n_a = pr.m_b = pr.n_b = m;
  kron2<T>(pr, MatrixView<const T>(std::span<const T>(a), m, m, m), MatrixView<const T>(std::span<const T>(b), m, m, m),
           BatchView<MatrixView<const T>>(MatrixView<const T>(std::span<const T>(x), m, m, m), batch, m * m),
           BatchView<MatrixView<T>>(MatrixView<T>(std::span<T>(y), m, m, m), batch, m * m));
  std::vector<double> ad(a.begin(), a.end()), bd(b.begin(), b.end());
  const double tol = std::is_same_v<T, float> ? 1e-5 : 1e-12;
  for (int p = 0; p < batch; p += std::max(1, batch / 7)) {
    std::vector<double> xd(x.begin() + p * m * m, x.begin() + (p + 1) * m * m);
    std::vector<float> yf(y.begin() + p * m * m, y.begin() + (p + 1) * m * m);
    if constexpr (std::is_same_v<T, float>) CHECK(err2(ad, bd, xd.data(), yf.data(), m) < tol);
    else {
      // double: compare in double directly
      double e = 0, s = 1;
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
          double acc = 0;
          for (int mm = 0; mm < m; ++mm)
            for (int l = 0; l < m; ++l) acc += ad[i + l * m] * xd[l + mm * m] * bd[j + mm * m];
          e = std::max(e, std::abs(acc - y[p * m * m + i + j * m]));
          s = std::max(s, std::abs(acc));
        }
      CHECK(e / s < tol);
    }
  }
}

template <typename T>
void test_kron3_identity_and_workspace(int m, int batch) {
  std::mt19937_64 g(77 + m);
  std::vector<T> id(m * m, T(0));
  for (int i = 0; i < m; ++i) id[i + i * m] = T(1);
  auto x = rnd<T>(m * m * m * batch, g);
  std::vector<T> y(x.size(), T(-1));
  KronProblem3D<T> pr;
  pr.m_a = pr.n_a = pr.m_b = pr.n_b = pr.m_c = pr.n_c = m;
  std::vector<T> work(kron3_workspace_size(pr, batch));
  const MatrixView<const T> I(std::span<const T>(id), m, m, m);
  kron3<T>(pr, I, I, I,
           BatchView<Array3View<const T>>(Array3View<const T>(std::span<const T>(x), m, m, m, m, m * m), batch, m * m * m),
           BatchView<Array3View<T>>(Array3View<T>(std::span<T>(y), m, m, m, m, m * m), batch, m * m * m),
           Workspace<T>(std::span<T>(work)));
  CHECK(y == x);
  // workspace too small: invalid_argument naming the counts (test_kron3.cpp:247-264)
  bool threw = false;
  try {
    kron3<T>(pr, I, I, I,
             BatchView<Array3View<const T>>(Array3View<const T>(std::span<const T>(x), m, m, m, m, m * m), batch,
                                            m * m * m),
             BatchView<Array3View<T>>(Array3View<T>(std::span<T>(y), m, m, m, m, m * m), batch, m * m * m),
             Workspace<T>(work.data(), static_cast<index_t>(work.size()) - 1));
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("kron3: workspace") != std::string::npos;
  }
  CHECK(threw);
}

void test_validation_messages() {
  std::vector<double> a(9), x(27), y(27);
  KronProblem2D<double> pr;
  pr.m_a = pr.n_a = pr.m_b = pr.n_b = 3;
  std::string msg;
  try {
    kron2<double>(pr, MatrixView<const double>(a.data(), 3, 3, 3, 9), MatrixView<const double>(a.data(), 3, 3, 3, 9),
                  BatchView<MatrixView<const double>>(MatrixView<const double>(x.data(), 3, 3, 3, 27), 3, 8),
                  BatchView<MatrixView<double>>(MatrixView<double>(y.data(), 3, 3, 3, 27), 3, 9));
  } catch (const std::invalid_argument& e) {
    msg = e.what();
  }
  CHECK(msg == "kron2: X: batch_stride (8) < (9), batch_stride < entry footprint");
  msg.clear();
  try {
    pr.m_a = 4;
    kron2<double>(pr, MatrixView<const double>(a.data(), 3, 3, 3, 9), MatrixView<const double>(a.data(), 3, 3, 3, 9),
                  BatchView<MatrixView<const double>>(MatrixView<const double>(x.data(), 3, 3, 3, 27), 3, 9),
                  BatchView<MatrixView<double>>(MatrixView<double>(y.data(), 3, 3, 3, 27), 3, 9));
  } catch (const std::invalid_argument& e) {
    msg = e.what();
  }
  CHECK(msg == "kron2: A: op(A) is 3 x 3, expected 4 x 3");
  bool over = false;
  try {
    KronProblem3D<float> p3;
    p3.m_a = p3.m_b = index_t(1) << 32;
    p3.n_c = 4;
    kron3_workspace_size(p3, 1);
  } catch (const std::overflow_error&) {
    over = true;
  }
  CHECK(over);
}

// kron1 (kron1.hpp:17-62) and gemm_a (gemm_a.hpp:18-76) through the drop-in
// headers with std::vector buffers, vs a double brute force.
template <typename T>
void test_kron1_gemm_a(int m, int batch) {
  std::mt19937_64 g(777 + m);
  const int n_a = m + 2;
  auto a = rnd<T>(m * n_a, g), x = rnd<T>(n_a * batch, g), y = rnd<T>(m * batch, g);
  const std::vector<T> y0 = y;
  const T alpha = T(0.5), beta = T(-1.5);
  kron1<T>(MatrixOp::NoTranspose, m, n_a, alpha, MatrixView<const T>(std::span<const T>(a), m, n_a, m),
           BatchView<VectorView<const T>>(VectorView<const T>(std::span<const T>(x), n_a), batch, n_a), beta,
           BatchView<VectorView<T>>(VectorView<T>(std::span<T>(y), m), batch, m));
  const double tol = std::is_same_v<T, float> ? 1e-5 : 1e-12;
  for (int p = 0; p < batch; p += std::max(1, batch / 9))
    for (int i = 0; i < m; ++i) {
      double w = beta * (double)y0[p * m + i];
      for (int l = 0; l < n_a; ++l) w += alpha * (double)a[i + l * m] * (double)x[p * n_a + l];
      CHECK(std::abs(w - (double)y[p * m + i]) <= tol * std::max(1.0, std::abs(w)) * 4);
    }
  // gemm_a, op(A) = A^T: A^p stored k x m
  const int k = m + 1, n = 3;
  auto A = rnd<T>(k * m * batch, g), B = rnd<T>(k * n, g), C = rnd<T>(m * n * batch, g);
  const std::vector<T> C0 = C;
  gemm_a<T>(MatrixOp::Transpose, MatrixOp::NoTranspose, m, n, k, alpha,
            BatchView<MatrixView<const T>>(MatrixView<const T>(std::span<const T>(A), k, m, k), batch, k * m),
            MatrixView<const T>(std::span<const T>(B), k, n, k), beta,
            BatchView<MatrixView<T>>(MatrixView<T>(std::span<T>(C), m, n, m), batch, m * n));
  for (int p = 0; p < batch; p += std::max(1, batch / 9))
    for (int c = 0; c < n; ++c)
      for (int i = 0; i < m; ++i) {
        double w = beta * (double)C0[p * m * n + i + c * m];
        for (int kk = 0; kk < k; ++kk) w += alpha * (double)A[p * k * m + kk + i * k] * (double)B[kk + c * k];
        CHECK(std::abs(w - (double)C[p * m * n + i + c * m]) <= tol * std::max(1.0, std::abs(w)) * 4);
      }
  // reference error text (test_kron1.cpp:209-235)
  bool threw = false;
  try {
    kron1<T>(MatrixOp::NoTranspose, m, n_a + 1, alpha, MatrixView<const T>(std::span<const T>(a), m, n_a, m),
             BatchView<VectorView<const T>>(VectorView<const T>(std::span<const T>(x), n_a), batch, n_a), beta,
             BatchView<VectorView<T>>(VectorView<T>(std::span<T>(y), m), batch, m));
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("kron1: A: op(A) is") == 0;
  }
  CHECK(threw);
}

// kb_?kron2_parts through the C++ wrapper: a host batch split into 3 ragged
// parts (all on device 0 here) == one kron2 over the whole batch, bit for bit.
template <typename T>
void test_parts(int m, int batch) {
  std::mt19937_64 g(99 + m);
  auto a = rnd<T>(m * m, g), b = rnd<T>(m * m, g), x = rnd<T>(m * m * batch, g);
  std::vector<T> y1(m * m * batch, T(0)), y2(m * m * batch, T(0));
  KronProblem2D<T> pr;
  pr.m_a = pr.n_a = pr.m_b = pr.n_b = m;
  const index_t e = (index_t)m * m;
  MatrixView<const T> va(std::span<const T>(a), m, m, m), vb(std::span<const T>(b), m, m, m);
  kron2<T>(pr, va, vb, BatchView<MatrixView<const T>>(MatrixView<const T>(std::span<const T>(x), m, m, m), batch, e),
           BatchView<MatrixView<T>>(MatrixView<T>(std::span<T>(y1), m, m, m), batch, e));
  const int cuts[4] = {0, batch / 3, batch / 3 + 1, batch};
  std::vector<b200::Part2<T>> parts;
  for (int i = 0; i < 3; ++i) {
    const index_t p0 = cuts[i], n = cuts[i + 1] - cuts[i];
    parts.push_back(b200::Part2<T>{
        0, BatchView<MatrixView<const T>>(MatrixView<const T>(std::span<const T>(x).subspan(p0 * e, n * e), m, m, m), n, e),
        BatchView<MatrixView<T>>(MatrixView<T>(std::span<T>(y2).subspan(p0 * e, n * e), m, m, m), n, e), nullptr});
  }
  b200::kron2_parts<T>(pr, va, vb, std::span<const b200::Part2<T>>(parts));
  CHECK(std::memcmp(y1.data(), y2.data(), sizeof(T) * y1.size()) == 0);
}

int main() {
  test_parts<float>(16, 1001);
  test_parts<double>(9, 333);
  for (int m : {1, 5, 16, 24}) {
    test_kron1_gemm_a<float>(m, 500);
    test_kron1_gemm_a<double>(m, 200);
  }
  for (int m : {1, 3, 10, 16}) {
    test_kron2<float>(m, 1000);
    test_kron2<double>(m, 300);
    test_kron3_identity_and_workspace<float>(m, 40);
    test_kron3_identity_and_workspace<double>(m, 20);
  }
  test_validation_messages();
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("test_dropin: all checks passed\n");
  return 0;
}
