// kronbench -- the reference's `bench` CLI (proj/tools/bench_main.cpp:22-42,
// bench_support.cpp) on the B200 library, through the unchanged drop-in C++
// API (include/kronbatch/kronbatch.hpp). Same flags, same generator, same
// verification protocol (warm-up run checked on min(batch, 16) sampled entries
// against a double-precision direct evaluation, rel_err_inf <= 1e-5 / 1e-12),
// same median-of-reps timing and the same CSV schema
//   size,precision,dims,batch,seconds,gflops,verified
// (so the reference's acceptance criterion 6 accepts it as KRONBATCH_BENCH),
// optionally followed by B200 columns (--b200-columns):
//   gbs,hbm_frac,roof_frac,mode
// Extra flags (not in the reference):
//   --b200-columns   append gbs,hbm_frac,roof_frac,mode to the CSV
//   --mb-per-size M  batch per size = ceil(M MiB / entry bytes of X) instead of --batch
//   --resident       X/Y live in device memory, timed with CUDA events on the
//                    library stream (kernel throughput); default is the
//                    reference's host-buffer call (end to end, PCIe staged)
//   --gpus N         shard host-resident batches over GPUs 0..N-1
//   --hbm-gbs G      roofline denominator (default: MEASURED_PEAKS.json value
//                    passed by the caller, else 6539.9)
// Build: make kronbench  (tools/kronbench/kronbench)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <kronbatch/kronbatch.hpp>

using kronbatch::index_t;

namespace {

enum class Prec { Single, Double };
enum class Dims { D2, D3 };
const char* name(Prec p) { return p == Prec::Single ? "single" : "double"; }
const char* name(Dims d) { return d == Dims::D2 ? "2d" : "3d"; }

struct Config {
  std::vector<int> sizes;
  bool single = true, dbl = true, d2 = true, d3 = true;
  index_t batch = 0;  // 0: 100000 single / 50000 double (bench_support.hpp:22-23)
  int reps = 10;
  double alpha = 1, beta = 0;
  std::uint64_t seed = 1;
  bool csv = false, verify_only = false, resident = false, b200_cols = false;
  int gpus = 1;
  long long bytes_per_size = 0;
  double hbm_gbs = 6539.9;
  std::string out_path;
};

struct Record {
  int size;
  Prec prec;
  Dims dims;
  index_t batch;
  double seconds, gflops, gbs;
  bool verified;
};

std::int64_t flops_kron(int m, Dims d) {  // bench_support.cpp:31-35
  const std::int64_t mm = m;
  return d == Dims::D2 ? 4 * mm * mm * mm : 6 * mm * mm * mm * mm;
}

// --sizes grammar of bench_main.cpp:24: comma-separated items, each a size
// "k" or an inclusive range "lo..hi", sizes >= 1.
std::vector<int> parse_sizes(const std::string& spec) {
  const std::string bad = "bad --sizes value '" + spec + "': expected \"lo..hi\" or a comma list";
  auto number = [&](const std::string& t) -> int {
    if (t.empty() || t.size() > 9 || t.find_first_not_of("0123456789") != std::string::npos)
      throw std::invalid_argument(bad);
    const int v = std::atoi(t.c_str());
    if (v < 1) throw std::invalid_argument(bad);
    return v;
  };
  std::vector<int> sizes;
  std::size_t start = 0;
  for (;;) {
    const std::size_t comma = spec.find(',', start);
    const std::string item = spec.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
    const std::size_t r = item.find("..");
    const int lo = number(r == std::string::npos ? item : item.substr(0, r));
    const int hi = r == std::string::npos ? lo : number(item.substr(r + 2));
    if (hi < lo) throw std::invalid_argument(bad);
    for (int v = lo; v <= hi; ++v) sizes.push_back(v);
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  return sizes;
}

double next_uniform(std::mt19937_64& g) {  // bench_support.hpp:82-84
  return static_cast<double>(g() >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

template <typename T>
struct Data {  // generate_batch (bench_support.hpp:148-170)
  int m;
  Dims dims;
  index_t batch, entry;
  std::vector<T> a, b, c, x, y;
  Data(std::uint64_t seed, int m_, Dims d, index_t batch_) : m(m_), dims(d), batch(batch_) {
    entry = d == Dims::D2 ? (index_t)m * m : (index_t)m * m * m;
    const std::size_t mm = (std::size_t)m * m, be = (std::size_t)entry * batch;
    a.resize(mm);
    b.resize(mm);
    if (d == Dims::D3) c.resize(mm);
    x.resize(be);
    y.resize(be);
    std::mt19937_64 g(seed + (std::uint64_t)m * 1000003u + (d == Dims::D3 ? 0x9e3779b97f4a7c15ull : 0));
    for (auto* v : {&a, &b, &c, &x, &y})
      for (T& e : *v) e = static_cast<T>(next_uniform(g));
  }
};

// Entries checked after the warm-up run: all of them up to 16, else 16
// entries evenly spread over the batch, always including the first and the
// LAST entry (the one whose offsets are largest: index-width bugs show there).
std::vector<index_t> sample_entries(index_t batch) {
  constexpr index_t kSample = 16;
  std::vector<index_t> out;
  if (batch <= kSample) {
    for (index_t i = 0; i < batch; ++i) out.push_back(i);
    return out;
  }
  for (index_t k = 0; k < kSample; ++k) out.push_back(k * (batch - 1) / (kSample - 1));
  return out;
}

// Direct double evaluation of one entry (the math of ref_kron2_apply /
// ref_kron3_apply: (B (x) A) vec X, (C (x) B (x) A) vec X), then alpha/beta.
template <typename T>
double entry_rel_err(const Data<T>& d, index_t p, const std::vector<double>& prior, const T* got, double alpha,
                     double beta) {
  const int m = d.m;
  const T* x = d.x.data() + p * d.entry;
  std::vector<double> want((std::size_t)d.entry, 0.0);
  if (d.dims == Dims::D2) {
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) {
        double s = 0;
        for (int mm = 0; mm < m; ++mm)
          for (int l = 0; l < m; ++l) s += (double)d.a[i + l * m] * (double)d.b[j + mm * m] * (double)x[l + mm * m];
        want[i + (std::size_t)j * m] = s;
      }
  } else {
    // stage the contraction in double (exact enough: reference is O(m^6) direct)
    std::vector<double> t1((std::size_t)d.entry), t2((std::size_t)d.entry);
    for (int n = 0; n < m; ++n)
      for (int mm = 0; mm < m; ++mm)
        for (int i = 0; i < m; ++i) {
          double s = 0;
          for (int l = 0; l < m; ++l) s += (double)d.a[i + l * m] * (double)x[l + mm * m + n * m * m];
          t1[i + mm * m + (std::size_t)n * m * m] = s;
        }
    for (int n = 0; n < m; ++n)
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
          double s = 0;
          for (int mm = 0; mm < m; ++mm) s += t1[i + mm * m + (std::size_t)n * m * m] * (double)d.b[j + mm * m];
          t2[i + j * m + (std::size_t)n * m * m] = s;
        }
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
          double s = 0;
          for (int n = 0; n < m; ++n) s += t2[i + j * m + (std::size_t)n * m * m] * (double)d.c[k + n * m];
          want[i + j * m + (std::size_t)k * m * m] = s;
        }
  }
  double scale = 1, err = 0;
  for (index_t i = 0; i < d.entry; ++i) {
    want[i] = alpha * want[i] + (beta == 0 ? 0.0 : beta * prior[i]);
    scale = std::max(scale, std::abs(want[i]));
  }
  for (index_t i = 0; i < d.entry; ++i) err = std::max(err, std::abs((double)got[i] - want[i]));
  return err / scale;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// median of the rep times (mean of the two middle ones for an even count)
double median(std::vector<double> v) {
  const std::size_t h = v.size() / 2;
  std::nth_element(v.begin(), v.begin() + (long)h, v.end());
  if (v.size() % 2) return v[h];
  const double upper = v[h];
  return 0.5 * (upper + *std::max_element(v.begin(), v.begin() + (long)h));
}

template <typename T>
Record run_one(const Config& cfg, int m, Dims dims, index_t batch, std::ostream& out) {
  using namespace kronbatch;
  Data<T> d(cfg.seed, m, dims, batch);
  const Prec prec = sizeof(T) == 4 ? Prec::Single : Prec::Double;
  const index_t e = d.entry;
  KronProblem2D<T> p2;
  KronProblem3D<T> p3;
  p2.m_a = p2.n_a = p2.m_b = p2.n_b = m;
  p3.m_a = p3.n_a = p3.m_b = p3.n_b = p3.m_c = p3.n_c = m;
  p2.alpha = p3.alpha = static_cast<T>(cfg.alpha);
  p2.beta = p3.beta = static_cast<T>(cfg.beta);

  // buffers the calls see: the host vectors, or device copies (--resident)
  T *X = d.x.data(), *Y = d.y.data();
  T *dX = nullptr, *dY = nullptr;
  const std::size_t bytes = sizeof(T) * (std::size_t)e * batch;
  cudaStream_t stream = nullptr;
  if (cfg.resident) {
    cuda_ok(cudaMalloc(&dX, std::max<std::size_t>(bytes, 16)), "cudaMalloc X");
    cuda_ok(cudaMalloc(&dY, std::max<std::size_t>(bytes, 16)), "cudaMalloc Y");
    cuda_ok(cudaMemcpy(dX, d.x.data(), bytes, cudaMemcpyHostToDevice), "upload X");
    cuda_ok(cudaMemcpy(dY, d.y.data(), bytes, cudaMemcpyHostToDevice), "upload Y");
    cuda_ok(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    X = dX;
    Y = dY;
  }
  b200::ExecConfig ec;
  if (cfg.gpus > 1 && !cfg.resident)
    for (int g = 0; g < cfg.gpus; ++g) ec.devices.push_back(g);
  ec.stream = stream;
  b200::ExecScope scope(ec);
  const index_t len = e * batch;
  auto invoke = [&] {
    if (dims == Dims::D2) {
      kron2<T>(p2, MatrixView<const T>(d.a.data(), m, m, m, m * m), MatrixView<const T>(d.b.data(), m, m, m, m * m),
               BatchView<MatrixView<const T>>(MatrixView<const T>(X, m, m, m, len), batch, e),
               BatchView<MatrixView<T>>(MatrixView<T>(Y, m, m, m, len), batch, e));
    } else {
      kron3<T>(p3, MatrixView<const T>(d.a.data(), m, m, m, m * m), MatrixView<const T>(d.b.data(), m, m, m, m * m),
               MatrixView<const T>(d.c.data(), m, m, m, m * m),
               BatchView<Array3View<const T>>(Array3View<const T>(X, m, m, m, m, m * m, len), batch, e),
               BatchView<Array3View<T>>(Array3View<T>(Y, m, m, m, m, m * m, len), batch, e),
               Workspace<T>(nullptr, kron3_workspace_size(p3, batch)));
    }
  };

  // priors of the sampled entries, warm-up = the verified run
  const std::vector<index_t> sample = sample_entries(batch);
  std::vector<std::vector<double>> priors;
  for (index_t p : sample) priors.emplace_back(d.y.begin() + p * e, d.y.begin() + (p + 1) * e);
  invoke();
  std::vector<T> yhost;
  const T* ygot = d.y.data();
  if (cfg.resident) {
    yhost.resize((std::size_t)e * batch);
    cuda_ok(cudaMemcpy(yhost.data(), dY, bytes, cudaMemcpyDeviceToHost), "download Y");
    ygot = yhost.data();
  }
  double max_rel = 0;
  const double tol = sizeof(T) == 4 ? 1e-5 : 1e-12;
  for (std::size_t s = 0; s < sample.size(); ++s) {
    const double r = entry_rel_err(d, sample[s], priors[s], ygot + sample[s] * e, cfg.alpha, cfg.beta);
    max_rel = std::max(max_rel, r);
    if (!(r <= tol))
      throw std::runtime_error("verification failed: size " + std::to_string(m) + " " + name(prec) + " " +
                               name(dims) + " batch " + std::to_string(batch) + " entry " +
                               std::to_string(sample[s]) + ": max rel err " + std::to_string(r));
  }
  Record rec{m, prec, dims, batch, 0, 0, 0, true};
  if (cfg.verify_only) {
    out << "size " << m << " " << name(prec) << " " << name(dims) << " batch " << batch << ": verified, "
        << sample.size() << " entries, max rel err " << max_rel << "\n";
  } else {
    std::vector<double> times((std::size_t)cfg.reps);
    if (cfg.resident) {
      b200::ExecConfig ea = ec;
      ea.asynchronous = true;
      b200::ExecScope as(ea);
      cudaEvent_t e0, e1;
      cuda_ok(cudaEventCreate(&e0), "event");
      cuda_ok(cudaEventCreate(&e1), "event");
      for (double& t : times) {
        cuda_ok(cudaEventRecord(e0, stream), "record");
        invoke();
        cuda_ok(cudaEventRecord(e1, stream), "record");
        cuda_ok(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        cuda_ok(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        t = ms * 1e-3;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    } else {
      for (double& t : times) {
        const auto t0 = std::chrono::steady_clock::now();
        invoke();
        t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
    rec.seconds = median(times);
    rec.gflops = (double)flops_kron(m, dims) * (double)batch / (rec.seconds * 1e9);
    const double moved = (double)sizeof(T) * (double)e * (double)batch * (cfg.beta == 0 ? 2.0 : 3.0);
    rec.gbs = moved / (rec.seconds * 1e9);
  }
  if (cfg.resident) {
    cudaFree(dX);
    cudaFree(dY);
    cudaStreamDestroy(stream);
  }
  return rec;
}

std::string fmt6(double v) {  // 6 significant digits, like printf %g
  std::ostringstream o;
  o << std::setprecision(6) << v;
  return o.str();
}

void usage() {
  std::cerr << "usage: kronbench [--sizes lo..hi|a,b,...] [--precision single|double|both] [--dims 2d|3d|both]\n"
               "                 [--batch N] [--reps R] [--alpha A] [--beta B] [--seed S] [--format table|csv]\n"
               "                 [--out FILE] [--verify-only] [--resident] [--gpus N] [--hbm-gbs G] [--b200-columns]\n"
               "                 [--mb-per-size M]\n";
}

}  // namespace

int main(int argc, char** argv) {
  Config cfg;
  std::string sizes = "1..16", precision = "both", dims = "both", format = "table";
  try {
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw std::invalid_argument(a + " needs a value");
        return argv[++i];
      };
      if (a == "--sizes") sizes = val();
      else if (a == "--precision") precision = val();
      else if (a == "--dims") dims = val();
      else if (a == "--batch") cfg.batch = std::stoll(val());
      else if (a == "--reps") cfg.reps = std::stoi(val());
      else if (a == "--alpha") cfg.alpha = std::stod(val());
      else if (a == "--beta") cfg.beta = std::stod(val());
      else if (a == "--seed") cfg.seed = std::stoull(val());
      else if (a == "--format") format = val();
      else if (a == "--out") cfg.out_path = val();
      else if (a == "--verify-only") cfg.verify_only = true;
      else if (a == "--resident") cfg.resident = true;
      else if (a == "--b200-columns") cfg.b200_cols = true;
      else if (a == "--mb-per-size") cfg.bytes_per_size = std::stoll(val()) << 20;
      else if (a == "--gpus") cfg.gpus = std::stoi(val());
      else if (a == "--hbm-gbs") cfg.hbm_gbs = std::stod(val());
      else if (a == "-h" || a == "--help") {
        usage();
        return 0;
      } else {
        throw std::invalid_argument("unknown option " + a);
      }
    }
    if (precision != "single" && precision != "double" && precision != "both")
      throw std::invalid_argument("--precision: single|double|both");
    if (dims != "2d" && dims != "3d" && dims != "both") throw std::invalid_argument("--dims: 2d|3d|both");
    if (format != "table" && format != "csv") throw std::invalid_argument("--format: table|csv");
    if (cfg.reps < 1 || cfg.batch < 0 || cfg.gpus < 1) throw std::invalid_argument("reps/batch/gpus must be positive");
    cfg.sizes = parse_sizes(sizes);
    std::sort(cfg.sizes.begin(), cfg.sizes.end());
    cfg.sizes.erase(std::unique(cfg.sizes.begin(), cfg.sizes.end()), cfg.sizes.end());
    cfg.single = precision != "double";
    cfg.dbl = precision != "single";
    cfg.d2 = dims != "3d";
    cfg.d3 = dims != "2d";
    cfg.csv = format == "csv";

    std::ofstream file;
    if (!cfg.out_path.empty()) {
      file.open(cfg.out_path);
      if (!file) throw std::runtime_error("cannot open output file " + cfg.out_path);
    }
    std::ostream& out = cfg.out_path.empty() ? std::cout : file;
    std::vector<Record> recs;
    for (int m : cfg.sizes)
      for (Prec p : {Prec::Single, Prec::Double}) {
        if ((p == Prec::Single && !cfg.single) || (p == Prec::Double && !cfg.dbl)) continue;
        for (Dims dd : {Dims::D2, Dims::D3}) {
          if ((dd == Dims::D2 && !cfg.d2) || (dd == Dims::D3 && !cfg.d3)) continue;
          index_t batch = cfg.batch > 0 ? cfg.batch : (p == Prec::Single ? 100000 : 50000);
          if (cfg.bytes_per_size > 0) {  // batch sized so X alone is bytes_per_size (BASELINE configs[4] sweep)
            const index_t entry = (dd == Dims::D2 ? (index_t)m * m : (index_t)m * m * m) * (p == Prec::Single ? 4 : 8);
            batch = (cfg.bytes_per_size + entry - 1) / entry;
          }
          recs.push_back(p == Prec::Single ? run_one<float>(cfg, m, dd, batch, out)
                                           : run_one<double>(cfg, m, dd, batch, out));
        }
      }
    if (cfg.verify_only) return 0;
    const double fp32 = 72.5, fp64 = 33.6;  // measured FFMA / DFMA peaks (profiles/r01_fma_tput.txt)
    auto roof_frac = [&](const Record& r) {
      const double ai = (double)flops_kron(r.size, r.dims) /
                        ((r.prec == Prec::Single ? 4.0 : 8.0) * 2.0 *
                         std::pow((double)r.size, r.dims == Dims::D2 ? 2 : 3));
      const double roof = std::min(r.prec == Prec::Single ? fp32 * 1e3 : fp64 * 1e3, cfg.hbm_gbs * ai);
      return r.gflops / roof;
    };
    const char* mode = cfg.resident ? "resident" : "host";
    if (cfg.csv) {
      // the reference schema (bench_support.cpp:346-352; acceptance criterion 6
      // checks it verbatim), plus the B200 columns with --b200-columns
      out << "size,precision,dims,batch,seconds,gflops,verified"
          << (cfg.b200_cols ? ",gbs,hbm_frac,roof_frac,mode" : "") << '\n';
      for (const Record& r : recs) {
        out << r.size << ',' << name(r.prec) << ',' << name(r.dims) << ',' << r.batch << ',' << fmt6(r.seconds) << ','
            << fmt6(r.gflops) << ',' << (r.verified ? "true" : "false");
        if (cfg.b200_cols)
          out << ',' << fmt6(r.gbs) << ',' << fmt6(r.gbs / cfg.hbm_gbs) << ',' << fmt6(roof_frac(r)) << ',' << mode;
        out << '\n';
      }
    } else {
      out << "batched Kronecker action on B200, GFlop/s (median of " << cfg.reps << " reps, alpha=" << fmt6(cfg.alpha)
          << " beta=" << fmt6(cfg.beta) << " seed=" << cfg.seed << ", " << mode << " buffers)\n\n";
      char buf[96];
      std::snprintf(buf, sizeof buf, "%5s", "size");
      out << buf;
      std::vector<std::pair<Prec, Dims>> cols;
      for (Prec p : {Prec::Single, Prec::Double})
        for (Dims dd : {Dims::D2, Dims::D3})
          if (((p == Prec::Single && cfg.single) || (p == Prec::Double && cfg.dbl)) &&
              ((dd == Dims::D2 && cfg.d2) || (dd == Dims::D3 && cfg.d3))) {
            cols.emplace_back(p, dd);
            std::snprintf(buf, sizeof buf, "  %10s %5s", (std::string(name(p)) + "-" + name(dd)).c_str(), "roof");
            out << buf;
          }
      out << "\n";
      for (int m : cfg.sizes) {
        std::snprintf(buf, sizeof buf, "%5d", m);
        out << buf;
        for (auto [p, dd] : cols)
          for (const Record& r : recs)
            if (r.size == m && r.prec == p && r.dims == dd) {
              std::snprintf(buf, sizeof buf, "  %10.1f %4.0f%%", r.gflops, 100 * roof_frac(r));
              out << buf;
            }
        out << "\n";
      }
    }
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
