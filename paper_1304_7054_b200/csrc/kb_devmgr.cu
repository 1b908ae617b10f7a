// kb_devmgr.cu -- device-buffer manager (lane pool) and host worker pools.
// See kb_devmgr.h for the design; this file has no kernels.
#include "kb_devmgr.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <map>
#include <unordered_map>

namespace kbrt {

void copy_stream(void* dst, const void* src, size_t bytes);  // kb_hostcopy.cpp

void cuda_check(cudaError_t e, const char* ctx) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Fail{e == cudaErrorMemoryAllocation ? 4 /*KB_ENOMEM*/ : 3 /*KB_ECUDA*/,
               std::string(ctx) + ": CUDA error: " + cudaGetErrorString(e)};
  }
}

// ------------------------------------------------------------- buffers ----

void* DevBuf::get(size_t bytes) {
  if (bytes <= cap) return p;
  const size_t want = std::max(bytes, cap + cap / 2);  // grow by >= 1.5x
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cuda_check(cudaMalloc(&p, want), "device buffer");
  cap = want;
  return p;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
}

void* HostBuf::get(size_t bytes) {
  if (bytes <= cap) return p;
  const size_t want = std::max(bytes, cap + cap / 2);
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  cuda_check(cudaHostAlloc(&p, want, cudaHostAllocPortable), "pinned bounce buffer");
  cap = want;
  return p;
}

void HostBuf::release() {
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
}

size_t Lane::bytes_held() const {
  size_t b = consts.cap;
  for (int i = 0; i < kSlots; ++i) b += scratch[i].cap + xs[i].cap + ys[i].cap + pk[0][i].cap + pk[1][i].cap;
  return b;
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev);
  if (dev != prev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
}

DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

int stage_slots() {
  static const int v = [] {
    const char* e = std::getenv("KB_STAGE_SLOTS");
    const int n = e ? std::atoi(e) : 3;
    return n < 1 ? 1 : (n > kSlots ? kSlots : n);
  }();
  return v;
}

long long stage_bytes() {
  static const long long v = [] {
    const char* e = std::getenv("KB_STAGE_MB");
    const long long mb = e ? std::atoll(e) : 128;
    return (mb < 1 ? 1 : mb) << 20;
  }();
  return v;
}

// ----------------------------------------------------------- lane pool ----

namespace {

constexpr int kMaxLanesPerDevice = 16;

struct LanePool {
  std::mutex mu;
  std::unordered_map<int, std::vector<Lane*>> idle;
  std::unordered_map<int, int> created;
  std::unordered_map<int, int> sms;
};

LanePool& pool() {
  static LanePool* p = new LanePool;  // never destroyed: lanes may outlive static teardown order
  return *p;
}

Lane* make_lane(int dev, int sm_count) {
  auto* l = new Lane;
  l->device = dev;
  l->sm_count = sm_count;
  try {
    cuda_check(cudaStreamCreateWithFlags(&l->stream, cudaStreamDefault), "stream");
    for (auto& s : l->slot_stream) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamDefault), "stream");
    cuda_check(cudaEventCreateWithFlags(&l->done, cudaEventDisableTiming), "event");
  } catch (...) {
    delete l;
    throw;
  }
  return l;
}

void destroy_lane(Lane* l) {
  DeviceGuard g(l->device);
  if (l->pending) cudaEventSynchronize(l->done);
  cudaStreamSynchronize(l->stream);
  for (auto& s : l->slot_stream) cudaStreamSynchronize(s);
  l->consts.release();
  l->hconsts.release();
  for (int i = 0; i < kSlots; ++i) {
    l->scratch[i].release();
    l->xs[i].release();
    l->ys[i].release();
    l->hx[i].release();
    l->hy[i].release();
    l->pk[0][i].release();
    l->pk[1][i].release();
    cudaStreamDestroy(l->slot_stream[i]);
  }
  cudaStreamDestroy(l->stream);
  cudaEventDestroy(l->done);
  delete l;
}

bool lane_ready(Lane* l) {
  if (!l->pending) return true;
  const cudaError_t q = cudaEventQuery(l->done);
  if (q == cudaErrorNotReady) return false;
  if (q != cudaSuccess) cudaGetLastError();
  l->pending = false;
  return true;
}

}  // namespace

static Lane* acquire_lane_impl(int dev, bool capturing) {
  LanePool& P = pool();
  Lane* wait_for = nullptr;
  int sm_count = 0;
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto& v = P.idle[dev];
    if (capturing && !v.empty()) {  // no cudaEventQuery inside a capture
      Lane* l = v.back();
      v.pop_back();
      l->pending = false;
      return l;
    }
    for (size_t i = v.size(); i-- > 0;) {
      if (lane_ready(v[i])) {
        Lane* l = v[i];
        v.erase(v.begin() + (long)i);
        return l;
      }
    }
    if (!v.empty() && P.created[dev] >= kMaxLanesPerDevice) {
      // every idle lane is still in use by async work: wait for the one released
      // first (its work completes first), so the host stays at most
      // kMaxLanesPerDevice calls ahead of the device instead of draining it
      wait_for = v.front();
      v.erase(v.begin());
    } else {
      auto it = P.sms.find(dev);
      if (it == P.sms.end()) {
        cuda_check(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev), "device query");
        P.sms[dev] = sm_count;
      } else {
        sm_count = it->second;
      }
      ++P.created[dev];
    }
  }
  if (wait_for) {
    cudaEventSynchronize(wait_for->done);
    wait_for->pending = false;
    return wait_for;
  }
  try {
    return make_lane(dev, sm_count);
  } catch (...) {
    std::lock_guard<std::mutex> lk(P.mu);
    --P.created[dev];
    throw;
  }
}

Lane* acquire_lane(int dev, bool capturing) {
  Lane* l = acquire_lane_impl(dev, capturing);
  l->used = false;
  return l;
}

void release_lane(Lane* l, cudaStream_t async_stream) {
  if (!l) return;
  l->pending = false;
  if (async_stream && l->used) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(async_stream, &st) != cudaSuccess) {
      cudaGetLastError();
      st = cudaStreamCaptureStatusNone;
    }
    // Under stream capture the graph owns the ordering (pooled buffers baked
    // into a graph are the caller's responsibility).
    if (st == cudaStreamCaptureStatusNone) {
      if (cudaEventRecord(l->done, async_stream) == cudaSuccess)
        l->pending = true;
      else
        cudaGetLastError();
    }
  }
  LanePool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  P.idle[l->device].push_back(l);
}

unsigned long long* stream_counter(int dev, cudaStream_t stream, bool capturing) {
  static std::mutex mu;
  static auto* counters = new std::map<std::pair<int, cudaStream_t>, unsigned long long*>;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(dev, stream);
  auto it = counters->find(key);
  if (it != counters->end()) return it->second;
  if (capturing) return nullptr;
  unsigned long long* c = nullptr;
  cuda_check(cudaMalloc(&c, 2 * sizeof(unsigned long long)), "tile counter");
  cuda_check(cudaMemset(c, 0, 2 * sizeof(unsigned long long)), "tile counter");
  (*counters)[key] = c;
  return c;
}

void release_all_lanes() {
  LanePool& P = pool();
  std::vector<Lane*> victims;
  {
    std::lock_guard<std::mutex> lk(P.mu);
    for (auto& kv : P.idle) {
      for (Lane* l : kv.second) victims.push_back(l);
      P.created[kv.first] -= (int)kv.second.size();
      kv.second.clear();
    }
  }
  for (Lane* l : victims) destroy_lane(l);
}

size_t pooled_device_bytes(int dev) {
  LanePool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  size_t b = 0;
  for (auto& kv : P.idle)
    if (dev < 0 || kv.first == dev)
      for (Lane* l : kv.second) b += l->bytes_held();
  return b;
}

int lane_count(int dev) {
  LanePool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  int n = 0;
  for (auto& kv : P.created)
    if (dev < 0 || kv.first == dev) n += kv.second;
  return n;
}

// -------------------------------------------------------- thread pools ----

namespace {

class ThreadPool {
 public:
  void post(std::function<void()> fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(fn));
    }
    cv_.notify_one();
  }
  // make sure at least `k` threads are idle-or-spawned for new work
  void ensure(int k) {
    std::lock_guard<std::mutex> lk(mu_);
    const int want = std::min(k + busy_, kMaxThreads);
    while (nthreads_ < want) {
      std::thread(&ThreadPool::loop, this).detach();  // persistent; never joined (process lifetime)
      ++nthreads_;
    }
  }

 private:
  static constexpr int kMaxThreads = 128;
  void loop() {
    for (;;) {
      std::function<void()> fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !q_.empty(); });
        fn = std::move(q_.front());
        q_.pop_front();
        ++busy_;
      }
      fn();
      std::lock_guard<std::mutex> lk(mu_);
      --busy_;
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  int nthreads_ = 0;
  int busy_ = 0;
};

ThreadPool& task_pool() {
  static ThreadPool* p = new ThreadPool;
  return *p;
}
ThreadPool& copy_pool() {
  static ThreadPool* p = new ThreadPool;
  return *p;
}

struct Latch {
  std::mutex mu;
  std::condition_variable cv;
  int left;
  explicit Latch(int n) : left(n) {}
  void arrive() {
    std::lock_guard<std::mutex> lk(mu);
    if (--left == 0) cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return left == 0; });
  }
};

}  // namespace

void parallel_tasks(int n, const std::function<void(int)>& fn) {
  if (n <= 0) return;
  if (n == 1) {
    fn(0);
    return;
  }
  std::vector<Fail> fails((size_t)n, Fail{0, {}});
  auto run = [&](int i) {
    try {
      fn(i);
    } catch (const Fail& f) {
      fails[(size_t)i] = f;
    } catch (const std::exception& e) {
      fails[(size_t)i] = Fail{5 /*KB_EINTERNAL*/, e.what()};
    } catch (...) {
      fails[(size_t)i] = Fail{5, "unknown exception"};
    }
  };
  Latch latch(n - 1);
  ThreadPool& tp = task_pool();
  tp.ensure(n - 1);
  for (int i = 1; i < n; ++i)
    tp.post([&, i] {
      run(i);
      latch.arrive();
    });
  run(0);
  latch.wait();  // host barrier: every slice is done
  for (auto& f : fails)
    if (f.code != 0) throw f;
}

int copy_threads() {
  static const int v = [] {
    const char* e = std::getenv("KB_COPY_THREADS");
    if (e) return std::max(0, std::atoi(e));
    // every host core: the caller copies too, so hw - 1 helpers (B200 box:
    // 16 vCPUs -> 88.6 GB/s of streaming copies, tools/microbench/memcpy_bw.cpp)
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::min<unsigned>(63u, hw > 1 ? hw - 1 : 1u);
  }();
  return v;
}

void parallel_copy(const CopyJob* jobs, int njobs) {
  constexpr size_t kPiece = size_t(4) << 20;
  size_t total = 0;
  for (int j = 0; j < njobs; ++j) total += jobs[j].bytes;
  const int helpers = std::min<int>(copy_threads(), (int)(total / kPiece));
  if (helpers <= 0) {
    for (int j = 0; j < njobs; ++j)
      if (jobs[j].bytes) copy_stream(jobs[j].dst, jobs[j].src, jobs[j].bytes);
    return;
  }
  struct Piece {
    char* d;
    const char* s;
    size_t n;
  };
  auto pieces = std::make_shared<std::vector<Piece>>();
  for (int j = 0; j < njobs; ++j)
    for (size_t off = 0; off < jobs[j].bytes; off += kPiece)
      pieces->push_back(Piece{static_cast<char*>(jobs[j].dst) + off, static_cast<const char*>(jobs[j].src) + off,
                              std::min(kPiece, jobs[j].bytes - off)});
  struct State {
    std::atomic<size_t> next{0};
    Latch done;
    explicit State(int h) : done(h) {}
  };
  auto st = std::make_shared<State>(helpers);
  auto work = [pieces, st] {
    for (size_t i; (i = st->next.fetch_add(1)) < pieces->size();) {
      const Piece& p = (*pieces)[i];
      copy_stream(p.d, p.s, p.n);
    }
  };
  ThreadPool& cp = copy_pool();
  cp.ensure(helpers);
  for (int h = 0; h < helpers; ++h)
    cp.post([work, st] {
      work();
      st->done.arrive();
    });
  work();
  st->done.wait();  // every helper has finished its last piece
}

}  // namespace kbrt
