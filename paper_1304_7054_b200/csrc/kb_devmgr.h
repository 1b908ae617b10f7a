// kb_devmgr.h -- the device-buffer manager and host worker pools of the
// runtime (the replacement for detail::run_chunked's per-thread scratch and
// OpenMP team, detail.hpp:140-180).
//
//  * Lane: one call's worth of device resources on one GPU -- the library
//    stream, the staged-pipeline streams, pooled device buffers (constants,
//    generic-kernel scratch, X/Y staging) and pinned host bounce buffers for
//    pageable callers. Lanes live in a process-wide per-device pool behind a
//    mutex: a call checks one out for its duration and returns it, so buffers
//    are allocated once and reused (no per-call cudaMalloc),
//    concurrent calls from different host threads get different lanes
//    (concurrent calls on disjoint buffers are allowed), and no
//    resource is tied to a host thread's lifetime.
//  * Asynchronous calls (KB_EXEC_ASYNC) return their lane with an event
//    recorded after the last kernel that reads its buffers; the next user of
//    the lane waits for that event before overwriting them.
//  * TaskPool: persistent host threads that run the per-GPU slices of a
//    sharded call (one task per slice, the caller runs slice 0 and waits:
//    the host barrier). CopyPool: persistent threads that split large
//    pageable <-> pinned memcpys.
//  * Every stream the library creates is a BLOCKING stream, so device work
//    is ordered after anything the caller queued on the legacy default
//    stream (e.g. a torch kernel that produced X).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace kbrt {

struct Fail {
  int code;
  std::string msg;
};

void cuda_check(cudaError_t e, const char* ctx);

constexpr int kSlots = 6;  // staged-pipeline streams / buffer slots per lane (upper bound)

// Growable device allocation (reused across calls).
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes);
  void release();
};

// Growable pinned host allocation (cudaHostAlloc, portable).
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes);
  void release();
};

struct Lane {
  int device = -1;
  int sm_count = 0;
  cudaStream_t stream = nullptr;                // library stream (blocking)
  cudaStream_t slot_stream[kSlots] = {};        // staged pipeline streams (blocking)
  cudaEvent_t done = nullptr;                   // last async use of this lane's buffers
  bool pending = false;                         // `done` recorded, maybe incomplete
  DevBuf consts;
  DevBuf scratch[kSlots];
  DevBuf xs[kSlots], ys[kSlots];                // device staging (host-resident X / Y)
  HostBuf hx[kSlots], hy[kSlots];               // pinned bounce buffers (pageable X / Y)
  DevBuf pk[2][kSlots];                         // tight X / Y for padded square calls (repack path)
  HostBuf hconsts;                              // pinned landing of device-resident constant matrices
  bool used = false;  // this checkout handed a device buffer (constants / scratch) to a kernel
  DevBuf& use(DevBuf& b) {
    used = true;
    return b;
  }
  size_t bytes_held() const;
};

// Check out a lane of `dev` (the caller must have made `dev` current). The
// returned lane's buffers are free to overwrite. `capturing`: the call is
// being captured into a CUDA graph -- no event queries / waits (illegal
// during capture); the graph's own dependencies order its pooled-buffer uses.
Lane* acquire_lane(int dev, bool capturing = false);
// Return a lane. If `async_stream` is non-null and the call handed one of the
// lane's device buffers to a kernel (Lane::use), that kernel may still be
// reading it: an event is recorded on the stream first, and the lane is only
// handed out again once the event has completed. (The square fast paths take
// their constants as kernel parameters and use no lane buffer, so their
// asynchronous calls return the lane immediately reusable.)
void release_lane(Lane* l, cudaStream_t async_stream);

// RAII checkout.
struct LaneLease {
  Lane* lane;
  cudaStream_t async_stream = nullptr;
  explicit LaneLease(int dev, bool capturing = false) : lane(acquire_lane(dev, capturing)) {}
  ~LaneLease() { release_lane(lane, async_stream); }
  LaneLease(const LaneLease&) = delete;
  LaneLease& operator=(const LaneLease&) = delete;
};

// Tile counter (2 x u64, zero between kernels) of dynamically scheduled kernels
// launched on `stream` of `dev`: kernels on one stream run one after another,
// and each one's last CTA rewinds the counter, so one counter per stream is
// safe and no per-call fencing is needed. Allocated on first use (never
// freed); nullptr if that first use is inside a CUDA-graph capture (the
// kernel then schedules statically).
unsigned long long* stream_counter(int dev, cudaStream_t stream, bool capturing);

// Free every idle lane (all devices). Lanes checked out right now are kept.
void release_all_lanes();
// Device bytes held by pooled lanes of `dev` (-1: all devices), for tests.
size_t pooled_device_bytes(int dev);
// Lanes created so far for `dev` (-1: all), for tests.
int lane_count(int dev);

// Run fn(i) for i in [0, n): i = 0 on the calling thread, the rest on
// persistent pool threads; returns when all are done (host barrier).
// Exceptions are captured per task; the first failing task's Fail is thrown.
void parallel_tasks(int n, const std::function<void(int)>& fn);

// memcpy of several (dst, src, bytes) jobs, split into pieces over the copy
// pool and the calling thread; returns when all bytes are copied.
struct CopyJob {
  void* dst;
  const void* src;
  size_t bytes;
};
void parallel_copy(const CopyJob* jobs, int njobs);
int copy_threads();

// Pipeline shape (env overrides for sweeps): chunks in flight, bytes of X+Y
// per chunk.
int stage_slots();
long long stage_bytes();

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

}  // namespace kbrt
