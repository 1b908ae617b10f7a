// kronbatch/b200.hpp -- glue between the drop-in template API and the C ABI
// of libkronbatch_b200.so (include/kronbatch_b200.h). Not part of the
// reference API; adds an optional per-thread execution scope (GPU set for
// batch sharding, CUDA stream, async) that the unchanged kron2/kron3
// signatures pick up implicitly.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <kronbatch/types.hpp>
#include <kronbatch_b200.h>

namespace kronbatch {
namespace b200 {

/// Per-thread execution settings used by kron2/kron3 calls on this thread.
struct ExecConfig {
  std::vector<std::int32_t> devices;  // >1: shard host-resident batches over these GPUs
  void* stream = nullptr;             // cudaStream_t for device-resident calls
  bool asynchronous = false;          // device buffers only: return before completion
  bool tf32 = false;                  // allow the 3xTF32 tensor-core kron3 (fp32, n = 16), 1e-5 parity
};

inline ExecConfig*& current_exec() {
  thread_local ExecConfig* cfg = nullptr;
  return cfg;
}

/// RAII: `kronbatch::b200::ExecScope s({0,1,2,3});` shards calls in scope.
class ExecScope {
 public:
  explicit ExecScope(ExecConfig cfg) : cfg_(std::move(cfg)), prev_(current_exec()) { current_exec() = &cfg_; }
  ~ExecScope() { current_exec() = prev_; }
  ExecScope(const ExecScope&) = delete;
  ExecScope& operator=(const ExecScope&) = delete;

 private:
  ExecConfig cfg_;
  ExecConfig* prev_;
};

struct ExecC {
  kb_exec e{};
  const kb_exec* ptr = nullptr;
  ExecC() {
    if (ExecConfig* c = current_exec()) {
      e.ndevices = static_cast<std::int32_t>(c->devices.size());
      e.devices = c->devices.empty() ? nullptr : c->devices.data();
      e.stream = c->stream;
      e.flags = (c->asynchronous ? KB_EXEC_ASYNC : 0u) | (c->tf32 ? KB_EXEC_TF32 : 0u);
      ptr = &e;
    }
  }
};

/// Rethrows an ABI status as the exception type the reference uses.
inline void check(int rc, const char* msg) {
  switch (rc) {
    case KB_OK: return;
    case KB_EINVAL: throw std::invalid_argument(msg);
    case KB_EOVERFLOW: throw std::overflow_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline char op_char(MatrixOp op) { return static_cast<char>(op); }

}  // namespace b200
}  // namespace kronbatch
