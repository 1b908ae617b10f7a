// kb_sizes.h -- per-size launch entry points of the square n <= 16 kernels
// (defined in kb_fast_dispatch.cuh, instantiated in kb_sz*.cu).
#pragma once

#include <cuda_runtime.h>

#include "kb_device.cuh"

namespace kb {

template <typename T, int N>
cudaError_t kron2_size(const Kron2Params<T>& p, const T* ha, const T* hw, int sm_count, cudaStream_t s);
template <typename T, int N>
cudaError_t kron3_size(const Kron3Params<T>& p, const T* ha, const T* hb, const T* hc, int sm_count, cudaStream_t s);

}  // namespace kb
