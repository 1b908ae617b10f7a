// kb_sz2_f32_n9_12.cu -- float kron2 kernels for n = 9, 10, 11, 12 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron2_size<float, 9>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 10>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 11>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 12>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
}  // namespace kb
