// kb_sz2_f32_n1_8.cu -- float kron2 kernels for n = 1, 2, 3, 4, 5, 6, 7, 8 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron2_size<float, 1>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 2>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 3>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 4>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 5>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 6>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 7>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 8>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
}  // namespace kb
