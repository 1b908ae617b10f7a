// kb_sz2_f32_n13_16.cu -- float kron2 kernels for n = 13, 14, 15, 16 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron2_size<float, 13>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 14>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 15>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t kron2_size<float, 16>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
}  // namespace kb
