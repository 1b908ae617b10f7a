// kb_sz3_f32_n10_11.cu -- float kron3 kernels for n = 10, 11 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<float, 10>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 11>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
}  // namespace kb
