// kb_sz3_f32_n1_7.cu -- float kron3 kernels for n = 1, 2, 3, 4, 5, 6, 7 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<float, 1>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 2>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 3>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 4>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 5>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 6>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<float, 7>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
}  // namespace kb
