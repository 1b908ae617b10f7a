// kb_sz3_f32_n16.cu -- float kron3 kernels for n = 16 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<float, 16>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                          cudaStream_t);
}  // namespace kb
