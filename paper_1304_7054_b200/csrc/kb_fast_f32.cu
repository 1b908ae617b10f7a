// kb_fast_f32.cu -- float instantiations of the square n <= 16 kron kernels
// (split per element type to keep nvcc compile units parallel).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t launch_kron2_fast<float>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
template cudaError_t launch_kron3_fast<float>(const Kron3Params<float>&, const float*, const float*, const float*, int,
                                              cudaStream_t);
}  // namespace kb
