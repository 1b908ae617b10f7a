// kb_fast3_f32.cu -- float instantiations of the square n <= 16 kron3 kernels
// (one compile unit per rank x element type so nvcc runs them in parallel).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t launch_kron3_fast<float>(const Kron3Params<float>&, const float*, const float*, const float*, int, cudaStream_t);
}  // namespace kb
