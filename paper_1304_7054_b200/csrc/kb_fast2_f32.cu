// kb_fast2_f32.cu -- float instantiations of the square n <= 16 kron2 kernels
// (one compile unit per rank x element type so nvcc runs them in parallel).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t launch_kron2_fast<float>(const Kron2Params<float>&, const float*, const float*, int, cudaStream_t);
}  // namespace kb
