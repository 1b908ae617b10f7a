// kb_fast2_f64.cu -- double instantiations of the square n <= 16 kron2 kernels
// (one compile unit per rank x element type so nvcc runs them in parallel).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t launch_kron2_fast<double>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
}  // namespace kb
