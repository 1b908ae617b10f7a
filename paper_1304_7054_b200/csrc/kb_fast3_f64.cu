// kb_fast3_f64.cu -- double instantiations of the square n <= 16 kron3 kernels
// (one compile unit per rank x element type so nvcc runs them in parallel).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t launch_kron3_fast<double>(const Kron3Params<double>&, const double*, const double*, const double*, int, cudaStream_t);
}  // namespace kb
