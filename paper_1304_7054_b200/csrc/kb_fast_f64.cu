// kb_fast_f64.cu -- double instantiations of the square n <= 16 kron kernels
// (split per element type to keep nvcc compile units parallel).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t launch_kron2_fast<double>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t launch_kron3_fast<double>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                              cudaStream_t);
}  // namespace kb
