// kb_sz2_f64_n13_16.cu -- double kron2 kernels for n = 13, 14, 15, 16 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron2_size<double, 13>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 14>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 15>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 16>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
}  // namespace kb
