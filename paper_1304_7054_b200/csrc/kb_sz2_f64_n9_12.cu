// kb_sz2_f64_n9_12.cu -- double kron2 kernels for n = 9, 10, 11, 12 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron2_size<double, 9>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 10>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 11>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 12>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
}  // namespace kb
