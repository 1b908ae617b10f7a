// kb_sz2_f64_n1_8.cu -- double kron2 kernels for n = 1, 2, 3, 4, 5, 6, 7, 8 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron2_size<double, 1>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 2>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 3>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 4>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 5>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 6>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 7>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
template cudaError_t kron2_size<double, 8>(const Kron2Params<double>&, const double*, const double*, int, cudaStream_t);
}  // namespace kb
