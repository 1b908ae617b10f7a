// kb_sz3_f64_n10_11.cu -- double kron3 kernels for n = 10, 11 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<double, 10>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 11>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
}  // namespace kb
