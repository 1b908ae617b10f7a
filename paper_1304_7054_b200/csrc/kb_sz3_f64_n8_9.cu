// kb_sz3_f64_n8_9.cu -- double kron3 kernels for n = 8, 9 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<double, 8>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 9>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
}  // namespace kb
