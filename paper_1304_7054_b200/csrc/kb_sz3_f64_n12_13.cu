// kb_sz3_f64_n12_13.cu -- double kron3 kernels for n = 12, 13 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<double, 12>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 13>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
}  // namespace kb
