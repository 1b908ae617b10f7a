// kb_sz3_f64_n14_15.cu -- double kron3 kernels for n = 14, 15 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<double, 14>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 15>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
}  // namespace kb
