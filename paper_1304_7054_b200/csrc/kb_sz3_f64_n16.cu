// kb_sz3_f64_n16.cu -- double kron3 kernels for n = 16 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<double, 16>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
}  // namespace kb
