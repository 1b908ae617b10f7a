// kb_sz3_f64_n1_7.cu -- double kron3 kernels for n = 1, 2, 3, 4, 5, 6, 7 (one compile unit per size group).
#include "kb_fast_dispatch.cuh"

namespace kb {
template cudaError_t kron3_size<double, 1>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 2>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 3>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 4>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 5>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 6>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
template cudaError_t kron3_size<double, 7>(const Kron3Params<double>&, const double*, const double*, const double*, int,
                                          cudaStream_t);
}  // namespace kb
