// Fused lattice kernels for FFT length 2^10 (see lattice_kernels.cuh).
#include "lattice_kernels.cuh"

namespace fmtgp {
template void lat_cols_launch<10>(const LatGeo&, const LatArgs&, bool, cudaStream_t);
template void lat_mid_launch<10>(const LatGeo&, const LatArgs&, cudaStream_t);
}  // namespace fmtgp
