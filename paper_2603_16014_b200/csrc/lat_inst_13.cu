// Fused lattice kernels for FFT length 2^13 (see lattice_kernels.cuh).
#include "lattice_kernels.cuh"

namespace fmtgp {
template void lat_cols_launch<13>(const LatGeo&, const LatArgs&, bool, cudaStream_t);
template void lat_mid_launch<13>(const LatGeo&, const LatArgs&, cudaStream_t);
}  // namespace fmtgp
