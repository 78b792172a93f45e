// Equal-n lattice fit in three fused kernels — see lattice.cuh.
#include "lattice_kernels.cuh"

namespace fmtgp {

constexpr int LAT_TILE_LOG = 13;
constexpr int LAT_MID_SMEM = 200 * 1024;

bool LatGeo::make(int m, int V, int T, int d, LatGeo& g) {
    if (m < 17 || m > 28 || T < 1 || T > 4 || V < 1 || d < 1 || d > MAXD) return false;
    g.m = m;
    g.lt = m - 1;
    // row length: all V class rows of one frequency block in smem, <= 512 threads of 16 elements
    int l2cap = 0;
    while (l2cap < LAT_TILE_LOG && (long long)V << (l2cap + 1) <= (1 << LAT_TILE_LOG) &&
           (long long)V * padded_len(2 << l2cap) * 16 <= LAT_MID_SMEM)
        ++l2cap;
    int l2 = std::min(l2cap, std::max(g.lt - LAT_TILE_LOG, (g.lt + 1) / 2));
    const int l1 = g.lt - l2;
    if (l2 < 8 || l1 < 8 || l2 > 13 || l1 > LAT_TILE_LOG) return false;  // instantiated FFT lengths (lat_inst_*.cu)
    g.l1 = l1;
    g.l2 = l2;
    g.lc = std::min(LAT_TILE_LOG - l1, l2);
    g.nblk_col = (1 << l2) >> g.lc;
    return true;
}

Geo LatGeo::slot_geo() const {
    Geo s{};
    s.m = m;
    s.lt = lt;
    s.two = 1;
    s.l1 = l1;
    s.l2 = l2;
    s.cap = std::max(l1, l2);
    s.C = 1 << (s.cap - l1);
    return s;
}

// yhat in the fused path's row-position order: yperm[t][row][p] = yhat[t][row][ip_freq(p)]
// (once per dataset, fmtgp_model_set_y)
template <int L2>
__global__ void k_lat_perm(const double2* __restrict__ yh, double2* __restrict__ yp, long long total) {
    constexpr int l2 = L2;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long rowbase = e & ~((1ll << l2) - 1);
        yp[e] = yh[rowbase + Ip<L2>::freq(int(e & ((1ll << l2) - 1)))];
    }
}

void lat_perm_yhat(const LatGeo& g, int T, long long half, const void* yhat, void* yperm, cudaStream_t s) {
    const long long total = (long long)T * half;
    const auto* src = static_cast<const double2*>(yhat);
    auto* dst = static_cast<double2*>(yperm);
    switch (g.l2) {
        case 8: k_lat_perm<8><<<148 * 8, 256, 0, s>>>(src, dst, total); break;
        case 9: k_lat_perm<9><<<148 * 8, 256, 0, s>>>(src, dst, total); break;
        case 10: k_lat_perm<10><<<148 * 8, 256, 0, s>>>(src, dst, total); break;
        case 11: k_lat_perm<11><<<148 * 8, 256, 0, s>>>(src, dst, total); break;
        case 12: k_lat_perm<12><<<148 * 8, 256, 0, s>>>(src, dst, total); break;
        default: k_lat_perm<13><<<148 * 8, 256, 0, s>>>(src, dst, total); break;
    }
}

// ------------------------------------------------------------------ dispatch (lat_inst_<L>.cu)
#define FMTGP_LAT_EXTERN(L)                                                                        \
    extern template void lat_cols_launch<L>(const LatGeo&, const LatArgs&, bool, cudaStream_t);  \
    extern template void lat_mid_launch<L>(const LatGeo&, const LatArgs&, cudaStream_t);
FMTGP_LAT_EXTERN(8)
FMTGP_LAT_EXTERN(9)
FMTGP_LAT_EXTERN(10)
FMTGP_LAT_EXTERN(11)
FMTGP_LAT_EXTERN(12)
FMTGP_LAT_EXTERN(13)

static void cols(const LatGeo& g, const LatArgs& a, bool inverse, cudaStream_t s) {
    switch (g.l1) {
        case 8: lat_cols_launch<8>(g, a, inverse, s); break;
        case 9: lat_cols_launch<9>(g, a, inverse, s); break;
        case 10: lat_cols_launch<10>(g, a, inverse, s); break;
        case 11: lat_cols_launch<11>(g, a, inverse, s); break;
        case 12: lat_cols_launch<12>(g, a, inverse, s); break;
        default: lat_cols_launch<13>(g, a, inverse, s); break;
    }
}

static void mid(const LatGeo& g, const LatArgs& a, cudaStream_t s) {
    switch (g.l2) {
        case 8: lat_mid_launch<8>(g, a, s); break;
        case 9: lat_mid_launch<9>(g, a, s); break;
        case 10: lat_mid_launch<10>(g, a, s); break;
        case 11: lat_mid_launch<11>(g, a, s); break;
        case 12: lat_mid_launch<12>(g, a, s); break;
        default: lat_mid_launch<13>(g, a, s); break;
    }
}

void lat_phase(const LatGeo& g, const LatArgs& a, int phase, cudaStream_t s) {
    if (phase == 1) cols(g, a, false, s);
    else if (phase == 2) mid(g, a, s);
    else if (a.want_grad) cols(g, a, true, s);
}

void lat_fit(const LatGeo& g, const LatArgs& a, cudaStream_t s) {
    for (int phase = 1; phase <= 3; ++phase) lat_phase(g, a, phase, s);
}

}  // namespace fmtgp
