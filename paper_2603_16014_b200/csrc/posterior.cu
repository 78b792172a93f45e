// Posterior mean at query points: tau_t + sum_l R_tl sum_i Q(x, x_{l,i}) c_{l,i}
// (posterior_mean_batch / kernel_against_data, /root/reference/proj/src/gp_core.cpp:386-421).
// Direct O(Q N d) sum like the reference, tiled: each CTA regenerates a tile of design
// points (never stored in HBM) into shared memory and every thread owns one query.
#include "kernels.cuh"
#include "posterior.cuh"

namespace fmtgp {

// SI kernel with a free (non-lattice) argument, bit-for-bit the reference's floating path:
// diff = x - x'; u = min(diff - floor(diff), -diff - floor(-diff)) (kernels.cpp:25-41).
__device__ __forceinline__ double si_free(double x, double xp, int alpha) {
    const double diff = x - xp;
    const double u1 = diff - floor(diff);
    const double u2 = -diff - floor(-diff);
    double u = fmin(u1, u2);
    if (u >= 1.0) u = 0.0;
    constexpr double pi2 = 9.869604401089358618834491;
    if (alpha == 1) return 2.0 * pi2 * (u * (u - 1.0) + 1.0 / 6.0);
    const double b4 = ((u - 2.0) * u + 1.0) * u * u - 1.0 / 30.0;
    return -(2.0 / 3.0) * pi2 * pi2 * b4;
}

// design point bits of task l, natural index i (ld_sequences.cpp:31-53 / 64-87)
__device__ __forceinline__ uint64_t point_word(const PostArgs& a, int l, uint64_t i, int j) {
    const uint64_t sh = a.shifts[l * a.d + j];
    if (a.lattice) {
        const uint64_t k = bitrev64(i, a.mgen);
        const uint64_t frac = ((k * a.g[j]) & (a.n_max - 1)) << (DIGITAL_BITS - a.mgen);
        return (frac + sh) & MASK53;
    }
    uint64_t z = sh;
    const uint64_t* c = a.cols + size_t(j) * a.m_cols;
    for (int p = 0; i; ++p, i >>= 1)
        if (i & 1) z ^= c[p];
    return z;
}

constexpr int PM_NT = 128, PM_TILE = 128;

__global__ void __launch_bounds__(PM_NT) k_post_mean(PostArgs a) {
    __shared__ uint64_t pts[PM_TILE * MAXD];
    __shared__ double wts[PM_TILE];
    const long long q = blockIdx.x * (long long)PM_NT + threadIdx.x;
    const bool live = q < a.count;
    double xq[MAXD];
    uint64_t xb[MAXD];
#pragma unroll
    for (int j = 0; j < MAXD; ++j)
        if (j < a.d) {
            xq[j] = live ? a.X[q * a.d + j] : 0.0;
            xb[j] = uint64_t(xq[j] * 0x1p53);  // frac_to_bits (ld_sequences.cpp:55-58)
        }
    double acc = 0.0;
    for (int l = 0; l < a.T; ++l) {
        const double Rtl = a.R[a.task * a.T + l];
        const long long nl = a.n[l];
        const double* cl = a.c + a.off[l];
        for (long long base = 0; base < nl; base += PM_TILE) {
            __syncthreads();
            for (int e = threadIdx.x; e < PM_TILE * a.d; e += PM_NT) {
                const int r = e / a.d, j = e - r * a.d;
                if (base + r < nl) pts[r * MAXD + j] = point_word(a, l, base + r, j);
            }
            for (int r = threadIdx.x; r < PM_TILE; r += PM_NT) wts[r] = base + r < nl ? Rtl * cl[base + r] : 0.0;
            __syncthreads();
            const int cnt = int(nl - base < PM_TILE ? nl - base : PM_TILE);
            for (int r = 0; r < cnt; ++r) {
                double prod = a.gamma;
#pragma unroll
                for (int j = 0; j < MAXD; ++j)
                    if (j < a.d) {
                        const uint64_t pw = pts[r * MAXD + j];
                        const double base_v = a.lattice ? si_free(xq[j], double(pw) * 0x1p-53, a.si_alpha)
                                                        : dsi_walsh(xb[j] ^ pw, a.b);
                        prod *= 1.0 + a.eta[j] * base_v;
                    }
                acc = fma(prod, wts[r], acc);
            }
        }
    }
    if (live) a.out[q] = a.tau + acc;
}

void posterior_mean(const PostArgs& a, cudaStream_t s) {
    const long long blocks = (a.count + PM_NT - 1) / PM_NT;
    ProfScope ps("posterior_mean", s);
    if (blocks > 0) k_post_mean<<<unsigned(blocks), PM_NT, 0, s>>>(a);
}

}  // namespace fmtgp
