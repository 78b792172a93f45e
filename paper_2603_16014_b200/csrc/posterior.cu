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

// grid (query blocks, training chunks): each CTA sums one chunk of the training points for its
// 128 queries into part[chunk][q]; k_post_combine adds the chunks in fixed order (deterministic)
template <bool LAT, int DC>
__global__ void __launch_bounds__(PM_NT) k_post_mean(PostArgs a) {
    __shared__ uint64_t pts[PM_TILE * DC];
    __shared__ double wts[PM_TILE];
    const long long q = blockIdx.x * (long long)PM_NT + threadIdx.x;
    const bool live = q < a.count;
    const int d = a.d;
    double xq[DC], eta[DC];
    uint64_t xb[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) {
        xq[j] = (j < d && live) ? a.X[q * d + j] : 0.0;
        xb[j] = uint64_t(xq[j] * 0x1p53);  // frac_to_bits (ld_sequences.cpp:55-58)
        eta[j] = j < d ? a.eta[j] : 0.0;
    }
    const long long g0 = blockIdx.y * a.chunk, g1 = g0 + a.chunk;
    double acc = 0.0;
    for (int l = 0; l < a.T; ++l) {
        const long long lo = a.off[l] > g0 ? a.off[l] : g0;
        const long long hi = a.off[l] + a.n[l] < g1 ? a.off[l] + a.n[l] : g1;
        if (lo >= hi) continue;
        const double Rtl = a.R[a.task * a.T + l];
        for (long long base = lo; base < hi; base += PM_TILE) {
            __syncthreads();
            const int cnt = int(hi - base < PM_TILE ? hi - base : PM_TILE);
            for (int e = threadIdx.x; e < cnt * d; e += PM_NT) {
                const int r = e / d, j = e - r * d;
                pts[r * DC + j] = point_word(a, l, uint64_t(base + r - a.off[l]), j);
            }
            for (int r = threadIdx.x; r < cnt; r += PM_NT) wts[r] = Rtl * a.c[base + r];
            __syncthreads();
#pragma unroll 2
            for (int r = 0; r < cnt; ++r) {
                double prod = a.gamma;
#pragma unroll
                for (int j = 0; j < DC; ++j)
                    if (j < d) {
                        const uint64_t pw = pts[r * DC + j];
                        const double bv = LAT ? si_free(xq[j], double(pw) * 0x1p-53, a.si_alpha)
                                              : dsi_walsh(xb[j] ^ pw, a.b);
                        prod *= 1.0 + eta[j] * bv;
                    }
                acc = fma(prod, wts[r], acc);
            }
        }
    }
    if (live) a.part[blockIdx.y * a.count + q] = acc;
}

__global__ void k_post_combine(PostArgs a) {
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= a.count) return;
    double s = 0.0;
    for (int k = 0; k < a.nsplit; ++k) s += a.part[k * a.count + q];
    a.out[q] = a.tau + s;
}

void posterior_split(long long count, long long N, int& nsplit, long long& chunk) {
    const long long qblocks = (count + PM_NT - 1) / PM_NT;
    long long want = (4 * 148 + qblocks - 1) / std::max(qblocks, 1ll);
    const long long tiles = (N + PM_TILE - 1) / PM_TILE;
    want = std::max(1ll, std::min(want, tiles));
    chunk = ((tiles + want - 1) / want) * PM_TILE;
    nsplit = int((N + chunk - 1) / chunk);
}

void posterior_mean(const PostArgs& a, cudaStream_t s) {
    const long long blocks = (a.count + PM_NT - 1) / PM_NT;
    if (blocks <= 0) return;
    ProfScope ps("posterior_mean", s);
    const dim3 grid(unsigned(blocks), unsigned(a.nsplit));
    const int dc = a.d <= 4 ? 4 : a.d <= 8 ? 8 : 16;
    if (a.lattice) {
        if (dc == 4) k_post_mean<true, 4><<<grid, PM_NT, 0, s>>>(a);
        else if (dc == 8) k_post_mean<true, 8><<<grid, PM_NT, 0, s>>>(a);
        else k_post_mean<true, 16><<<grid, PM_NT, 0, s>>>(a);
    } else {
        if (dc == 4) k_post_mean<false, 4><<<grid, PM_NT, 0, s>>>(a);
        else if (dc == 8) k_post_mean<false, 8><<<grid, PM_NT, 0, s>>>(a);
        else k_post_mean<false, 16><<<grid, PM_NT, 0, s>>>(a);
    }
    k_post_combine<<<unsigned((a.count + 255) / 256), 256, 0, s>>>(a);
}

}  // namespace fmtgp
