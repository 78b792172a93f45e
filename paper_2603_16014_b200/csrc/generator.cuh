// Kernel-generator evaluation on the fly (no point sets in HBM).
//
// Restates, for device use:
//   si_bernoulli_1d   /root/reference/proj/src/kernels.cpp:25-41
//   dsi_order_1d      kernels.cpp:43-82   (X3 via a 3x bit spread instead of a set-bit loop)
//   dsi_walsh_1d      kernels.cpp:84-89
//   SpatialKernel()   kernels.cpp:91-103  gamma * prod_j (1 + eta_j * base_j)
//   lattice_points    ld_sequences.cpp:31-53 (exact 53-bit fixed point)
//   digital_net_points ld_sequences.cpp:64-87
//
// Generator column of pair (a, b), a <= b (fast_gram.cpp:76-80): q(i) = Q(x_{a,i}, x_{b,0})
// with x_{b,0} = Delta_b.  Everything about the pair folds into one 53-bit offset per
// dimension: lattice D = ((j g mod n_a) << (53 - m_a)) + (Delta_a - Delta_b) mod 2^53 in
// DFT input order j (fft_bitrev's bit reversal composes with the radical-inverse order,
// SURVEY.md §7 fact 1); digital w = z_i xor (Delta_a xor Delta_b) in natural order.
#pragma once

#include "common.cuh"

namespace fmtgp {

struct Spatial {
    int family;    // 0: SI lattice (Bernoulli), 1: DSI digital (Walsh)
    int d;
    int si_alpha;  // 1 -> B2, 2 -> B4
    int pad_;
    double b[4];   // DSI order weights; zero weights skipped (kernels.cpp:86-87)
};

__device__ __forceinline__ double si_base(uint64_t D, int alpha) {
    D &= MASK53;
    const uint64_t Dn = (uint64_t(1) << 53) - D;
    const uint64_t uu = D < Dn ? D : Dn;  // min(frac(x-x'), frac(x'-x)), kernels.cpp:28-32
    const double u = double(uu) * 0x1p-53;
    constexpr double pi2 = 9.869604401089358618834491;
    if (alpha == 1) return 2.0 * pi2 * (u * (u - 1.0) + 1.0 / 6.0);
    const double b4 = ((u - 2.0) * u + 1.0) * u * u - 1.0 / 30.0;
    return -(2.0 / 3.0) * pi2 * pi2 * b4;
}

__device__ __forceinline__ uint64_t spread3_17(uint64_t x) {
    x &= 0x1FFFFull;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__device__ __forceinline__ double pow2i(int e) {  // exact 2^e for -1022 <= e <= 1023
    return __longlong_as_double((long long)(1023 + e) << 52);
}

// dsi_order_1d(alpha, x, x') with w = bits(x) xor bits(x') (kernels.cpp:43-82).
__device__ __forceinline__ double dsi_order(uint64_t w, int alpha) {
    w &= MASK53;
    if (w == 0) {
        return alpha == 1 ? 1.0 : alpha == 2 ? 1.5 : alpha == 3 ? 25.0 / 18.0 : 407.0 / 294.0;
    }
    const int clz = __clzll((long long)w);
    const int ptop = 63 - clz;  // leading one position
    const int beta = 53 - ptop;  // 1-based index of the first one digit
    const double u = double(w) * 0x1p-53;
    const double t1 = pow2i(-beta);
    const double db = double(beta);
    switch (alpha) {
        case 1:
            return 1.0 - 3.0 * t1;
        case 2:
            return -1.0 - db * u + 2.5 * (1.0 - t1);
        case 3: {
            const double t2 = t1 * t1;
            return -1.0 + db * u * u - 5.0 * (1.0 - t1) * u + (43.0 / 18.0) * (1.0 - t2);
        }
        default: {
            const double t2 = t1 * t1, t3 = t2 * t1;
            // X3(u) = sum over one digits a of 8^-a: the two leading 17-digit windows,
            // spread 3x into integers (exact), cover every term above 2^-102 relative.
            const uint64_t top = w << clz;
            const double x3 = double(spread3_17(top >> 47)) * pow2i(-3 * (69 - ptop)) +
                              double(spread3_17(top >> 30)) * pow2i(-3 * (86 - ptop));
            return -1.0 - (2.0 / 3.0) * db * u * u * u + 5.0 * (1.0 - t1) * u * u -
                   (43.0 / 9.0) * (1.0 - t2) * u + (701.0 / 294.0) * (1.0 - t3) - db * x3 / 3.0;
        }
    }
}

// Order-4 with X3 from an 8-bit table T8[b] = sum_i bit(7-i of b) 8^-i (exact 24-bit values):
// X3 = 2^(-3 beta) (T8[b0] + 2^-24 (T8[b1] + 2^-24 T8[b2])) over the three leading bytes of
// the normalised word — same value as the set-bit loop of kernels.cpp:69-75 to ~1 ulp.
__device__ __forceinline__ double dsi_order4_t8(uint64_t w, const double* __restrict__ T8) {
    w &= MASK53;
    if (w == 0) return 407.0 / 294.0;
    const int clz = __clzll((long long)w);
    const int beta = clz - 10;  // 53 - (63 - clz)
    const double u = double(w) * 0x1p-53;
    const double t1 = pow2i(-beta);
    const double t2 = t1 * t1, t3 = t2 * t1;
    const double db = double(beta);
    const uint64_t top = w << clz;
    const double x3s = fma(fma(T8[(top >> 40) & 255], 0x1p-24, T8[(top >> 48) & 255]), 0x1p-24, T8[top >> 56]);
    const double x3 = x3s * pow2i(-3 * beta);
    return -1.0 - (2.0 / 3.0) * db * u * u * u + 5.0 * (1.0 - t1) * u * u - (43.0 / 9.0) * (1.0 - t2) * u +
           (701.0 / 294.0) * (1.0 - t3) - db * x3 / 3.0;
}

__device__ __forceinline__ double dsi_walsh(uint64_t w, const double* b) {
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
        if (b[a] != 0.0) acc += b[a] * dsi_order(w, a + 1);
    return acc;
}

// Base kernel value of dimension-j coordinate word (D for SI, w for DSI).
__device__ __forceinline__ double base_value(const Spatial& sp, uint64_t word) {
    return sp.family == 0 ? si_base(word, sp.si_alpha) : dsi_walsh(word, sp.b);
}

// Coordinate word of pair element: lattice DFT-order j, digital natural-order i.
struct PointGen {
    int family;
    int m;                      // log2 n_a of the generating task
    const uint64_t* g;          // lattice [d]
    const uint64_t* cols;       // digital [d][m_cols]
    int m_cols;

    __device__ __forceinline__ uint64_t lattice_word(uint64_t j, int dim, uint64_t off) const {
        const uint64_t mask = (uint64_t(1) << m) - 1;
        const uint64_t frac = ((j * __ldg(g + dim)) & mask) << (DIGITAL_BITS - m);
        return (frac + off) & MASK53;
    }
    __device__ __forceinline__ uint64_t digital_z(uint64_t i, int dim) const {
        uint64_t z = 0;
        const uint64_t* c = cols + size_t(dim) * m_cols;
        for (int p = 0; i; ++p, i >>= 1)
            if (i & 1) z ^= __ldg(c + p);
        return z;
    }
};

// q = gamma * prod_j (1 + eta_j * kappa_j), and optionally d q / d eta_j through
// prefix/suffix products (1 + eta kappa can vanish).
template <bool GRAD>
__device__ __forceinline__ double product_kernel(const double* kappa, const double* eta, int d, double gamma,
                                                 double* dq_deta) {
    double f[MAXD];
    double prod = gamma;
#pragma unroll
    for (int j = 0; j < MAXD; ++j)
        if (j < d) {
            f[j] = 1.0 + eta[j] * kappa[j];
            prod *= f[j];
        }
    if (GRAD) {
        double pre = gamma;
#pragma unroll
        for (int j = 0; j < MAXD; ++j)
            if (j < d) {
                dq_deta[j] = pre * kappa[j];
                pre *= f[j];
            }
        double suf = 1.0;
#pragma unroll
        for (int j = MAXD - 1; j >= 0; --j)
            if (j < d) {
                dq_deta[j] *= suf;
                suf *= f[j];
            }
    }
    return prod;
}

// Compile-time-dimension product kernel (register-resident, no MAXD padding).
template <int D, bool GRAD>
__device__ __forceinline__ double product_kernel_d(const double* kappa, const double* eta, double gamma,
                                                   double* dq_deta) {
    double f[D];
    double prod = gamma;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        f[j] = 1.0 + eta[j] * kappa[j];
        prod *= f[j];
    }
    if (GRAD) {
        double pre = gamma;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            dq_deta[j] = pre * kappa[j];
            pre *= f[j];
        }
        double suf = 1.0;
#pragma unroll
        for (int j = D - 1; j >= 0; --j) {
            dq_deta[j] *= suf;
            suf *= f[j];
        }
    }
    return prod;
}

}  // namespace fmtgp
