// Transform passes with fused sources (generator / gathered data) and sinks
// (spectrum epilogue, gradient dot, coefficient scatter).
//
// Length-n real transforms:
//   lattice (SI):  V̄ a = DFT(bitrev a) (transforms.cpp:58-77) of a REAL column, computed as
//                  a half-length complex FFT of z(j) = a(2j) + i a(2j+1) plus the standard
//                  real-FFT post-processing; only the Hermitian half is stored: slot k holds
//                  A(k) for 1 <= k < n/2 and slot 0 packs (A(0), A(n/2)), both real.
//   digital (DSI): FWHT (transforms.cpp:19-30), real, natural order, n slots.
// One CTA transforms a tile of 2^11..2^13 elements; longer vectors use a two-pass four-step
// decomposition n' = N1 * N2 (column pass then row pass, intermediate through L2/HBM).
// Lattice slot layout of a two-pass transform: position k1*N2 + k2 <-> frequency
// k = k1 + N1*k2 (the row pass's natural output), identical for every vector of that length,
// which is all the per-frequency solve needs.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "generator.cuh"
#include "transform.cuh"

namespace cg = cooperative_groups;

namespace fmtgp {

constexpr int MAX_CAP_LOG = 13;  // elements per transform CTA <= 2^13 (NT = tile / EPT <= 512 threads)

// --------------------------------------------------------------------- geometry
struct Geo {
    int m;        // log2 n (task length)
    int lt;       // log2 of the transformed length: m-1 (lattice) or m (digital)
    int cap;      // log2 elements per CTA tile (11..13)
    int two;      // two-pass?
    int l1, l2;   // two-pass split lt = l1 + l2 (l2 = cap: a row fills one tile)
    int C;        // columns per CTA in the column pass
    // `total` = elements of all vectors transformed together; tiles shrink (down to 2^11) so
    // that small problems still launch >= ~2 CTAs per SM.
    __host__ __device__ static Geo make(int m, int lattice, long long total = 0) {
        Geo g{};
        g.m = m;
        g.lt = lattice ? (m > 0 ? m - 1 : 0) : m;
        int cap = MAX_CAP_LOG;
        while (cap > 11 && total > 0 && (total >> cap) < 296) --cap;
        while (g.lt > 2 * cap && cap < MAX_CAP_LOG) ++cap;
        g.cap = cap;
        g.two = g.lt > cap;
        if (g.two) {
            g.l2 = cap;
            g.l1 = g.lt - cap;
            g.C = 1 << (cap - g.l1);
        } else {
            g.l1 = 0;
            g.l2 = g.lt;
            g.C = 1;
        }
        return g;
    }
    __host__ __device__ long long slots(int lattice) const {
        return lattice ? (m > 0 ? (1ll << (m - 1)) : 1) : (1ll << m);
    }
    // position of lattice frequency k (0 <= k < n/2) in the slot layout
    __host__ __device__ long long pos_of(long long k) const {
        if (!two) return k;
        const long long N1 = 1ll << l1;
        return (k & (N1 - 1)) * (1ll << l2) + (k >> l1);
    }
};

// --------------------------------------------------------------------- sources
// Generator column of (pair, candidate) at transform-input index idx (lattice: DFT order,
// digital: natural order), WITHOUT R and scale (those go to the spectrum epilogue).
struct GenSrc {
    Spatial sp;
    PointGen pg;
    const uint64_t* offs;   // [P][MAXD] pair offsets
    const double* eta;      // [ncand][d]
    const double* gamma;    // [ncand]
    const int* vec_pair;    // [nvec_per_cand] -> global pair id
    int nvpc;               // vectors per candidate in this launch

    __device__ __forceinline__ void coords(int v, int& p, int& c) const {
        c = v / nvpc;
        p = vec_pair[v - c * nvpc];
    }
    __device__ __forceinline__ double kappa_all(int p, uint64_t idx, double* kappa) const {
        const uint64_t* off = offs + size_t(p) * MAXD;
        if (sp.family == 0) {
#pragma unroll
            for (int j = 0; j < MAXD; ++j)
                if (j < sp.d) kappa[j] = si_base(pg.lattice_word(idx, j, __ldg(off + j)), sp.si_alpha);
        } else {
#pragma unroll
            for (int j = 0; j < MAXD; ++j)
                if (j < sp.d) kappa[j] = dsi_walsh(pg.digital_z(idx, j) ^ __ldg(off + j), sp.b);
        }
        return 0.0;
    }
    __device__ __forceinline__ double operator()(int v, uint64_t idx) const {
        int p, c;
        coords(v, p, c);
        double kappa[MAXD];
        kappa_all(p, idx, kappa);
        return product_kernel<false>(kappa, eta + size_t(c) * sp.d, sp.d, __ldg(gamma + c), nullptr);
    }
};

// GenSrc with register arrays sized by a compile-time dimension cap DC >= d (4, 8 or 16):
// the generic MAXD = 16 arrays made the fused transform kernels spill.
template <int DC>
__device__ __forceinline__ double product_kernel_c(const double* kappa, const double* eta, int d, double gamma,
                                                   double* dq, bool grad) {
    double f[DC];
    double prod = gamma;
#pragma unroll
    for (int j = 0; j < DC; ++j)
        if (j < d) {
            f[j] = 1.0 + __ldg(eta + j) * kappa[j];
            prod *= f[j];
        }
    if (grad) {
        double pre = gamma;
#pragma unroll
        for (int j = 0; j < DC; ++j)
            if (j < d) {
                dq[j] = pre * kappa[j];
                pre *= f[j];
            }
        double suf = 1.0;
#pragma unroll
        for (int j = DC - 1; j >= 0; --j)
            if (j < d) {
                dq[j] *= suf;
                suf *= f[j];
            }
    }
    return prod;
}

template <int DC>
struct GenSrcD {
    GenSrc g;
    __device__ __forceinline__ void kappa_c(int p, uint64_t idx, double* kappa) const {
        const uint64_t* off = g.offs + size_t(p) * MAXD;
        if (g.sp.family == 0) {
#pragma unroll
            for (int j = 0; j < DC; ++j)
                if (j < g.sp.d) kappa[j] = si_base(g.pg.lattice_word(idx, j, __ldg(off + j)), g.sp.si_alpha);
        } else {
#pragma unroll
            for (int j = 0; j < DC; ++j)
                if (j < g.sp.d) kappa[j] = dsi_walsh(g.pg.digital_z(idx, j) ^ __ldg(off + j), g.sp.b);
        }
    }
    __device__ __forceinline__ double operator()(int v, uint64_t idx) const {
        int p, c;
        g.coords(v, p, c);
        double kappa[DC];
        kappa_c(p, idx, kappa);
        return product_kernel_c<DC>(kappa, g.eta + size_t(c) * g.sp.d, g.sp.d, __ldg(g.gamma + c), nullptr, false);
    }
};

// Data vector gathered into transform order: lattice y(bitrev_m(j)) (V̄ = DFT o bitrev),
// digital y(i).  src + vec_off[v] is the task's block.
struct ArraySrc {
    const double* src;
    const long long* vec_off;  // [nvec]
    int m;
    int bitrev;
    __device__ __forceinline__ double operator()(int v, uint64_t idx) const {
        const uint64_t i = bitrev ? bitrev64(idx, m) : idx;
        return __ldg(src + vec_off[v] + i);
    }
};

// Plain buffer already in transform-input order (the split generator's output).
struct BufSrc {
    const double* buf;  // [nvec][n]
    long long n;
    __device__ __forceinline__ double operator()(int v, uint64_t idx) const { return buf[v * n + idx]; }
};

// Kernel column of a query point against task l's design (posterior variance): value at
// transform-input index idx of vector v = (query q, task l) is R_{t,l} Q(x_q, x_{l, i(idx)})
// with the reference's floating SI difference for the free query coordinate
// (kernel_against_data, gp_core.cpp:386-397).
struct QuerySrc {
    int family, d, si_alpha, m, ntg, pad_;
    double b[4];
    double gamma;
    const double* X;          // [count][d]
    const double* eta;        // [d]
    const double* Rrow;       // [T] R_{task, l}
    const uint64_t* g;        // lattice [d]
    const uint64_t* cols;     // digital [d][m_cols]
    int m_cols;
    const uint64_t* shifts;   // [T][d]
    const int* vec_task;      // [ntg] task of each vector of the group
    __device__ double operator()(int v, uint64_t idx) const {
        const int q = v / ntg, l = vec_task[v - q * ntg];
        double prod = gamma;
        for (int j = 0; j < d; ++j) {
            const uint64_t sh = shifts[l * d + j];
            const double xq = X[(long long)q * d + j];
            double base;
            if (family == 0) {
                const uint64_t frac = ((idx * g[j]) & ((uint64_t(1) << m) - 1)) << (DIGITAL_BITS - m);
                const double xp = double((frac + sh) & MASK53) * 0x1p-53;
                const double diff = xq - xp;
                const double u1 = diff - floor(diff), u2 = -diff - floor(-diff);
                double u = fmin(u1, u2);
                if (u >= 1.0) u = 0.0;
                constexpr double pi2 = 9.869604401089358618834491;
                base = si_alpha == 1 ? 2.0 * pi2 * (u * (u - 1.0) + 1.0 / 6.0)
                                     : -(2.0 / 3.0) * pi2 * pi2 * (((u - 2.0) * u + 1.0) * u * u - 1.0 / 30.0);
            } else {
                uint64_t z = sh;
                const uint64_t* c = cols + size_t(j) * m_cols;
                uint64_t i = idx;
                for (int p = 0; i; ++p, i >>= 1)
                    if (i & 1) z ^= c[p];
                base = dsi_walsh(uint64_t(xq * 0x1p53) ^ z, b);
            }
            prod *= 1.0 + eta[j] * base;
        }
        return Rrow[l] * prod;
    }
};

// --------------------------------------------------------------------- forward sinks
// lam = coef * A + xi, coef = R_ab * sqrt(n_b / n_a) (fast_gram.cpp:82-85).
// Lattice slot 0 packs (A(0), A(n/2)): both real, both get + xi.
struct SpecSink {
    void* out;              // double2 (lattice) or double (digital)
    const long long* voff;  // [nvec_per_cand] slot offset of each vector
    long long cstride;      // slots per candidate
    const double* coef;     // [ncand][nvpc]
    const double* xi;       // [ncand][nvpc]
    int nvpc;
    __device__ __forceinline__ void put(int v, long long pos, double2 A) const {
        const int c = v / nvpc, q = v - c * nvpc;
        const double s = __ldg(coef + v), x = __ldg(xi + v);
        double2* o = static_cast<double2*>(out) + c * cstride + voff[q] + pos;
        *o = make_double2(fma(s, A.x, x), pos == 0 ? fma(s, A.y, x) : s * A.y);
    }
    __device__ __forceinline__ void put(int v, long long pos, double A) const {
        const int c = v / nvpc, q = v - c * nvpc;
        double* o = static_cast<double*>(out) + c * cstride + voff[q] + pos;
        *o = fma(__ldg(coef + v), A, __ldg(xi + v));
    }
};

struct ScaleSink {  // yhat = n^{-1/2} * transform
    void* out;
    const long long* voff;
    double scale;
    __device__ __forceinline__ void put(int v, long long pos, double2 A) const {
        static_cast<double2*>(out)[voff[v] + pos] = cscale(A, scale);
    }
    __device__ __forceinline__ void put(int v, long long pos, double A) const {
        static_cast<double*>(out)[voff[v] + pos] = A * scale;
    }
};

// --------------------------------------------------------------------- inverse sinks
// Gradient dot: for W = unnormalised inverse transform of M_ab (real), accumulate
// sum_j W(j) * dq(j)/deta_k (k < d) and sum_j W(j) q(j) (slot d).  Lattice receives the
// half-length complex z'(j): W(2j) = 2 Re z', W(2j+1) = 2 Im z'.
struct GradSink {
    GenSrc gen;
    double* partial;  // [nvec][nblk][MAXD+1]
    int nblk;
    int acc_n;        // d + 1
};

// Coefficients c = V chat scattered to natural point order:
//   lattice c(bitrev_m(j)) = sqrt(n) * IDFT_n(chat)(j):  c(bitrev(2j)) = s Re z'(j), ... with
//   s = sqrt(n) / (n/2);  digital c = n^{-1/2} H chat.
struct CoefSink {
    double* out;
    const long long* voff;  // [nvec] element offset of the task block
    int m;
    double scale;
};

// --------------------------------------------------------------------- helpers
// Real-FFT post-processing: A(k) from Z(k), Z(N'-k); wk = exp(-2 pi i k / n).
__device__ __forceinline__ double2 r2c_post(double2 Zk, double2 Zp, double2 wk) {
    const double2 E = make_double2(0.5 * (Zk.x + Zp.x), 0.5 * (Zk.y - Zp.y));
    const double2 D = make_double2(Zk.x - Zp.x, Zk.y + Zp.y);  // Zk - conj(Zp)
    const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);     // -i D / 2
    return cadd(E, cmul(wk, O));
}
// Inverse pre-processing: Z(k) from A(k), A(N'-k); wk = exp(-2 pi i k / n) (conjugated inside).
__device__ __forceinline__ double2 c2r_pre(double2 Ak, double2 Ap, double2 wk) {
    const double2 E = make_double2(0.5 * (Ak.x + Ap.x), 0.5 * (Ak.y - Ap.y));
    const double2 D = make_double2(0.5 * (Ak.x - Ap.x), 0.5 * (Ak.y + Ap.y));
    const double2 O = cmulc(D, wk);  // D * exp(+2 pi i k/n)
    return make_double2(E.x - O.y, E.y + O.x);  // E + i O
}

// --------------------------------------------------------------------- per-frequency solve
// Hermitian LDL^H of A (upper pairs, row by row), T <= 8.  Pivots are the diagonal Schur
// complements of Algorithm 1 (fast_gram.cpp:167-178): logdet = sum log d_s.
// Returns 0 ok, 1 non-positive pivot (SchurBreakdown), 2 non-real diagonal (FastMtgpError).
// ldl_core multiplies the pivots into a running product pm * 2^pe (pm frexp-normalised, so no
// pivot range can overflow it): a kernel that solves many frequencies takes ONE log at the end.
template <int T, bool CX>
__device__ __forceinline__ int ldl_core(const typename Sc<CX>::T* A, const typename Sc<CX>::T* r, bool want_inv,
                                        double& pm, int& pe, double& quad, typename Sc<CX>::T* chat,
                                        typename Sc<CX>::T* Ainv, double* imx, double* rex) {
    using S = Sc<CX>;
    using V = typename S::T;
    V L[T][T];
    double dinv[T], piv[T];
    int status = 0;
    double pprod = 1.0;  // this frequency's pivot product (T <= 8 covariance pivots: no overflow)
    // pair index of (a,b), a <= b, row by row (fast_gram.cpp:35-40)
    auto pidx = [](int a, int b) { return a * T - a * (a - 1) / 2 + (b - a); };
#pragma unroll
    for (int s = 0; s < T; ++s) {
        double dd = S::re(A[pidx(s, s)]);
        // non-real check is global per stage (|Im S| vs 1e-8 max(1, max Re S)), fast_gram.cpp:167-172;
        // real (digital) spectra have no imaginary part to test
        if constexpr (CX) imx[s] = fmax(imx[s], fabs(S::im(A[pidx(s, s)])));
#pragma unroll
        for (int k = 0; k < s; ++k) dd -= S::abs2(L[s][k]) * piv[k];
        if (!(dd > 0.0)) {
            status = 1;
            dd = 1.0;
        }
        if constexpr (CX) rex[s] = fmax(rex[s], dd);
        piv[s] = dd;
        dinv[s] = 1.0 / dd;
        pprod *= dd;
#pragma unroll
        for (int i = s + 1; i < T; ++i) {
            V acc = S::conj(A[pidx(s, i)]);
#pragma unroll
            for (int k = 0; k < s; ++k) acc = S::sub(acc, S::scale(S::mulc(L[i][k], L[s][k]), piv[k]));
            L[i][s] = S::scale(acc, dinv[s]);
        }
    }
    {
        int e;
        pm = frexp(pm * pprod, &e);  // one renormalisation per frequency
        pe += e;
    }
    // z = L^-1 r, quad = sum |z|^2 / d
    V z[T];
    quad = 0.0;
#pragma unroll
    for (int i = 0; i < T; ++i) {
        V acc = r[i];
#pragma unroll
        for (int k = 0; k < i; ++k) acc = S::sub(acc, S::mul(L[i][k], z[k]));
        z[i] = acc;
        quad += S::abs2(acc) * dinv[i];
    }
    // chat = L^-H D^-1 z
#pragma unroll
    for (int i = T - 1; i >= 0; --i) {
        V acc = S::scale(z[i], dinv[i]);
#pragma unroll
        for (int k = i + 1; k < T; ++k) acc = S::sub(acc, S::mul(S::conj(L[k][i]), chat[k]));
        chat[i] = acc;
    }
    if (want_inv) {
        // X = L^-1 (unit lower); Ainv_ab = sum_{s >= max(a,b)} conj(X_sa) X_sb / d_s
        V X[T][T];
#pragma unroll
        for (int j = 0; j < T; ++j)
#pragma unroll
            for (int i = j + 1; i < T; ++i) {
                V acc = S::sub(S::zero(), L[i][j]);
#pragma unroll
                for (int k = j + 1; k < i; ++k) acc = S::sub(acc, S::mul(L[i][k], X[k][j]));
                X[i][j] = acc;
            }
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int b = a; b < T; ++b) {
                V acc = S::zero();
#pragma unroll
                for (int s = b; s < T; ++s) {
                    // conj(X_sa) X_sb with X_ss = 1
                    V term;
                    if (s == a) term = S::one();  // then b == a == s
                    else if (s == b) term = S::conj(X[s][a]);
                    else term = S::mulc(X[s][b], X[s][a]);
                    acc = S::add(acc, S::scale(term, dinv[s]));
                }
                Ainv[pidx(a, b)] = acc;
            }
    }
    return status;
}

__device__ __forceinline__ double log_of(double pm, int pe) { return log(pm) + double(pe) * 0.69314718055994530942; }

// One frequency: logdet = sum log d_s.
template <int T, bool CX>
__device__ __forceinline__ int ldl_solve(const typename Sc<CX>::T* A, const typename Sc<CX>::T* r, bool want_inv,
                                         double& logdet, double& quad, typename Sc<CX>::T* chat,
                                         typename Sc<CX>::T* Ainv, double* imx, double* rex) {
    double pm = 1.0;
    int pe = 0;
    const int st = ldl_core<T, CX>(A, r, want_inv, pm, pe, quad, chat, Ainv, imx, rex);
    logdet = log_of(pm, pe);
    return st;
}

// --------------------------------------------------------------------- split-mode generator helpers
template <int D>
struct GenSmem {
    uint64_t lo[D][32], mid[D][32];
    double T8[256];
    double eta[D];
};

template <int D>
__device__ __forceinline__ void gen_smem_init(GenSmem<D>& t, const GenSrc& g, int c, bool load_eta = true) {
    if (g.sp.family == 1) {
        for (int e = threadIdx.x; e < D * 64; e += blockDim.x) {
            const int j = e >> 6, r = e & 63;
            const int shift = r < 32 ? 0 : 5;
            const int val = r & 31;
            uint64_t z = 0;
            const uint64_t* col = g.pg.cols + size_t(j) * g.pg.m_cols;
            for (int p = 0; p < 5; ++p)
                if (((val >> p) & 1) && p + shift < g.pg.m_cols) z ^= __ldg(col + p + shift);
            if (r < 32) t.lo[j][val] = z;
            else t.mid[j][val] = z;
        }
        for (int b = threadIdx.x; b < 256; b += blockDim.x) {
            double acc = 0.0;
            for (int i = 7; i >= 0; --i)  // smallest terms first
                if ((b >> (7 - i)) & 1) acc += pow2i(-3 * i);
            t.T8[b] = acc;
        }
    }
    if (load_eta)
        for (int j = threadIdx.x; j < D; j += blockDim.x) t.eta[j] = g.eta[size_t(c) * D + j];
}

template <int D>
__device__ __forceinline__ void kappa_d(const GenSrc& g, const GenSmem<D>& t, const uint64_t* off, uint64_t idx,
                                        double* kappa) {
    if (g.sp.family == 0) {
#pragma unroll
        for (int j = 0; j < D; ++j) kappa[j] = si_base(g.pg.lattice_word(idx, j, off[j]), g.sp.si_alpha);
        return;
    }
    const uint64_t hi = idx >> 10;
    const bool only4 = g.sp.b[0] == 0.0 && g.sp.b[1] == 0.0 && g.sp.b[2] == 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        uint64_t z = t.lo[j][idx & 31] ^ t.mid[j][(idx >> 5) & 31];
        if (hi) {
            const uint64_t* col = g.pg.cols + size_t(j) * g.pg.m_cols + 10;
            uint64_t h = hi;
            for (int q = 0; h; ++q, h >>= 1)
                if (h & 1) z ^= __ldg(col + q);
        }
        const uint64_t w = z ^ off[j];
        kappa[j] = only4 ? g.sp.b[3] * dsi_order4_t8(w, t.T8) : dsi_walsh(w, g.sp.b);
    }
}

}  // namespace fmtgp
