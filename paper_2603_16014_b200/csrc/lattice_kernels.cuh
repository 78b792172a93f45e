// Kernel templates of the fused lattice path (lattice.cu documents the design).  Instantiated
// per FFT length in lat_inst_<L>.cu (the L1 / L3 column kernels on the column length N1 = 2^L,
// the L2 row kernel on the row length N2 = 2^L) so the six lengths compile in parallel.
#pragma once

#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>

#include "ipfft.cuh"
#include "lattice.cuh"

namespace fmtgp {

namespace cg = cooperative_groups;

constexpr int LAT_NT = 512;  // one radix-16 group per thread per FFT stage, 2^13-element tiles

// compile-time switches of measured variants (tools/r03_variants.sh builds A/B libraries)
#ifndef LAT_GEN_PROD
#define LAT_GEN_PROD 1     // L1 / L3 lattice generator in product form (LatGen::init_prod)
#endif
#ifndef LAT_L2_PAIRFORM
#define LAT_L2_PAIRFORM 1  // L2 solve: pair form of the real-FFT post/pre-processing, branch-free main loop
#endif
#ifndef LAT_L2_UNROLL
#define LAT_L2_UNROLL 1    // unroll factor of that loop
#endif
constexpr int LAT_UNROLL_V = LAT_L2_UNROLL;

// ------------------------------------------------------------------ generator on the fly
// Lattice coordinate of real DFT-order index i against the class offset (lattice_word in
// generator.cuh, ld_sequences.cpp:31-53): with off = oh 2^(53-m) + olo (olo < 2^(53-m)),
//   D = ((i g + oh) mod 2^m) 2^(53-m) + olo,   x = D 2^-53 = t 2^-m + olo 2^-53  (exact in fp64),
// so the 64-bit multiply / shift / mask chain becomes one 32-bit IMAD + LOP, the conversion of t
// one exact DADD (u32_to_f64: no quarter-rate I2F.F64) and one DFMA.  The generator works with
// y = x - 1/2 = t 2^-m + (olo 2^-53 - 1/2), exact (a multiple of 2^-53 below 1/2 in magnitude).
// The Bernoulli kernels are polynomials in w = x^2 - x = y^2 - 1/4 = -u (1 - u), symmetric under
// u -> 1 - u, so the reference's symmetrisation u = min(x, 1 - x) (kernels.cpp:28-32) is implied:
//   B2: kappa = 2 pi^2 (u^2 - u + 1/6)            = ka y^2 + kb,     ka = 2 pi^2,      kb = -pi^2 / 6
//   B4: kappa = -(2/3) pi^4 (u^2 (u - 1)^2 - 1/30) = ka w^2 + kb,     ka = -(2/3) pi^4, kb = pi^4 / 45
// and f = 1 + eta kappa = A + B v with v = y^2 (B2) or w^2 (B4), A = 1 + eta kb, B = eta ka:
// two fp64 operations per dimension after y (three for B4).  Dimensions are padded to the register
// cap DC with A = 1, B = 0 (f = 1 exactly), so the unrolled loops carry no per-dimension predicates.
template <int ALPHA>
struct LatPoly {
    static constexpr double pi2 = 9.869604401089358618834491;
    static constexpr double ka = ALPHA == 1 ? 2.0 * pi2 : -(2.0 / 3.0) * pi2 * pi2;
    static constexpr double kb = ALPHA == 1 ? -pi2 / 6.0 : pi2 * pi2 / 45.0;  // B2: pi^2/3 - ka/4 (y form)
};

template <int DC, int ALPHA>
struct LatGen {
    uint32_t gm[DC], oh[DC];
    double ol[DC], A[DC], B[DC];  // ol: olo 2^-53 - 1/2
    double gam, inv_n;
    uint32_t mask;
    __device__ __forceinline__ void init(const LatArgs& a, int c, int o) {
        mask = (a.m >= 32) ? 0xffffffffu : ((1u << a.m) - 1u);
        inv_n = pow2i(-a.m);
        gam = __ldg(a.gamma + c);
        const int sh = DIGITAL_BITS - a.m;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            if (j < a.d) {
                const uint64_t off = __ldg(a.cofs + size_t(o) * MAXD + j) & MASK53;
                const double eta = __ldg(a.eta + size_t(c) * a.d + j);
                gm[j] = uint32_t(__ldg(a.g + j)) & mask;
                oh[j] = uint32_t(off >> sh) & mask;
                ol[j] = fma(double(off & ((uint64_t(1) << sh) - 1)), 0x1p-53, -0.5);  // exact
                A[j] = fma(eta, LatPoly<ALPHA>::kb, 1.0);
                B[j] = eta * LatPoly<ALPHA>::ka;
            } else {
                gm[j] = oh[j] = 0u;
                ol[j] = -0.5;
                B[j] = 0.0;
                A[j] = 1.0;
            }
        }
    }
    // v_j = y^2 (B2) or w^2 (B4) of dimension j at real DFT-order index i
    __device__ __forceinline__ double v(int j, uint32_t i) const {
        const uint32_t t = (i * gm[j] + oh[j]) & mask;
        const double y = fma(u32_to_f64(t), inv_n, ol[j]);  // x - 1/2, exact
        if (ALPHA == 1) return y * y;
        const double w = fma(y, y, -0.25);
        return w * w;
    }
    // q(i) = gamma prod_j (1 + eta_j kappa_j)  (SpatialKernel, kernels.cpp:91-103)
    __device__ __forceinline__ double q(uint32_t i) const {
        double prod = gam;
#pragma unroll
        for (int j = 0; j < DC; ++j) prod *= fma(B[j], v(j, i), A[j]);
        return prod;
    }
    // ---- product form (every eta_j kappa-slope B_j != 0): f_j = B_j g_j with g_j = v_j + A_j / B_j, so
    //   q = Gam prod_j g_j,  Gam = gamma prod_j B_j,   g_j = fma(y, y, c_j)  (B2; B4: fma(w, w, c_j))
    // — one fp64 operation per dimension less than A + B v — and kappa_j = ka h_j, h_j = v_j + kb / ka:
    //   dq/deta_j = [gamma ka prod_{k != j} B_k] h_j prod_{k != j} g_k,
    // the bracket applied once per reduced sum (dscale).  Padded dimensions generate y = 0 and g = 1.
    // init_prod() returns false when some B_j is too small to divide by (callers then use q / dq_acc).
    static constexpr double ke = LatPoly<ALPHA>::kb / LatPoly<ALPHA>::ka;  // -1/12 (B2), -1/30 (B4)
    __device__ __forceinline__ bool init_prod(const LatArgs& a, int c, int o) {
        init(a, c, o);
        bool ok = true;
        double G = gam;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            if (j < a.d) {
                ok = ok && fabs(B[j]) > 1e-100;
                G *= B[j];
                A[j] = A[j] / B[j];  // c_j
            } else {
                ol[j] = 0.0;                              // y = 0
                A[j] = ALPHA == 1 ? 1.0 : 15.0 / 16.0;    // g = 1 exactly
            }
        }
        if (ok) gam = G;
        return ok;
    }
    __device__ __forceinline__ double yv(int j, uint32_t i) const {
        const uint32_t t = (i * gm[j] + oh[j]) & mask;
        const double y = fma(u32_to_f64(t), inv_n, ol[j]);
        return ALPHA == 1 ? y : fma(y, y, -0.25);
    }
    __device__ __forceinline__ double q_prod(uint32_t i) const {
        double prod = gam;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            const double u = yv(j, i);
            prod *= fma(u, u, A[j]);
        }
        return prod;
    }
    // acc_j += W h_j prod_{k != j} g_k (unscaled; see dscale)
    __device__ __forceinline__ void dq_acc_prod(uint32_t i, double W, double* acc) const {
        double g[DC], h[DC];
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            const double u = yv(j, i);
            g[j] = fma(u, u, A[j]);
            h[j] = fma(u, u, ke);
        }
        if constexpr (DC == 4) {  // pair tree: 12 operations instead of 14
            const double Wa = W * (g[0] * g[1]), Wb = W * (g[2] * g[3]);
            acc[0] = fma(h[0], g[1] * Wb, acc[0]);
            acc[1] = fma(h[1], g[0] * Wb, acc[1]);
            acc[2] = fma(h[2], g[3] * Wa, acc[2]);
            acc[3] = fma(h[3], g[2] * Wa, acc[3]);
        } else if constexpr (DC == 2) {
            acc[0] = fma(h[0], g[1] * W, acc[0]);
            acc[1] = fma(h[1], g[0] * W, acc[1]);
        } else {
            double pre = W, t[DC];
#pragma unroll
            for (int j = 0; j < DC; ++j) {
                t[j] = pre * h[j];
                pre *= g[j];
            }
            double suf = 1.0;
#pragma unroll
            for (int j = DC - 1; j >= 0; --j) {
                acc[j] = fma(t[j], suf, acc[j]);
                suf *= g[j];
            }
        }
    }
    // factor of acc_j after the reduction: gamma ka prod_{k != j, k < d} B_k (from the hyperparameters)
    static __device__ double dscale(const LatArgs& a, int c, int j) {
        double s = __ldg(a.gamma + c) * LatPoly<ALPHA>::ka;
        for (int k = 0; k < a.d; ++k)
            if (k != j) s *= __ldg(a.eta + size_t(c) * a.d + k) * LatPoly<ALPHA>::ka;
        return s;
    }
    // acc_j += W dq/deta_j = W gamma kappa_j prod_{k != j} f_k  (prefix / suffix products: f may vanish)
    __device__ __forceinline__ void dq_acc(uint32_t i, double W, double* acc) const {
        double vv[DC], f[DC];
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            vv[j] = v(j, i);
            f[j] = fma(B[j], vv[j], A[j]);
        }
        double pre = gam * W;
        double dq[DC];
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            dq[j] = pre * fma(LatPoly<ALPHA>::ka, vv[j], LatPoly<ALPHA>::kb);
            pre *= f[j];
        }
        double suf = 1.0;
#pragma unroll
        for (int j = DC - 1; j >= 0; --j) {
            acc[j] = fma(dq[j], suf, acc[j]);
            suf *= f[j];
        }
    }
};

// ------------------------------------------------------------------ exchange-block layout
// Row k1 -> (owner rank h, local row i): cluster q = min(k1, N1 - k1) (rows 0 and N1/2 form
// cluster 0), side = 1 for the upper row of the pair.
__device__ __forceinline__ int row_owner(int k1, int N1, int lqp, int& i) {
    int q, side;
    if (k1 == 0) q = 0, side = 0;
    else if (k1 == (N1 >> 1)) q = 0, side = 1;
    else if (k1 < (N1 >> 1)) q = k1, side = 0;
    else q = N1 - k1, side = 1;
    const int h = q >> lqp;
    i = 2 * (q - (h << lqp)) + side;
    return h;
}
// element (row owner h, class o, local row i, local column jl) of candidate c's exchange blocks
// offset inside one candidate's blocks (< V n' <= 2^31: 32-bit arithmetic)
__device__ __forceinline__ unsigned xoff(const LatArgs& a, int h, int o, int i, int jl) {
    return ((unsigned(h * a.V + o) * unsigned(a.R) + unsigned(i)) << a.lwc) + unsigned(jl);
}
__device__ __forceinline__ size_t xaddr(const LatArgs& a, int c, int h, int o, int i, int jl) {
    return size_t(c) * a.V * a.half + (((size_t(h) * a.V + o) * a.R + i) << a.lwc) + jl;
}
// forward blocks (L1 -> L2), column-chunked: [kc][h][o][i][jl mod WC/K] (== xoff when K = 1)
__device__ __forceinline__ unsigned xoff_f(const LatArgs& a, int h, int o, int i, int jl) {
    const int lw = a.lwc - a.lkc, kc = jl >> lw;
    return ((unsigned(((kc << a.lg) + h) * a.V + o) * unsigned(a.R) + unsigned(i)) << lw) +
           unsigned(jl & ((1 << lw) - 1));
}
// return blocks (L2 -> L3), row-chunked: [kr][h][o][i mod R/K][jl] (== xoff when K = 1)
__device__ __forceinline__ unsigned xoff_r(const LatArgs& a, int h, int o, int i, int jl) {
    const int lr = a.lqp + 1 - a.lkc, kr = i >> lr;
    return ((unsigned((((kr << a.lg) + h) * a.V + o) << lr) + unsigned(i & ((1 << lr) - 1))) << a.lwc) + unsigned(jl);
}

// ------------------------------------------------------------------ L1: generator x column FFT
// In-place DIF column FFT (ipfft.cuh) of C = 2^lc columns of N1 = 2^l1 rows (C N1 = 16 NT):
// stage 0 is fused with the generator (each thread generates its radix-16 group straight into
// registers), the twiddle-free tail stage with the store of the exchange blocks (row k1 =
// ip_freq of the position).  The four-step twiddle w_{n'}^(k1 j2) is applied by L2 on its inputs.
__device__ __forceinline__ void cluster_arrive_rel() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acq() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_count() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}

template <int NT, int DC, int ALPHA, int L1>
__global__ void __launch_bounds__(NT) k_lat_col_fwd(LatArgs a, int l2, int lc) {
    using IP = Ip<L1>;
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    constexpr int N1 = 1 << L1, ld = padded_len(N1);
    constexpr int M_log = L1 - 4;  // stage-0 stride; also log2 of the 16-position chunks per column
    cg::cluster_group cl = cg::this_cluster();
    // K CTAs of a cluster take K adjacent column blocks; after the column FFT each CTA stores a
    // quarter (1/K) of the rows of ALL K*C columns, reading the other CTAs' columns over DSMEM,
    // so every row segment written is K*C*16 contiguous bytes instead of 16
    const int K = int(cluster_count()), crank = int(cluster_rank());
    int lk = 0;
    while ((1 << lk) < K) ++lk;
    const int C = 1 << lc, kcl = lk + lc;
    // thread -> column vec, stage-0 group j1; its tail chunk is positions p0 .. p0+15 of the same column
    const int vec = threadIdx.x >> M_log, j1 = threadIdx.x & ((1 << M_log) - 1), p0 = j1 << 4;
    const double2* src[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) src[r] = r < K ? cl.map_shared_rank(sm, r) : sm;
    Tw16 t0;
    t0.load(a.tw, j1, L1);  // the same for every tile
    // zero the per-fit flags once per fit (L2 / L3 run after this kernel)
    if (blockIdx.x == 0 && a.chunk <= 0) {
        for (int t = threadIdx.x; t < a.nc; t += NT) a.bad[t] = 0x7f7f7f7f;
        for (int t = threadIdx.x; t < a.nc * MAXT * 2; t += NT) a.imre[t] = 0ull;
    }
    pdl_trigger();
    // persistent over cluster tiles (K column blocks x class x candidate): a tile's exchange-block
    // stores drain while the next tile's generator (registers only) runs
    // a chunked launch (a.chunk >= 0) covers the cluster blocks of column chunk a.chunk only
    const int ncbk = a.ncb >> (lk + (a.chunk >= 0 ? a.lkc : 0));
    const int bk0 = a.chunk >= 0 ? a.chunk * ncbk : 0;
    const int ntiles = ncbk * a.V * a.nc, nclus = int(gridDim.x) >> lk, cid = int(blockIdx.x) >> lk;
    cluster_arrive_relaxed();
#pragma unroll 1
    for (int tile = cid; tile < ntiles; tile += nclus) {
        const int bk = bk0 + tile % ncbk, v = tile / ncbk, c = v / a.V, o = v - c * a.V;
        const int bx = (bk << lk) + crank;
        const uint32_t c0 = uint32_t(a.rank * a.ncb + bx) << lc;  // global first column of this CTA
        double2 x[16];
        {
            LatGen<DC, ALPHA> G;
#if LAT_GEN_PROD
            if (G.init_prod(a, c, o)) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t J = (uint32_t(j1 + (r << M_log)) << l2) + c0 + uint32_t(vec);
                    x[r] = make_double2(G.q_prod(2u * J), G.q_prod(2u * J + 1u));
                }
            } else
#endif
            {
                G.init(a, c, o);
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t J = (uint32_t(j1 + (r << M_log)) << l2) + c0 + uint32_t(vec);
                    x[r] = make_double2(G.q(2u * J), G.q(2u * J + 1u));
                }
            }
        }
        dif16_regs(x, t0);
        cluster_wait_acq();  // every CTA of the cluster has read the previous tile out of smem
        {
            double2* xs = sm + vec * ld + S(j1);
#pragma unroll
            for (int r = 0; r < 16; ++r) xs[ip_off<M_log>(brev_c<16>(r))] = x[r];
        }
        __syncthreads();
        ip_mid_stages<NT, L1, false, true, false, true>(sm, C, ld, a.tw);  // warp-local after stage 0 (ipfft.cuh)
        // tail stage, results back in place
        {
            double2* xs = sm + vec * ld + S(p0);
#pragma unroll
            for (int r = 0; r < 16; ++r) x[r] = xs[r];
            tail_regs<L1>(x, -1);
#pragma unroll
            for (int r = 0; r < 16; ++r) xs[tail_out_pos<L1>(r)] = x[r];
        }
        cl.sync();
        // transposed store: positions [crank N1/K, (crank+1) N1/K) x the cluster's K*C columns
        const int jlb = ((a.rank * a.ncb + (bk << lk)) << lc) - a.rank * a.WC;
        double2* Yc = a.Y + size_t(c) * a.V * a.half;
#pragma unroll 4
        for (int u = 0; u < 16; ++u) {
            const int e = int(threadIdx.x) + u * NT;
            const int cc = e & ((1 << kcl) - 1);
            const int p = (crank << (L1 - lk)) + (e >> kcl);
            const int k1 = IP::freq(p);
            int i;
            const int h = row_owner(k1, N1, a.lqp, i);
            Yc[xoff_f(a, h, o, i, jlb + cc)] = src[cc >> lc][(cc & (C - 1)) * ld + S(p)];
        }
        // relaxed: the remote reads above have completed (their values were stored), and a
        // release here would wait for every outstanding exchange-block store to drain
        cluster_arrive_relaxed();
    }
    cluster_wait_acq();  // no CTA leaves while another still reads its smem
}

// ------------------------------------------------------------------ L2: row FFT + solve + inverse row FFT
// Closed-form 2 x 2 Hermitian solve: ldl_core<2, true>'s outputs (pivots a and det / a, their
// product det into pm 2^pe, quad = r^H A^-1 r, chat = A^-1 r, A^-1, the non-real / pivot maxima
// of Algorithm 1's two stages, fast_gram.cpp:167-178) with one reciprocal instead of two and no
// triangular solves.  A = [A00, A01, A11] (pair order), status 1 on a non-positive pivot.
template <bool TRACK_IM = true>
__device__ __forceinline__ int herm2_solve(const double2* A, const double2* r, double& pm, int& pe, double& quad,
                                           double2* chat, double2* Ainv, double* imx, double* rex) {
    int status = 0;
    double a = A[0].x;
    const double d = A[2].x;
    const double2 b = A[1];
    if constexpr (TRACK_IM) {  // (the pair-form loop tracks max |Im H| of the diagonal class instead)
        imx[0] = fmax(imx[0], fabs(A[0].y));
        imx[1] = fmax(imx[1], fabs(A[2].y));
    }
    if (!(a > 0.0)) status = 1, a = 1.0;
    double det = fma(a, d, -(b.x * b.x + b.y * b.y));  // a * (second pivot)
    if (!(det > 0.0)) status = 1, det = a;              // second pivot -> 1, as ldl_core
    const double ip = 1.0 / (a * det);
    const double idet = a * ip;                          // 1 / det
    rex[0] = fmax(rex[0], a);
    rex[1] = fmax(rex[1], det * (det * ip));             // det / a
    {
        int e;
        pm = frexp(pm * det, &e);
        pe += e;
    }
    Ainv[0] = make_double2(d * idet, 0.0);
    Ainv[1] = make_double2(-b.x * idet, -b.y * idet);
    Ainv[2] = make_double2(a * idet, 0.0);
    // chat = A^-1 r: A^-1 = [[d, -b], [-conj b, a]] / det
    if constexpr (TRACK_IM) {
        chat[0] = cscale(csub(cscale(r[0], d), cmul(b, r[1])), idet);
        chat[1] = cscale(csub(cscale(r[1], a), cmulc(r[0], b)), idet);
    } else {  // from the entries of A^-1 just formed: 6 operations per component instead of 10
        const double2 o = Ainv[1];
        chat[0] = make_double2(fma(o.x, r[1].x, fma(-o.y, r[1].y, Ainv[0].x * r[0].x)),
                               fma(o.x, r[1].y, fma(o.y, r[1].x, Ainv[0].x * r[0].y)));
        chat[1] = make_double2(fma(o.x, r[0].x, fma(o.y, r[0].y, Ainv[2].x * r[1].x)),
                               fma(o.x, r[0].y, fma(-o.y, r[0].x, Ainv[2].x * r[1].y)));
    }
    quad = r[0].x * chat[0].x + r[0].y * chat[0].y + r[1].x * chat[1].x + r[1].y * chat[1].y;
    return status;
}
__device__ __forceinline__ int lat_row_of(int q, int rank, int N1) {
    if (q == 0) return rank == 0 ? 0 : N1 / 2;
    return rank == 0 ? q : N1 - q;
}

// Class of pair y (row-by-row pair order) when every task has its own shift (the BASELINE
// designs): all diagonal pairs share offset 0 (class 0), every off-diagonal pair is its own class.
template <int T>
__host__ __device__ constexpr int cls_distinct(int y) {
    int q = 0, off = 0;
    for (int a = 0; a < T; ++a)
        for (int b = a; b < T; ++b, ++q) {
            if (q == y) return a == b ? 0 : 1 + off;
            if (a != b) ++off;
        }
    return 0;
}

template <int T>
__host__ __device__ constexpr bool pair_is_diag(int y) {
    int q = 0;
    for (int a = 0; a < T; ++a)
        for (int b = a; b < T; ++b, ++q)
            if (q == y) return a == b;
    return false;
}

// DIST: the class map is cls_distinct<T> (compile time: no per-pair class selects); otherwise
// it comes from LatArgs::pair_ofs.
// Row transforms are in place (ipfft.cuh): DIF stage 0 applies the four-step twiddle
// w_{n'}^(row j2), j2 = gj1 + r N2/16, split as a per-CTA step table on its inputs (s_ostep[r])
// and a per-thread base merged into the stage's output twiddles (Tw16B: the base is never
// multiplied into the inputs); the middle stage reads its twiddles from a shared-memory table
// (IpTw); the solve walks the DIF output in POSITION order (bank-conflict free; yhat comes in the
// matching permuted layout, LatArgs::yperm), and the last DIT stage applies the conjugates on
// its way to HBM.
template <int NT, int T, bool DIST, int L2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT) k_lat_mid(LatArgs a, int l1) {
    constexpr int l2 = L2;
    using IP = Ip<L2>;
    constexpr int P = T * (T + 1) / 2;
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);  // [V][padded N2]
    constexpr auto S = sidx<true>;
    __shared__ double s_coef[P], s_xi[P], s_wR[P];
    __shared__ double s_coefh[P], s_wRh[P];  // halves: the pair-form loop works with 2 H and Z / 2
    __shared__ int s_cls[P];
    __shared__ double2 s_ostep[16], s_rstep[16];
    __shared__ double2 s_tw[IpTw<L2>::N];  // middle-stage twiddles, filled in the prologue
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank());
    // local row index of this CTA's row in the exchange blocks (a chunked launch: row chunk a.chunk)
    const int li = (a.chunk >= 0 ? a.chunk << (a.lqp + 1 - a.lkc) : 0) + int(blockIdx.x);
    const int q = a.rank * a.QP + (li >> 1), c = blockIdx.y, V = DIST ? P - T + 1 : a.V;
    auto cls = [&](int y) { return DIST ? cls_distinct<T>(y) : s_cls[y]; };
    constexpr int N2 = 1 << L2, lds = padded_len(N2);
    const int N1 = 1 << l1, lt = l1 + l2;
    constexpr int M_log = L2 - 4;
    const int row = lat_row_of(q, rank, N1);
    const long long half = a.half;
    const bool selfrow = q == 0;  // rows 0 and N1/2 pair with themselves
    const int rowA = selfrow ? row : q, rowB = selfrow ? row : N1 - q;
    // prologue independent of L1 (overlaps its tail under programmatic dependent launch)
    if (threadIdx.x < P) {
        const int p = threadIdx.x;
        s_coef[p] = __ldg(a.coef + size_t(c) * P + p);
        s_xi[p] = __ldg(a.xi + size_t(c) * P + p);
        s_wR[p] = (a.pair_a[p] == a.pair_b[p] ? 1.0 : 2.0) * __ldg(a.Rpair + size_t(c) * P + p);
        s_coefh[p] = 0.5 * s_coef[p];
        s_wRh[p] = 0.5 * s_wR[p];
        s_cls[p] = a.pair_ofs[p];
    } else if (threadIdx.x >= 32 && threadIdx.x < 48) {
        const int u = threadIdx.x - 32;  // four-step step table: w^(row M u), M = N2 / 16
        s_ostep[u] = twiddle(a.tw, (uint64_t(u) << M_log) * uint64_t(row), lt);
    } else if (threadIdx.x >= 64 && threadIdx.x < 80) {
        // real-FFT step table: the solve's position pA advances by NT per iteration, i.e. the top
        // DIF digit by NT / 2^(l2-4), so k2a advances by that much: w_{2 N2}^(u (NT >> (l2-4)))
        const int u = threadIdx.x - 64;
        s_rstep[u] = twiddle(a.tw, uint64_t(u) * uint64_t(L2 >= 4 ? (NT >> (L2 - 4)) : 0), l2 + 1);
    }
    ip_tw_fill<NT, L2>(s_tw, a.tw);
    // this thread's radix-16 group of stage 0 / the last DIT stage: class gvec, offset gj1
    const bool has_g = int(threadIdx.x) < (V << M_log);
    const int gvec = threadIdx.x >> M_log, gj1 = threadIdx.x & ((1 << M_log) - 1);
    // stage-0 twiddles w_{N2}^(gj1 k2) merged with this thread's four-step base w_{n'}^(row gj1)
    Tw16B t0;
    t0.load(a.tw, gj1, l2, twiddle(a.tw, uint64_t(gj1) * uint64_t(row), lt));
    // solve iteration space (positions pA of row A; Hermitian partner position pB of row B):
    //   non-self clusters: rank r takes pA in [r N2/2, (r+1) N2/2), partner N2-1-k2a -> pB = N2-1-pA
    //   row N1/2 (rank 1 of cluster 0): pA in [0, N2/2), same partner map
    //   row 0 (rank 0 of cluster 0): partner (N2 - k2a) mod N2 in the same row; every position,
    //   kept when k2a <= N2/2
    const bool row0 = selfrow && rank == 0;
    const int pbeg = (selfrow ? 0 : rank * (N2 / 2)), pend = row0 ? N2 : pbeg + N2 / 2;
    // real-FFT post-processing twiddle exp(-2 pi i k / n), k = rowA + N1 k2a: w_n^rowA w_{2N2}^k2a =
    // (per-thread base at the first position) x (per-CTA step table, s_rstep): no table walk per slot
    const double2 wrow = cmul(twiddle(a.tw, uint64_t(rowA), a.m),
                              twiddle(a.tw, uint64_t(IP::freq(pbeg + int(threadIdx.x)) & (N2 - 1)), l2 + 1));
    const double2* yp = a.yperm;
    // L2 prefetches (cp.async.bulk.prefetch.L2): this CTA's yhat rows (independent of L1), and —
    // after L1 — the exchange-block rows and yhat rows of the CTA one wave later on this SM
    // (local row li + 148: clusters launch in blockIdx order), so its load phase hits L2
    auto bulk_prefetch = [](const void* base, unsigned bytes) {
        for (unsigned off = 0; off < bytes; off += 32768u) {
            const unsigned n = bytes - off < 32768u ? bytes - off : 32768u;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(reinterpret_cast<const char*>(base) + off),
                         "r"(n)
                         : "memory");
        }
    };
    auto prefetch_yhat = [&](int lrow, int t, int side) {
        const int q2 = a.rank * a.QP + (lrow >> 1), rk = lrow & 1;
        const bool self2 = q2 == 0, row02 = self2 && rk == 0;
        const int r2 = lat_row_of(q2, rk, N1);
        const long long ra = self2 ? r2 : q2, rb = self2 ? r2 : N1 - q2;
        const int pb = self2 ? 0 : rk * (N2 / 2), pe = row02 ? N2 : pb + N2 / 2;
        const long long r0 = side ? rb : ra;
        const long long lo = side ? (row02 ? 0 : N2 - pe) : pb, hi = side ? (row02 ? N2 : N2 - pb) : pe;
        bulk_prefetch(yp + size_t(t) * half + (r0 << l2) + lo, unsigned((hi - lo) * sizeof(double2)));
    };
    constexpr int WAVE = 148;
    if (threadIdx.x < 2 * T) prefetch_yhat(li, threadIdx.x >> 1, threadIdx.x & 1);
    else if ((a.next_pf & 1) && threadIdx.x >= 64 && threadIdx.x < 64 + 2 * T && li + WAVE < a.R)
        prefetch_yhat(li + WAVE, (threadIdx.x - 64) >> 1, (threadIdx.x - 64) & 1);
    pdl_wait();
    pdl_trigger();
    if ((a.next_pf & 2) && a.lkc == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + a.nrank * V && li + WAVE < a.R) {
        const int sr = (threadIdx.x - 32) / V, oo = (threadIdx.x - 32) - sr * V;
        bulk_prefetch(a.Y + size_t(c) * a.V * a.half + xoff(a, sr, oo, li + WAVE, 0),
                      unsigned(a.WC * sizeof(double2)));
    }
    double2* const Yc = a.Y + size_t(c) * a.V * a.half;
    for (int e = threadIdx.x; e < (V << l2); e += NT) {
        const int oo = e >> l2, k2 = e & (N2 - 1);
        const int sr = k2 >> a.lwc;  // column owner
        cp_async16(&sm[oo * lds + S(k2)], &Yc[xoff_f(a, sr, oo, li, k2 & (a.WC - 1))]);
    }
    cp_async_wait_all();
    __syncthreads();
    if (has_g) {
        double2* xs = sm + gvec * lds + S(gj1);
        double2 x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = r ? cmul(xs[ip_off<M_log>(r)], s_ostep[r]) : xs[0];  // s_ostep[0] = 1
        reg_dft<16>(x, -1);
        t0.each0([&](int k2, double2 w) { x[brev_c<16>(k2)] = cmul(x[brev_c<16>(k2)], w); });
#pragma unroll
        for (int r = 0; r < 16; ++r) xs[ip_off<M_log>(brev_c<16>(r))] = x[r];
    }
    __syncthreads();
    ip_mid_stages<NT, L2, false, true, true>(sm, V, lds, a.tw, s_tw);  // warp-local after stage 0 (ipfft.cuh)
    ip_tail_stage<NT, L2, true>(sm, V, lds, -1);
    cl.sync();  // both rows transformed: partner rows readable over DSMEM

    double2* rem = cl.map_shared_rank(sm, rank ^ 1);
    double2* bufA = (selfrow || rank == 0) ? sm : rem;
    double2* bufB = (selfrow || rank == 1) ? sm : rem;
    const bool grad = a.want_grad != 0;
    double acc[2 + P];
#pragma unroll
    for (int x = 0; x < 2 + P; ++x) acc[x] = 0.0;
    double imx[T], rex[T];
#pragma unroll
    for (int t = 0; t < T; ++t) imx[t] = rex[t] = 0.0;
    long long first_bad = 0x7f7f7f7fll;
    double lpm = 1.0;  // running pivot product of the slots k >= 1 (weight 2): one log per thread
    int lpe = 0;
    auto partner = [&](int pA, int k2a, int& k2b) {
        if (row0) {
            k2b = (N2 - k2a) & (N2 - 1);
            return IP::pos(k2b);
        }
        k2b = N2 - 1 - k2a;
        return N2 - 1 - pA;
    };
#if LAT_L2_PAIRFORM
    // Main loop of every cluster but q = 0 (no packed slot 0, no self-paired slot): both sides of a
    // Hermitian pair in one pass.  With S = za + conj(zb), D = za - conj(zb), w = exp(-2 pi i k / n):
    //   2 H(k) = S - i w D,   2 H(N' - k) = conj(S) - i conj(w) conj(D)   (r2c_post of both sides),
    // and for the class adjoints ZA, ZB (computed with half weights): E = ZA + conj(ZB),
    // D' = ZA - conj(ZB), O = D' conj(w): z(k) = E + i O, z(N' - k) = conj(E) + i conj(O) (c2r_pre
    // of both sides) — 12 fp64 operations per class each instead of 2 x 14.  The factors 1/2 move
    // into the per-pair tables (s_coefh, s_wRh) and the Parseval weight 2.
    if (!selfrow) {
        double hmax = 0.0;  // T = 2: max |Im 2H| of the diagonal class (both diagonal entries scale it)
#pragma unroll(LAT_UNROLL_V)
        for (int pA = pbeg + int(threadIdx.x), it = 0; pA < pend; pA += NT, ++it) {
            const int k2a = IP::freq(pA), pB = N2 - 1 - pA, k2b = N2 - 1 - k2a;
            double2 rA[T], rB[T];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                rA[t] = yp[size_t(t) * half + ((long long)rowA << l2) + pA];
                rB[t] = yp[size_t(t) * half + ((long long)rowB << l2) + pB];
            }
            const double2 w = cmul(wrow, s_rstep[it]);
            double2 HA[P], HB[P];
            auto post2 = [&](int o, double2& ha, double2& hb) {
                const double2 za = bufA[o * lds + S(pA)], zb = bufB[o * lds + S(pB)];
                const double Sx = za.x + zb.x, Sy = za.y - zb.y, Dx = za.x - zb.x, Dy = za.y + zb.y;
                const double P1 = fma(w.x, Dy, w.y * Dx), P2 = fma(w.y, Dy, -(w.x * Dx));
                ha = make_double2(Sx + P1, Sy + P2);
                hb = make_double2(Sx - P1, P2 - Sy);
            };
            if constexpr (DIST) {
                double2 ca[P - T + 1], cb[P - T + 1];
#pragma unroll
                for (int o = 0; o < P - T + 1; ++o) post2(o, ca[o], cb[o]);
#pragma unroll
                for (int x = 0; x < P; ++x) HA[x] = ca[cls_distinct<T>(x)], HB[x] = cb[cls_distinct<T>(x)];
            } else {
#pragma unroll
                for (int x = 0; x < P; ++x) post2(s_cls[x], HA[x], HB[x]);
            }
            if constexpr (T == 2) hmax = fmax(hmax, fmax(fabs(HA[0].y), fabs(HB[0].y)));
            double2 ZA[P], ZB[P];
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const double2* H = side == 0 ? HA : HB;
                double2 A[P], r[T], ch[T], Ai[P];
#pragma unroll
                for (int x = 0; x < P; ++x)
                    A[x] = make_double2(fma(s_coefh[x], H[x].x, s_xi[x]), s_coefh[x] * H[x].y);
#pragma unroll
                for (int t = 0; t < T; ++t) r[t] = side == 0 ? rA[t] : rB[t];
                double qd;
                int st;
                if constexpr (T == 2) st = herm2_solve<false>(A, r, lpm, lpe, qd, ch, Ai, imx, rex);
                else st = ldl_core<T, true>(A, r, grad, lpm, lpe, qd, ch, Ai, imx, rex);
                if (st == 1) {
                    const long long sl = side == 0 ? ((long long)rowA << l2) + k2a : ((long long)rowB << l2) + k2b;
                    if (sl < first_bad) first_bad = sl;
                }
                acc[1] += 2.0 * qd;  // slot k >= 1 stands for frequencies k and n - k
                if (grad) {
                    // M = A^-1 - chat chat^H; its diagonal is real (Im = 0 exactly, not a rounding residue)
                    double2 Mq[P];
                    int x = 0;
#pragma unroll
                    for (int i = 0; i < T; ++i)
#pragma unroll
                        for (int j = i; j < T; ++j, ++x) {
                            if (i == j) Mq[x] = make_double2(Ai[x].x - fma(ch[i].x, ch[i].x, ch[i].y * ch[i].y), 0.0);
                            else Mq[x] = csub(Ai[x], cmulc(ch[i], ch[j]));
                        }
                    x = 0;
#pragma unroll
                    for (int i = 0; i < T; ++i)
#pragma unroll
                        for (int j = i; j < T; ++j, ++x) {  // H holds 2 H: the Parseval weight 2
                            if (i == j) acc[2 + x] = fma(Mq[x].x, H[x].x, acc[2 + x]);
                            else acc[2 + x] += Mq[x].x * H[x].x + Mq[x].y * H[x].y;
                        }
#pragma unroll
                    for (int o = 0; o < P; ++o) {
                        double2 z = make_double2(0.0, 0.0);
#pragma unroll
                        for (int y = 0; y < P; ++y)
                            if (cls(y) == o) {
                                z.x = fma(s_wRh[y], Mq[y].x, z.x);
                                if (!pair_is_diag<T>(y)) z.y = fma(s_wRh[y], Mq[y].y, z.y);
                            }
                        if (side == 0) ZA[o] = z;
                        else ZB[o] = z;
                    }
                }
            }
            if (grad) {
#pragma unroll
                for (int o = 0; o < P; ++o) {
                    if (o >= V) break;
                    if (DIST && o == 0) {  // class 0 = the diagonal pairs: a real adjoint (5 operations)
                        const double Ex = ZA[0].x + ZB[0].x, Dx = ZA[0].x - ZB[0].x, Ox = Dx * w.x;
                        bufA[S(pA)] = make_double2(fma(Dx, w.y, Ex), Ox);
                        bufB[S(pB)] = make_double2(fma(-Dx, w.y, Ex), Ox);
                        continue;
                    }
                    const double Ex = ZA[o].x + ZB[o].x, Ey = ZA[o].y - ZB[o].y;
                    const double Dx = ZA[o].x - ZB[o].x, Dy = ZA[o].y + ZB[o].y;
                    const double Ox = fma(Dx, w.x, Dy * w.y), Oy = fma(Dy, w.x, -(Dx * w.y));
                    bufA[o * lds + S(pA)] = make_double2(Ex - Oy, Ey + Ox);
                    bufB[o * lds + S(pB)] = make_double2(Ex + Oy, Ox - Ey);
                }
            }
        }
        if constexpr (T == 2) {
            imx[0] = fmax(imx[0], fabs(s_coefh[0]) * hmax);
            imx[1] = fmax(imx[1], fabs(s_coefh[2]) * hmax);
        }
    }
#endif
#pragma unroll 1
    for (int pA = pbeg + int(threadIdx.x), it = 0; pA < pend; pA += NT, ++it) {
        if (LAT_L2_PAIRFORM && !selfrow) break;  // done above
        const int k2a = IP::freq(pA);
        if (row0 && k2a > N2 / 2) continue;  // its partner's thread owns the pair
        int k2b;
        const int pB = partner(pA, k2a, k2b);
        const long long kA = rowA + ((long long)k2a << l1);
        const long long slA = ((long long)rowA << l2) + k2a, slB = ((long long)rowB << l2) + k2b;
        double2 rA[T], rB[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            rA[t] = yp[size_t(t) * half + ((long long)rowA << l2) + pA];
            rB[t] = yp[size_t(t) * half + ((long long)rowB << l2) + pB];
        }
        if (kA == 0) {
            // packed slot 0: frequency 0 (.x) and Nyquist (.y), two real systems; tau zeroes the
            // frequency-0 residual (gp_core.cpp:67-88) — k_solve_class's p == 0 branch
            double H0[P], HN[P], A0[P], AN[P], r0[T], rN[T], c0v[T], cN[T], I0[P], IN[P], l0, lN, q0, qN;
#pragma unroll
            for (int x = 0; x < P; ++x) {
                const double2 z = sm[cls(x) * lds + S(0)];
                H0[x] = z.x + z.y;
                HN[x] = z.x - z.y;
                A0[x] = fma(s_coef[x], H0[x], s_xi[x]);
                AN[x] = fma(s_coef[x], HN[x], s_xi[x]);
            }
#pragma unroll
            for (int t = 0; t < T; ++t) r0[t] = 0.0, rN[t] = rA[t].y;
            const int st0 = ldl_solve<T, false>(A0, r0, grad, l0, q0, c0v, I0, imx, rex);
            const int stN = ldl_solve<T, false>(AN, rN, grad, lN, qN, cN, IN, imx, rex);
            if (st0 == 1 || stN == 1) first_bad = 0;
            acc[0] += l0 + lN;
            acc[1] += q0 + qN;
            if (grad) {
                double M0[P], MN[P];
                int x = 0;
#pragma unroll
                for (int i = 0; i < T; ++i)
#pragma unroll
                    for (int j = i; j < T; ++j, ++x) {
                        M0[x] = I0[x] - c0v[i] * c0v[j];
                        MN[x] = IN[x] - cN[i] * cN[j];
                    }
#pragma unroll
                for (int y = 0; y < P; ++y) acc[2 + y] += M0[y] * H0[y] + MN[y] * HN[y];
#pragma unroll
                for (int o = 0; o < P; ++o) {
                    if (o >= V) break;
                    double z0 = 0.0, zN = 0.0;
#pragma unroll
                    for (int y = 0; y < P; ++y)
                        if (cls(y) == o) z0 = fma(s_wR[y], M0[y], z0), zN = fma(s_wR[y], MN[y], zN);
                    sm[o * lds + S(0)] = make_double2(0.5 * (z0 + zN), 0.5 * (z0 - zN));  // inverse pre, k = 0
                }
            }
            continue;
        }
        const bool self = slA == slB;  // k = N'/2 (row 0, k2 = N2/2)
        const double2 wA = cmul(wrow, s_rstep[it]);  // exp(-2 pi i k / n), k = rowA + N1 k2a
        const double2 wB = make_double2(-wA.x, wA.y);          // exp(-2 pi i (N' - k)/n) = -conj(wA)
        double2 HA[P], HB[P];
#pragma unroll
        for (int x = 0; x < P; ++x) {
            const int o = cls(x);
            const double2 za = bufA[o * lds + S(pA)], zb = bufB[o * lds + S(pB)];
            HA[x] = r2c_post(za, zb, wA);
            HB[x] = r2c_post(zb, za, wB);
        }
        double2 ZA[P], ZB[P];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            if (side == 1 && self) break;
            const double2* H = side == 0 ? HA : HB;
            const long long sl = side == 0 ? slA : slB;
            double2 A[P], r[T], ch[T], Ai[P];
#pragma unroll
            for (int x = 0; x < P; ++x) A[x] = make_double2(fma(s_coef[x], H[x].x, s_xi[x]), s_coef[x] * H[x].y);
#pragma unroll
            for (int t = 0; t < T; ++t) r[t] = side == 0 ? rA[t] : rB[t];
            double qd;
            int st;
            if constexpr (T == 2) st = herm2_solve(A, r, lpm, lpe, qd, ch, Ai, imx, rex);
            else st = ldl_core<T, true>(A, r, grad, lpm, lpe, qd, ch, Ai, imx, rex);
            if (st == 1 && sl < first_bad) first_bad = sl;
            acc[1] += 2.0 * qd;  // slot k >= 1 stands for frequencies k and n - k
            if (grad) {
                double2 Mq[P];
                int x = 0;
#pragma unroll
                for (int i = 0; i < T; ++i)
#pragma unroll
                    for (int j = i; j < T; ++j, ++x) Mq[x] = csub(Ai[x], cmulc(ch[i], ch[j]));
#pragma unroll
                for (int y = 0; y < P; ++y) acc[2 + y] += 2.0 * (Mq[y].x * H[y].x + Mq[y].y * H[y].y);
#pragma unroll
                for (int o = 0; o < P; ++o) {
                    double2 z = make_double2(0.0, 0.0);
#pragma unroll
                    for (int y = 0; y < P; ++y)
                        if (cls(y) == o) z = make_double2(fma(s_wR[y], Mq[y].x, z.x), fma(s_wR[y], Mq[y].y, z.y));
                    if (side == 0) ZA[o] = z;
                    else ZB[o] = z;
                }
            }
        }
        if (grad) {
            // inverse real-FFT pre-processing of the class adjoints, written back in place
#pragma unroll
            for (int o = 0; o < P; ++o) {
                if (o >= V) break;
                if (self) {
                    bufA[o * lds + S(pA)] = c2r_pre(ZA[o], ZA[o], wA);
                } else {
                    bufA[o * lds + S(pA)] = c2r_pre(ZA[o], ZB[o], wA);
                    bufB[o * lds + S(pB)] = c2r_pre(ZB[o], ZA[o], wB);
                }
            }
        }
    }
    cl.sync();  // every DSMEM access of the cluster is done
    acc[0] += 2.0 * log_of(lpm, lpe);

    __shared__ double redv[(NT / 32) * (2 + P)];
    block_sum_vec<NT, 2 + P>(acc, redv);
    if (threadIdx.x == 0) {
        double* pm = a.part_mid + (size_t(c) * a.R + li) * (2 + P);
#pragma unroll
        for (int x = 0; x < 2 + P; ++x) pm[x] = acc[x];
    }
    if (first_bad != 0x7f7f7f7fll) atomicMin(a.bad + c, int(first_bad));
#pragma unroll
    for (int t = 0; t < T; ++t) {
        double vi = imx[t], vr = rex[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            vi = fmax(vi, __shfl_xor_sync(0xffffffffu, vi, o));
            vr = fmax(vr, __shfl_xor_sync(0xffffffffu, vr, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMax(a.imre + ((size_t)c * MAXT + t) * 2 + 0, (unsigned long long)__double_as_longlong(vi));
            atomicMax(a.imre + ((size_t)c * MAXT + t) * 2 + 1, (unsigned long long)__double_as_longlong(vr));
        }
    }
    if (!grad) return;
    // inverse row FFT (block_sum_vec's barriers ordered the solve's writes): DIT tail, middle
    // stages, then stage 0 fused with the conjugate four-step twiddle and the store
    ip_tail_stage<NT, L2, (IP::A16 > 1)>(sm, V, lds, +1);  // warp-local unless stage 0 follows
    ip_mid_stages<NT, L2, true, true, true>(sm, V, lds, a.tw, s_tw);
    if (has_g) {
        t0.load(a.tw, gj1, l2, twiddle(a.tw, uint64_t(gj1) * uint64_t(row), lt));
        const double2* xs = sm + gvec * lds + S(gj1);
        double2 x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = xs[ip_off<M_log>(r)];
        t0.each0([&](int k2, double2 w) { x[k2] = cmulc(x[k2], w); });  // conj of the merged twiddles
        reg_dft<16>(x, +1);
        double2* const Yo = (a.Yout ? a.Yout : a.Y) + size_t(c) * a.V * a.half;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int j2 = gj1 + (brev_c<16>(r) << M_log);
            Yo[xoff_r(a, j2 >> a.lwc, gvec, li, j2 & (a.WC - 1))] = r ? cmulc(x[r], s_ostep[brev_c<16>(r)]) : x[0];
        }
    }
}

// ------------------------------------------------------------------ L3: inverse column FFT -> gradient dot
// In-place DIT: the tail stage is fused with the exchange-block loads, stage 0 with the
// gradient dot (W(2j) = 2 Re z, W(2j+1) = 2 Im z consumed in registers).
template <int NT, int DC, int ALPHA, int L1>
__global__ void __launch_bounds__(NT) k_lat_col_inv(LatArgs a, int l2, int lc) {
    using IP = Ip<L1>;
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    __shared__ int s_last;
    __shared__ double redv[(NT / 32) * DC];
    constexpr int N1 = 1 << L1, ld = padded_len(N1);
    constexpr int M_log = L1 - 4;
    // thread -> column vec; tail chunk p0 .. p0+15 and stage-0 group j1 of that column
    const int vec = threadIdx.x >> M_log, j1 = threadIdx.x & ((1 << M_log) - 1), p0 = j1 << 4;
    const int kb = IP::freq(p0);
    Tw16 t0;  // held across tiles (reloading it per tile measured 1.26 vs 1.13 ms)
    t0.load(a.tw, j1, L1);
    const int ntiles = a.ncb * a.V * a.nc;
    // the tail stage's inputs of a tile: 16 scattered exchange-block elements per thread, copied
    // asynchronously into this thread's chunk of smem (frequency kb | freq_lo(r) at position p0 + r)
    auto issue = [&](int tile) {
        const int bx = tile % a.ncb, v = tile / a.ncb, c = v / a.V, o = v - c * a.V;
        const int jl = ((a.rank * a.ncb + bx) << lc) + vec - a.rank * a.WC;
        const double2* Cc = a.Cbuf + size_t(c) * a.V * a.half;
        double2* xs = sm + vec * ld + S(p0);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            int i;
            const int h = row_owner(kb | IP::freq_lo(r), N1, a.lqp, i);
            cp_async16(xs + r, &Cc[xoff_r(a, h, o, i, jl)]);
        }
    };
    // gradient-dot partials: one slot per (candidate x class, CTA), accumulated in registers over
    // the CTA's consecutive tiles of that class (tiles are ordered class-major) and reduced across
    // the CTA once per run; slots of runs this CTA has no tile of are written as zeros
    const int nslot = int(gridDim.x);
    double acc[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) acc[j] = 0.0;
    int vcur = -1;
    auto slot = [&](int vv) { return a.part_dot + (size_t(vv) * nslot + blockIdx.x) * (MAXD + 1); };
    bool prodrun = false;  // the current run accumulates in product form (same candidate: CTA-uniform)
    auto flush = [&](int vv) {
        block_sum_vec<NT, DC>(acc, redv);
        if (threadIdx.x == 0) {
            double* out = slot(vv);
#pragma unroll
            for (int j = 0; j < DC; ++j)
                if (j < a.d) out[j] = prodrun ? 2.0 * acc[j] * LatGen<DC, ALPHA>::dscale(a, vv / a.V, j) : acc[j];
        }
        prodrun = false;
#pragma unroll
        for (int j = 0; j < DC; ++j) acc[j] = 0.0;
    };
    auto zero_slots = [&](int v0, int v1) {
        if (threadIdx.x == 0)
            for (int vv = v0; vv < v1; ++vv)
                for (int j = 0; j < a.d; ++j) slot(vv)[j] = 0.0;
    };
    pdl_wait();
    if (int(blockIdx.x) < ntiles) issue(blockIdx.x);
    // persistent over tiles: the next tile's loads run under this tile's gradient dot
#pragma unroll 1
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int bx = tile % a.ncb, v = tile / a.ncb, c = v / a.V, o = v - c * a.V;
        const uint32_t c0 = uint32_t(a.rank * a.ncb + bx) << lc;  // global first column
        double2 x[16];
        cp_async_wait_all();
        {
            double2* xs = sm + vec * ld + S(p0);
#pragma unroll
            for (int r = 0; r < 16; ++r) x[r] = xs[r];
            tail_regs<L1>(x, +1);
#pragma unroll
            for (int r = 0; r < 16; ++r) xs[tail_out_pos<L1>(r)] = x[r];
        }
        __syncthreads();  // (warp-local barriers here measured slower: the kernel spills)
        ip_mid_stages<NT, L1, true>(sm, 1 << lc, ld, a.tw);
        {
            const double2* xs = sm + vec * ld + S(j1);
#pragma unroll
            for (int r = 0; r < 16; ++r) x[r] = xs[ip_off<M_log>(r)];
        }
        __syncthreads();  // smem free: start the next tile's loads
        if (tile + int(gridDim.x) < ntiles) issue(tile + gridDim.x);
        dit16_regs(x, t0);
        if (v != vcur) {  // CTA-uniform: a new (candidate, class) run starts
            if (vcur >= 0) flush(vcur);
            zero_slots(vcur + 1, v);
            vcur = v;
        }
        {
            LatGen<DC, ALPHA> G;
#if LAT_GEN_PROD
            // product form (LatGen::init_prod): the run's sums are unscaled, flush applies dscale
            if (G.init_prod(a, c, o)) {
                prodrun = true;
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t J = (uint32_t(j1 + (brev_c<16>(r) << M_log)) << l2) + c0 + uint32_t(vec);
                    G.dq_acc_prod(2u * J, x[r].x, acc);  // W(2j) = 2 Re z, W(2j+1) = 2 Im z: the 2 is in flush
                    G.dq_acc_prod(2u * J + 1u, x[r].y, acc);
                }
            } else
#endif
            {
                G.init(a, c, o);
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t J = (uint32_t(j1 + (brev_c<16>(r) << M_log)) << l2) + c0 + uint32_t(vec);
                    G.dq_acc(2u * J, 2.0 * x[r].x, acc);  // W(2j) = 2 Re z, W(2j+1) = 2 Im z
                    G.dq_acc(2u * J + 1u, 2.0 * x[r].y, acc);
                }
            }
        }
    }
    if (vcur >= 0) flush(vcur);
    zero_slots(vcur + 1, a.V * a.nc);
    // last-CTA reduction (one acq_rel ticket per CTA; thread 0 wrote every slot of this CTA), fixed order
    if (threadIdx.x == 0) {
        const unsigned ticket = atom_add_acq_rel_gpu(a.counter, 1u);
        s_last = ticket == gridDim.x - 1;
        if (s_last) a.counter[0] = 0;  // self-reset for the next replay
    }
    __syncthreads();
    if (s_last) {
#pragma unroll 1
        for (int c = 0; c < a.nc; ++c) {
            ClassSums t{};
            t.T = a.T;
            t.P = a.P;
            t.V = a.V;
            t.d = a.d;
            t.nrows = a.R;  // L2 CTAs per candidate on this rank
            t.nblk = nslot;
            t.dstride = MAXD + 1;
            t.mid = a.part_mid + size_t(c) * t.nrows * (2 + a.P);
            t.dot = a.part_dot + size_t(c) * a.V * nslot * (MAXD + 1);
            t.pair_a = a.pair_a;
            t.pair_b = a.pair_b;
            t.Rpair = a.Rpair + size_t(c) * a.P;
            t.gamma = __ldg(a.gamma + c);
            t.out = a.out + size_t(c) * NOUT;
            class_sums_out<NT>(t);
        }
    }
}

// ------------------------------------------------------------------ launchers (per length)
template <class K>
static void set_smem_lat(K kern, size_t bytes) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

inline int lat_sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// column-kernel cluster size (lattice_kernels.cuh k_lat_col_*): K adjacent column blocks per
// cluster, row segments of K * C * 16 bytes; FMTGP_LAT_CLUSTER overrides (1, 2 or 4)
inline int lat_cluster_k(int ncb) {
    static int k = [] {
        const char* e = std::getenv("FMTGP_LAT_CLUSTER");
        const int v = e ? std::atoi(e) : 4;
        return v >= 4 ? 4 : v >= 2 ? 2 : 1;
    }();
    int K = k;
    while (K > 1 && (ncb % K) != 0) K >>= 1;
    return K;
}

template <class Kern, class... Args>
static cudaError_t launch_cluster(Kern kern, int grid, int K, size_t smem, cudaStream_t s, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(LAT_NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(K);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// persistent grid: as many whole clusters as fit at once (one CTA per SM: the tile fills smem)
template <class Kern>
static int lat_cluster_grid(Kern kern, int K, size_t smem, int tiles) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(K * 64));
    cfg.blockDim = dim3(LAT_NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(K);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, kern, &cfg) != cudaSuccess || nclus <= 0) {
        cudaGetLastError();
        nclus = lat_sm_count() / K;
    }
    return K * std::max(1, std::min(nclus, tiles));
}

template <int DC, int ALPHA, int L1>
static void lat_cols(const LatGeo& g, const LatArgs& a, size_t sm_col, bool inverse, cudaStream_t s) {
    const int nb = a.chunk >= 0 ? a.ncb >> a.lkc : a.ncb;  // column blocks of this launch
    const int K = lat_cluster_k(nb);
    const int tiles = (nb / K) * a.V * a.nc;
    if (!inverse) {
        auto k = k_lat_col_fwd<LAT_NT, DC, ALPHA, L1>;
        set_smem_lat(k, sm_col);
        if (K > 1) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        ProfScope ps("lat_col_fwd", s);
        CK_LAUNCH(launch_cluster(k, lat_cluster_grid(k, K, sm_col, tiles), K, sm_col, s, false, a, g.l2, g.lc));
    } else {
        // inverse: no cluster (the next tile's scattered loads are asynchronous copies that run
        // under the gradient dot; a DSMEM-transposed variant measured slower)
        auto k = k_lat_col_inv<LAT_NT, DC, ALPHA, L1>;
        set_smem_lat(k, sm_col);
        ProfScope ps("lat_col_inv", s);
        const int grid = std::min(std::min(a.ncb * a.V * a.nc, lat_sm_count()), LAT_MAX_INV_GRID);
        CK_LAUNCH(launch_cluster(k, grid, 1, sm_col, s, true, a, g.l2, g.lc));
    }
}

template <int ALPHA, int L1>
static void lat_cols_d(const LatGeo& g, const LatArgs& a, size_t sm_col, bool inverse, cudaStream_t s) {
    if (a.d <= 2) lat_cols<2, ALPHA, L1>(g, a, sm_col, inverse, s);
    else if (a.d <= 4) lat_cols<4, ALPHA, L1>(g, a, sm_col, inverse, s);
    else if (a.d <= 8) lat_cols<8, ALPHA, L1>(g, a, sm_col, inverse, s);
    else lat_cols<16, ALPHA, L1>(g, a, sm_col, inverse, s);
}

template <int L1>
void lat_cols_launch(const LatGeo& g, const LatArgs& a, bool inverse, cudaStream_t s) {
    const size_t sm_col = size_t(1 << g.lc) * padded_len(1 << L1) * sizeof(double2);
    if (a.si_alpha == 1) lat_cols_d<1, L1>(g, a, sm_col, inverse, s);
    else lat_cols_d<2, L1>(g, a, sm_col, inverse, s);
}

template <int T, int L2>
static void lat_mid_t(const LatGeo& g, const LatArgs& a, cudaStream_t s) {
    const size_t sm = size_t(a.V) * padded_len(1 << L2) * sizeof(double2);
    auto k = a.distinct ? k_lat_mid<LAT_NT, T, true, L2> : k_lat_mid<LAT_NT, T, false, L2>;
    set_smem_lat(k, sm);
    ProfScope ps("lat_mid", s);
    const int rows = a.chunk >= 0 ? a.R >> a.lkc : a.R;
    CK_LAUNCH(launch_pdl(k, dim3(unsigned(rows), a.nc), dim3(LAT_NT), sm, s, true, a, g.l1));
}

template <int L2>
void lat_mid_launch(const LatGeo& g, const LatArgs& a, cudaStream_t s) {
    switch (a.T) {
        case 1: lat_mid_t<1, L2>(g, a, s); break;
        case 2: lat_mid_t<2, L2>(g, a, s); break;
        case 3: lat_mid_t<3, L2>(g, a, s); break;
        default: lat_mid_t<4, L2>(g, a, s); break;
    }
}

}  // namespace fmtgp
