// Device kernels of the fast-MTGP fit path (sm_100a, fp64).  See passes.cuh for the
// transform conventions and kernels.cuh for the launch API.
#include <climits>
#include <mutex>
#include <utility>
#include <vector>

#include "kernels.cuh"

namespace fmtgp {

thread_local Profiler* g_prof = nullptr;

// ============================================================================ twiddles
__global__ void k_init_twiddles(double2* tab) {
    const int L = blockIdx.y;
    const int cnt = L <= TW_BASE_LOG ? (1 << L) : (1 << TW_BASE_LOG);
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < cnt; u += gridDim.x * blockDim.x) {
        double s, c;
        // exp(-2 pi i u / 2^L) = cos(pi x) - i sin(pi x), x = 2u / 2^L (exact)
        sincospi(ldexp(double(u), 1 - L), &s, &c);
        tab[(size_t(L) << TW_BASE_LOG) + u] = make_double2(c, -s);
    }
}

void init_twiddles(double2* tab, cudaStream_t s) {
    k_init_twiddles<<<dim3(32, 27), 256, 0, s>>>(tab);
}

// Per-vector binding of a transform source: the column kernels call bind_src(src, v) once per
// CTA and the result per element, so sources can hoist per-vector constants into registers
// (QuerySrcLat below); by default the element call is src(v, idx).
template <class Src>
struct BoundSrc {
    const Src& s;
    int v;
    __device__ __forceinline__ double operator()(uint64_t idx) const { return s(v, idx); }
};
template <class Src>
__device__ __forceinline__ BoundSrc<Src> bind_src(const Src& s, int v) {
    return BoundSrc<Src>{s, v};
}

// ============================================================================ forward, single CTA
template <int NT, class Src, class Snk>
__global__ void __launch_bounds__(NT) k_fwd_small_lat(Src src, Snk snk, int m, const double2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.x;
    if (m == 0) {
        if (threadIdx.x == 0) snk.put(v, 0, make_double2(src(v, 0), 0.0));
        return;
    }
    const int lp = m - 1, Np = 1 << lp;
    const auto gen = bind_src(src, v);
    for (int e = threadIdx.x; e < Np; e += NT) sm[S(e)] = make_double2(gen(2ull * e), gen(2ull * e + 1));
    __syncthreads();
    smem_fft<NT, true>(sm, lp, 1, padded_len(Np), -1, tw);
    for (int k = threadIdx.x; k <= Np / 2; k += NT) {
        if (k == 0) {
            const double2 Z0 = sm[S(0)];
            snk.put(v, 0, make_double2(Z0.x + Z0.y, Z0.x - Z0.y));
            continue;
        }
        const int kp = Np - k;
        const double2 Zk = sm[S(k)], Zp = sm[S(kp)];
        snk.put(v, k, r2c_post(Zk, Zp, twiddle(tw, k, m)));
        if (kp != k) snk.put(v, kp, r2c_post(Zp, Zk, twiddle(tw, kp, m)));
    }
}

template <int NT, class Src, class Snk>
__global__ void __launch_bounds__(NT) k_fwd_small_dig(Src src, Snk snk, int m) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.x, n = 1 << m;
    for (int e = threadIdx.x; e < n; e += NT) sm[S(e)] = src(v, e);
    __syncthreads();
    smem_wht<NT, true>(sm, m, 1, padded_len(n));
    for (int e = threadIdx.x; e < n; e += NT) snk.put(v, e, sm[S(e)]);
}

// ============================================================================ forward, two pass
template <int NT, class Src>
__global__ void __launch_bounds__(NT) k_fwd_col_lat(Src src, double2* __restrict__ Y, int l1, int l2, int lc,
                                                    long long vstride, const double2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.y, C = 1 << lc, N1 = 1 << l1, ld = padded_len(N1);
    const long long c0 = (long long)blockIdx.x << lc;
    const auto gen = bind_src(src, v);
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int j1 = e >> lc, c = e & (C - 1);
        const uint64_t j = (uint64_t(j1) << l2) + c0 + c;
        sm[c * ld + S(j1)] = make_double2(gen(2 * j), gen(2 * j + 1));
    }
    __syncthreads();
    smem_fft<NT, true>(sm, l1, C, ld, -1, tw);
    double2* out = Y + v * vstride;
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int k1 = e >> lc, c = e & (C - 1);
        const uint64_t j2 = c0 + c;
        out[((long long)k1 << l2) + j2] = cmul(sm[c * ld + S(k1)], twiddle(tw, j2 * uint64_t(k1), l1 + l2));
    }
}

template <int NT, class Src>
__global__ void __launch_bounds__(NT) k_fwd_col_dig(Src src, double* __restrict__ Y, int l1, int l2, int lc,
                                                    long long vstride) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.y, C = 1 << lc, N1 = 1 << l1, ld = padded_len(N1);
    const long long c0 = (long long)blockIdx.x << lc;
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int j1 = e >> lc, c = e & (C - 1);
        sm[c * ld + S(j1)] = src(v, (uint64_t(j1) << l2) + c0 + c);
    }
    __syncthreads();
    smem_wht<NT, true>(sm, l1, C, ld);
    double* out = Y + v * vstride;
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int k1 = e >> lc, c = e & (C - 1);
        out[((long long)k1 << l2) + c0 + c] = sm[c * ld + S(k1)];
    }
}

__device__ __forceinline__ int row_of_cluster(int q, int rank, int N1) {
    if (q == 0) return rank == 0 ? 0 : N1 / 2;
    return rank == 0 ? q : N1 - q;
}

template <int NT, class Snk>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT)
    k_fwd_row_lat(const double2* __restrict__ Y, Snk snk, int l1, int l2, long long vstride, int m,
                  const double2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank());
    const int q = blockIdx.x >> 1, v = blockIdx.y;
    const int N1 = 1 << l1, N2 = 1 << l2;
    const int row = row_of_cluster(q, rank, N1);
    const double2* in = Y + v * vstride + ((long long)row << l2);
    for (int e = threadIdx.x; e < N2; e += NT) cp_async_el(&sm[S(e)], &in[e]);
    cp_async_wait_all();
    __syncthreads();
    smem_fft<NT, true>(sm, l2, 1, padded_len(N2), -1, tw);
    cl.sync();
    const bool self = (row == 0) || (row == N1 / 2);
    const double2* psm = self ? sm : cl.map_shared_rank(sm, rank ^ 1);
    for (int k2 = threadIdx.x; k2 < N2; k2 += NT) {
        const long long k = row + ((long long)k2 << l1);
        if (k == 0) {
            const double2 Z0 = sm[S(0)];
            snk.put(v, 0, make_double2(Z0.x + Z0.y, Z0.x - Z0.y));
            continue;
        }
        const int kc = (row == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
        snk.put(v, ((long long)row << l2) + k2, r2c_post(sm[S(k2)], psm[S(kc)], twiddle(tw, uint64_t(k), m)));
    }
    cl.sync();
}

template <int NT, class Snk>
__global__ void __launch_bounds__(NT) k_fwd_row_dig(const double* __restrict__ Y, Snk snk, int l2, long long vstride) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    constexpr auto S = sidx<true>;
    const int row = blockIdx.x, v = blockIdx.y, N2 = 1 << l2;
    const double* in = Y + v * vstride + ((long long)row << l2);
    for (int e = threadIdx.x; e < N2; e += NT) cp_async_el(&sm[S(e)], &in[e]);
    cp_async_wait_all();
    __syncthreads();
    smem_wht<NT, true>(sm, l2, 1, padded_len(N2));
    for (int e = threadIdx.x; e < N2; e += NT) snk.put(v, ((long long)row << l2) + e, sm[S(e)]);
}

// ============================================================================ generator / gradient-dot (split mode)
// One element per thread per sweep: for small problems the generator, not the transform,
// sets the parallelism.  Compile-time dimension D keeps kappa / dq / accumulators in
// registers.  Digital z_i comes from two 32-entry XOR tables per dimension in smem, X3 of
// the order-4 Walsh kernel from an 8-bit table.
constexpr int GEN_NT = 256;
constexpr int GEN_EPT = 4;  // elements per thread per block (dot kernel partial count)

// out[v][idx] = gamma prod_j (1 + eta_j kappa_j) in transform-input order
template <int D>
__global__ void __launch_bounds__(GEN_NT) k_gen_fill(GenSrc g, double* __restrict__ out, long long n) {
    __shared__ GenSmem<D> t;
    const int v = blockIdx.y;
    int p, c;
    g.coords(v, p, c);
    gen_smem_init<D>(t, g, c);
    uint64_t off[D];
#pragma unroll
    for (int j = 0; j < D; ++j) off[j] = __ldg(g.offs + size_t(p) * MAXD + j);
    const double gam = __ldg(g.gamma + c);
    __syncthreads();
    for (long long idx = blockIdx.x * (long long)GEN_NT + threadIdx.x; idx < n; idx += (long long)gridDim.x * GEN_NT) {
        double kappa[D];
        kappa_d<D>(g, t, off, idx, kappa);
        out[v * n + idx] = product_kernel_d<D, false>(kappa, t.eta, gam, nullptr);
    }
}

// partial[v][blk][.] = sum_idx W(idx) * (dq/deta_j, q)  (W already in transform-input order)
template <int D>
__global__ void __launch_bounds__(GEN_NT) k_gen_dot(GradSink gs, const double* __restrict__ W, long long n) {
    __shared__ GenSmem<D> t;
    __shared__ double red[32];
    const GenSrc& g = gs.gen;
    const int v = blockIdx.y;
    int p, c;
    g.coords(v, p, c);
    gen_smem_init<D>(t, g, c);
    uint64_t off[D];
#pragma unroll
    for (int j = 0; j < D; ++j) off[j] = __ldg(g.offs + size_t(p) * MAXD + j);
    const double gam = __ldg(g.gamma + c);
    __syncthreads();
    double acc[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) acc[j] = 0.0;
    for (long long idx = blockIdx.x * (long long)GEN_NT + threadIdx.x; idx < n; idx += (long long)gridDim.x * GEN_NT) {
        double kappa[D], dq[D];
        kappa_d<D>(g, t, off, idx, kappa);
        const double q = product_kernel_d<D, true>(kappa, t.eta, gam, dq);
        const double w = W[v * n + idx];
#pragma unroll
        for (int j = 0; j < D; ++j) acc[j] = fma(w, dq[j], acc[j]);
        acc[D] = fma(w, q, acc[D]);
    }
    double* out = gs.partial + ((size_t)v * gs.nblk + blockIdx.x) * (MAXD + 1);
#pragma unroll
    for (int j = 0; j <= D; ++j) {
        const double s = block_sum<GEN_NT>(acc[j], red);
        if (threadIdx.x == 0) out[j == D ? MAXD : j] = s;
    }
}

// ============================================================================ inverse sinks (device side)
struct GradAcc {
    double a[MAXD + 1];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i <= MAXD; ++i) a[i] = 0.0;
    }
};

__device__ __forceinline__ void grad_add(const GradSink& gs, int v, uint64_t idx, double W, GradAcc& acc) {
    int p, c;
    gs.gen.coords(v, p, c);
    double kappa[MAXD], dq[MAXD];
    gs.gen.kappa_all(p, idx, kappa);
    const int d = gs.gen.sp.d;
    const double q = product_kernel<true>(kappa, gs.gen.eta + size_t(c) * d, d, __ldg(gs.gen.gamma + c), dq);
#pragma unroll
    for (int j = 0; j < MAXD; ++j)
        if (j < d) acc.a[j] = fma(W, dq[j], acc.a[j]);
    acc.a[MAXD] = fma(W, q, acc.a[MAXD]);
}

template <int NT>
__device__ void grad_flush(const GradSink& gs, int v, int blk, GradAcc& acc) {
    __shared__ double red[32];
    const int d = gs.gen.sp.d;
    double* out = gs.partial + ((size_t)v * gs.nblk + blk) * (MAXD + 1);
#pragma unroll
    for (int j = 0; j <= MAXD; ++j) {
        if (j < d || j == MAXD) {
            const double s = block_sum<NT>(acc.a[j], red);
            if (threadIdx.x == 0) out[j] = s;
        }
    }
}

struct SinkGrad {  // fused dot (large problems)
    using Acc = GradAcc;
    GradSink gs;
    int lattice, m;
    __device__ __forceinline__ void lat(int v, uint64_t j, double2 z, GradAcc& acc) const {
        if (m == 0) {
            grad_add(gs, v, 0, z.x, acc);
            return;
        }
        grad_add(gs, v, 2 * j, 2.0 * z.x, acc);
        grad_add(gs, v, 2 * j + 1, 2.0 * z.y, acc);
    }
    __device__ __forceinline__ void dig(int v, uint64_t j, double w, GradAcc& acc) const { grad_add(gs, v, j, w, acc); }
    template <int NT>
    __device__ __forceinline__ void flush(int v, int blk, GradAcc& acc) const {
        grad_flush<NT>(gs, v, blk, acc);
    }
};

template <int DC>
struct GradAccD {
    double a[DC + 1];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i <= DC; ++i) a[i] = 0.0;
    }
};

// Fused gradient dot with DC-sized register arrays (large problems).
template <int DC>
struct SinkGradD {
    GradSink gs;
    int lattice, m;
    using Acc = GradAccD<DC>;
    __device__ __forceinline__ void add(int v, uint64_t idx, double W, Acc& acc) const {
        int p, c;
        gs.gen.coords(v, p, c);
        double kappa[DC], dq[DC];
        GenSrcD<DC>{gs.gen}.kappa_c(p, idx, kappa);
        const int d = gs.gen.sp.d;
        const double q = product_kernel_c<DC>(kappa, gs.gen.eta + size_t(c) * d, d, __ldg(gs.gen.gamma + c), dq, true);
#pragma unroll
        for (int j = 0; j < DC; ++j)
            if (j < d) acc.a[j] = fma(W, dq[j], acc.a[j]);
        acc.a[DC] = fma(W, q, acc.a[DC]);
    }
    __device__ __forceinline__ void lat(int v, uint64_t j, double2 z, Acc& acc) const {
        if (m == 0) {
            add(v, 0, z.x, acc);
            return;
        }
        add(v, 2 * j, 2.0 * z.x, acc);
        add(v, 2 * j + 1, 2.0 * z.y, acc);
    }
    __device__ __forceinline__ void dig(int v, uint64_t j, double w, Acc& acc) const { add(v, j, w, acc); }
    template <int NT>
    __device__ __forceinline__ void flush(int v, int blk, Acc& acc) const {
        __shared__ double redv[(NT / 32) * (DC + 1)];
        block_sum_vec<NT, DC + 1>(acc.a, redv);
        if (threadIdx.x == 0) {
            double* out = gs.partial + ((size_t)v * gs.nblk + blk) * (MAXD + 1);
            const int d = gs.gen.sp.d;
            for (int j = 0; j < d; ++j) out[j] = acc.a[j];
            out[MAXD] = acc.a[DC];
        }
    }
};

struct SinkStoreW {  // W in transform-input order for k_gen_dot (small problems)
    using Acc = GradAcc;
    double* W;
    long long n;
    int m;
    __device__ __forceinline__ void lat(int v, uint64_t j, double2 z, GradAcc&) const {
        double* o = W + v * n;
        if (m == 0) {
            o[0] = z.x;
            return;
        }
        o[2 * j] = 2.0 * z.x;
        o[2 * j + 1] = 2.0 * z.y;
    }
    __device__ __forceinline__ void dig(int v, uint64_t j, double w, GradAcc&) const { W[v * n + j] = w; }
    template <int NT>
    __device__ __forceinline__ void flush(int, int, GradAcc&) const {}
};

struct SinkCoef {
    using Acc = GradAcc;
    CoefSink cs;
    int lattice, m;
    __device__ __forceinline__ void lat(int v, uint64_t j, double2 z, GradAcc&) const {
        double* o = cs.out + cs.voff[v];
        if (m == 0) {
            o[0] = z.x * cs.scale;
            return;
        }
        o[bitrev64(2 * j, m)] = 2.0 * cs.scale * z.x;
        o[bitrev64(2 * j + 1, m)] = 2.0 * cs.scale * z.y;
    }
    __device__ __forceinline__ void dig(int v, uint64_t j, double w, GradAcc&) const {
        cs.out[cs.voff[v] + j] = w * cs.scale;
    }
    template <int NT>
    __device__ __forceinline__ void flush(int, int, GradAcc&) const {}
};

// ============================================================================ inverse, single CTA
template <int NT, class Snk>
__global__ void __launch_bounds__(NT) k_inv_small_lat(const double2* __restrict__ in, const long long* in_off,
                                                      long long cstride, int nvpc, Snk snk, int m,
                                                      const double2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.x;
    const int c = v / nvpc;
    const double2* x = in + c * cstride + in_off[v - c * nvpc];
    typename Snk::Acc acc;
    acc.zero();
    if (m == 0) {
        if (threadIdx.x == 0) snk.lat(v, 0, x[0], acc);
        snk.template flush<NT>(v, 0, acc);
        return;
    }
    const int lp = m - 1, Np = 1 << lp;
    for (int k = threadIdx.x; k <= Np / 2; k += NT) {
        if (k == 0) {
            const double2 A = x[0];
            sm[S(0)] = make_double2(0.5 * (A.x + A.y), 0.5 * (A.x - A.y));
            continue;
        }
        const int kp = Np - k;
        const double2 Ak = x[k], Ap = x[kp];
        sm[S(k)] = c2r_pre(Ak, Ap, twiddle(tw, k, m));
        if (kp != k) sm[S(kp)] = c2r_pre(Ap, Ak, twiddle(tw, kp, m));
    }
    __syncthreads();
    smem_fft<NT, true>(sm, lp, 1, padded_len(Np), +1, tw);
    for (int j = threadIdx.x; j < Np; j += NT) snk.lat(v, j, sm[S(j)], acc);
    snk.template flush<NT>(v, 0, acc);
}

template <int NT, class Snk>
__global__ void __launch_bounds__(NT) k_inv_small_dig(const double* __restrict__ in, const long long* in_off,
                                                      long long cstride, int nvpc, Snk snk, int m) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.x, n = 1 << m;
    const int c = v / nvpc;
    const double* x = in + c * cstride + in_off[v - c * nvpc];
    for (int e = threadIdx.x; e < n; e += NT) cp_async_el(&sm[S(e)], &x[e]);
    cp_async_wait_all();
    __syncthreads();
    smem_wht<NT, true>(sm, m, 1, padded_len(n));
    typename Snk::Acc acc;
    acc.zero();
    for (int e = threadIdx.x; e < n; e += NT) snk.dig(v, e, sm[S(e)], acc);
    snk.template flush<NT>(v, 0, acc);
}

// ============================================================================ inverse, two pass
template <int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT)
    k_inv_row_lat(const double2* __restrict__ in, const long long* in_off, long long cstride, int nvpc,
                  double2* __restrict__ U, long long vstride, int l1, int l2, int m, const double2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank());
    const int q = blockIdx.x >> 1, v = blockIdx.y;
    const int N1 = 1 << l1, N2 = 1 << l2;
    const int row = row_of_cluster(q, rank, N1);
    const int c = v / nvpc;
    const double2* x = in + c * cstride + in_off[v - c * nvpc] + ((long long)row << l2);
    for (int e = threadIdx.x; e < N2; e += NT) cp_async_el(&sm[S(e)], &x[e]);
    cp_async_wait_all();
    cl.sync();
    const bool self = (row == 0) || (row == N1 / 2);
    const double2* psm = self ? sm : cl.map_shared_rank(sm, rank ^ 1);
    double2 zr[EPT];
#pragma unroll
    for (int t = 0; t < EPT; ++t) {
        const int k2 = threadIdx.x + t * NT;
        if (k2 < N2) {
            const long long k = row + ((long long)k2 << l1);
            if (k == 0) {
                const double2 A = sm[S(0)];
                zr[t] = make_double2(0.5 * (A.x + A.y), 0.5 * (A.x - A.y));
            } else {
                const int kc = (row == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
                zr[t] = c2r_pre(sm[S(k2)], psm[S(kc)], twiddle(tw, uint64_t(k), m));
            }
        }
    }
    cl.sync();
#pragma unroll
    for (int t = 0; t < EPT; ++t) {
        const int k2 = threadIdx.x + t * NT;
        if (k2 < N2) sm[S(k2)] = zr[t];
    }
    __syncthreads();
    smem_fft<NT, true>(sm, l2, 1, padded_len(N2), +1, tw);
    double2* out = U + v * vstride + ((long long)row << l2);
    for (int j2 = threadIdx.x; j2 < N2; j2 += NT)
        out[j2] = cmulc(sm[S(j2)], twiddle(tw, uint64_t(j2) * uint64_t(row), l1 + l2));
}

template <int NT>
__global__ void __launch_bounds__(NT) k_inv_row_dig(const double* __restrict__ in, const long long* in_off,
                                                    long long cstride, int nvpc, double* __restrict__ U,
                                                    long long vstride, int l2) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    constexpr auto S = sidx<true>;
    const int row = blockIdx.x, v = blockIdx.y, N2 = 1 << l2;
    const int c = v / nvpc;
    const double* x = in + c * cstride + in_off[v - c * nvpc] + ((long long)row << l2);
    for (int e = threadIdx.x; e < N2; e += NT) cp_async_el(&sm[S(e)], &x[e]);
    cp_async_wait_all();
    __syncthreads();
    smem_wht<NT, true>(sm, l2, 1, padded_len(N2));
    double* out = U + v * vstride + ((long long)row << l2);
    for (int e = threadIdx.x; e < N2; e += NT) out[e] = sm[S(e)];
}

template <int NT, class Snk>
__global__ void __launch_bounds__(NT) k_inv_col_lat(const double2* __restrict__ U, long long vstride, Snk snk, int l1,
                                                    int l2, int lc, const double2* __restrict__ tw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sm = reinterpret_cast<double2*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.y, C = 1 << lc, N1 = 1 << l1, ld = padded_len(N1);
    const long long c0 = (long long)blockIdx.x << lc;
    const double2* x = U + v * vstride;
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int k1 = e >> lc, c = e & (C - 1);
        cp_async_el(&sm[c * ld + S(k1)], &x[((long long)k1 << l2) + c0 + c]);
    }
    cp_async_wait_all();
    __syncthreads();
    smem_fft<NT, true>(sm, l1, C, ld, +1, tw);
    typename Snk::Acc acc;
    acc.zero();
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int j1 = e >> lc, c = e & (C - 1);
        const uint64_t j = (uint64_t(j1) << l2) + c0 + c;
        snk.lat(v, j, sm[c * ld + S(j1)], acc);
    }
    snk.template flush<NT>(v, blockIdx.x, acc);
}

template <int NT, class Snk>
__global__ void __launch_bounds__(NT) k_inv_col_dig(const double* __restrict__ U, long long vstride, Snk snk, int l1,
                                                    int l2, int lc) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sm = reinterpret_cast<double*>(smraw);
    constexpr auto S = sidx<true>;
    const int v = blockIdx.y, C = 1 << lc, N1 = 1 << l1, ld = padded_len(N1);
    const long long c0 = (long long)blockIdx.x << lc;
    const double* x = U + v * vstride;
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int k1 = e >> lc, c = e & (C - 1);
        cp_async_el(&sm[c * ld + S(k1)], &x[((long long)k1 << l2) + c0 + c]);
    }
    cp_async_wait_all();
    __syncthreads();
    smem_wht<NT, true>(sm, l1, C, ld);
    typename Snk::Acc acc;
    acc.zero();
    for (int e = threadIdx.x; e < (C << l1); e += NT) {
        const int j1 = e >> lc, c = e & (C - 1);
        snk.dig(v, (uint64_t(j1) << l2) + c0 + c, sm[c * ld + S(j1)], acc);
    }
    snk.template flush<NT>(v, blockIdx.x, acc);
}

// ============================================================================ launchers
// Opt a kernel into > 48 KB dynamic smem once (host call; kept out of graph captures).
template <class K>
static void set_smem(K kern, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> done;
    std::lock_guard<std::mutex> lock(mu);
    const void* key = reinterpret_cast<const void*>(kern);
    for (auto& e : done)
        if (e.first == key && e.second >= bytes) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    done.push_back({key, bytes});
}

// threads for a tile of 2^tl elements (EPT per thread), 32..512
static int nt_for(int tl) {
    int nt = 1 << (tl > 4 ? tl - 4 : 0);
    return nt < 32 ? 32 : (nt > 512 ? 512 : nt);
}

template <class Src, class Snk>
static void fwd_impl(int lattice, const Geo& g, int nvec, const Src& src, const Snk& snk, void* work,
                     const double2* tw, cudaStream_t s) {
    const size_t es = lattice ? sizeof(double2) : sizeof(double);
    if (!g.two) {
        const size_t sm = size_t(padded_len(1 << g.lt)) * es;
        const int nt = nt_for(g.lt);
        if (lattice) {
            FM_NT_DISPATCH(nt, {
                auto k = k_fwd_small_lat<NT, Src, Snk>;
                set_smem(k, sm);
                ProfScope ps("fwd_small_lat", s);
                k<<<nvec, NT, sm, s>>>(src, snk, g.m, tw);
            })
        } else {
            FM_NT_DISPATCH(nt, {
                auto k = k_fwd_small_dig<NT, Src, Snk>;
                set_smem(k, sm);
                ProfScope ps("fwd_small_dig", s);
                k<<<nvec, NT, sm, s>>>(src, snk, g.m);
            })
        }
        return;
    }
    const size_t sm = size_t(std::max((1 << (g.cap - g.l1)) * padded_len(1 << g.l1), padded_len(1 << g.l2))) * es;
    const long long vstride = 1ll << g.lt;
    const int lc = g.cap - g.l1;
    const int ncol_blk = (1 << g.l2) >> lc;
    const int nt = nt_for(g.cap);
    FM_NT_DISPATCH(nt, {
        if (lattice) {
            auto kc = k_fwd_col_lat<NT, Src>;
            set_smem(kc, sm);
            {
                ProfScope ps("fwd_col_lat", s);
                kc<<<dim3(ncol_blk, nvec), NT, sm, s>>>(src, static_cast<double2*>(work), g.l1, g.l2, lc, vstride, tw);
            }
            auto kr = k_fwd_row_lat<NT, Snk>;
            set_smem(kr, sm);
            ProfScope ps("fwd_row_lat", s);
            kr<<<dim3(1 << g.l1, nvec), NT, sm, s>>>(static_cast<const double2*>(work), snk, g.l1, g.l2, vstride, g.m,
                                                     tw);
        } else {
            auto kc = k_fwd_col_dig<NT, Src>;
            set_smem(kc, sm);
            {
                ProfScope ps("fwd_col_dig", s);
                kc<<<dim3(ncol_blk, nvec), NT, sm, s>>>(src, static_cast<double*>(work), g.l1, g.l2, lc, vstride);
            }
            auto kr = k_fwd_row_dig<NT, Snk>;
            set_smem(kr, sm);
            ProfScope ps("fwd_row_dig", s);
            kr<<<dim3(1 << g.l1, nvec), NT, sm, s>>>(static_cast<const double*>(work), snk, g.l2, vstride);
        }
    })
}

static int gen_blocks(long long n, int ept = 1) {
    long long b = (n + GEN_NT * ept - 1) / (GEN_NT * ept);
    return int(b > 4096 ? 4096 : b);
}

void fwd_gen(int lattice, const Geo& g, int nvec, const GenSrc& src, const SpecSink& snk, void* work, void* genbuf,
             const double2* tw, cudaStream_t s) {
    if (genbuf) {  // split: generator at full parallelism, then transform the buffer
        const long long n = 1ll << g.m;
        {
            ProfScope ps("gen_fill", s);
            FM_D_DISPATCH(src.sp.d, k_gen_fill<D><<<dim3(gen_blocks(n), nvec), GEN_NT, 0, s>>>(
                                        src, static_cast<double*>(genbuf), n))
        }
        fwd_impl(lattice, g, nvec, BufSrc{static_cast<const double*>(genbuf), n}, snk, work, tw, s);
        return;
    }
    const int d = src.sp.d;
    if (d <= 4) fwd_impl(lattice, g, nvec, GenSrcD<4>{src}, snk, work, tw, s);
    else if (d <= 8) fwd_impl(lattice, g, nvec, GenSrcD<8>{src}, snk, work, tw, s);
    else fwd_impl(lattice, g, nvec, GenSrcD<16>{src}, snk, work, tw, s);
}

void fwd_array(int lattice, const Geo& g, int nvec, const ArraySrc& src, const ScaleSink& snk, void* work,
               const double2* tw, cudaStream_t s) {
    fwd_impl(lattice, g, nvec, src, snk, work, tw, s);
}

// Lattice query column with compile-time dimension cap and Bernoulli order: 32-bit exact lattice
// coordinate (x_p = t 2^-m + sh_lo 2^-53, the same value as QuerySrc's 64-bit chain) and the
// floating difference to the query coordinate (kernel_against_data, gp_core.cpp:386-397).
// Bound per vector (query, task): every per-dimension constant lives in registers, the element
// costs per dimension one 32-bit IMAD + LOP, one DADD (u32_to_f64), diff = (x_q - sh_lo 2^-53) - t 2^-m
// (one DFMA), u = frac(diff) and the Bernoulli polynomial in w = u^2 - u (symmetric under
// u -> 1 - u, so the reference's min(frac(d), frac(-d)) of kernels.cpp:28-32 is implied), then
// f = A + B v as in lattice.cu's LatGen (B2: v = w; B4: v = w^2).
template <int DC, int ALPHA>
struct QuerySrcLat {
    QuerySrc q;
    __device__ __forceinline__ double operator()(int v, uint64_t idx) const {
        const int qi = q.ntg == 1 ? v : v / q.ntg;
        const int l = __ldg(q.vec_task + (v - qi * q.ntg));
        const int sb = DIGITAL_BITS - q.m;
        const uint32_t mask = (1u << q.m) - 1u;
        const double inv_n = pow2i(-q.m);
        double prod = q.gamma;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            if (j < q.d) {
                const uint64_t sh = __ldg(q.shifts + l * q.d + j);
                const uint32_t t = (uint32_t(idx) * uint32_t(__ldg(q.g + j)) + uint32_t(sh >> sb)) & mask;
                const double xp = fma(double(t), inv_n, double(sh & ((uint64_t(1) << sb) - 1)) * 0x1p-53);
                const double diff = __ldg(q.X + (long long)qi * q.d + j) - xp;
                const double u1 = diff - floor(diff), u2 = -diff - floor(-diff);
                double u = fmin(u1, u2);
                if (u >= 1.0) u = 0.0;
                constexpr double pi2 = 9.869604401089358618834491;
                const double base = ALPHA == 1 ? 2.0 * pi2 * (u * (u - 1.0) + 1.0 / 6.0)
                                               : -(2.0 / 3.0) * pi2 * pi2 * (((u - 2.0) * u + 1.0) * u * u - 1.0 / 30.0);
                prod *= 1.0 + __ldg(q.eta + j) * base;
            }
        }
        return __ldg(q.Rrow + l) * prod;
    }
    struct Bound {
        uint32_t gm[DC], oh[DC];
        double c[DC], A[DC], B[DC];
        double scale, inv_n;
        uint32_t mask;
        __device__ __forceinline__ double operator()(uint64_t idx) const {
            double prod = scale;
#pragma unroll
            for (int j = 0; j < DC; ++j) {
                const uint32_t t = (uint32_t(idx) * gm[j] + oh[j]) & mask;
                // |diff| < 1, and w = u^2 - u of u = frac(diff) equals a^2 - a for a = |diff| on
                // both sides of 0 ((1 - a)(-a) for diff < 0): no floor, no I2F (both quarter rate)
                const double a = fabs(fma(-u32_to_f64(t), inv_n, c[j]));
                const double w = fma(a, a, -a);
                prod *= fma(B[j], ALPHA == 1 ? w : w * w, A[j]);
            }
            return prod;
        }
    };
    __device__ __forceinline__ Bound bind(int v) const {
        Bound b;
        const int qi = q.ntg == 1 ? v : v / q.ntg;
        const int l = __ldg(q.vec_task + (v - qi * q.ntg));
        const int sb = DIGITAL_BITS - q.m;
        b.mask = (1u << q.m) - 1u;
        b.inv_n = pow2i(-q.m);
        b.scale = __ldg(q.Rrow + l) * q.gamma;
        constexpr double pi2 = 9.869604401089358618834491;
        // base = ka v + kb: B2 2 pi^2 (w + 1/6); B4 -(2/3) pi^4 (w^2 - 1/30)
        constexpr double ka = ALPHA == 1 ? 2.0 * pi2 : -(2.0 / 3.0) * pi2 * pi2;
        constexpr double kb = ALPHA == 1 ? pi2 / 3.0 : pi2 * pi2 / 45.0;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
            if (j < q.d) {
                const uint64_t sh = __ldg(q.shifts + l * q.d + j);
                const double eta = __ldg(q.eta + j);
                b.gm[j] = uint32_t(__ldg(q.g + j)) & b.mask;
                b.oh[j] = uint32_t(sh >> sb) & b.mask;
                b.c[j] = __ldg(q.X + (long long)qi * q.d + j) - double(sh & ((uint64_t(1) << sb) - 1)) * 0x1p-53;
                b.A[j] = fma(eta, kb, 1.0);
                b.B[j] = eta * ka;
            } else {
                b.gm[j] = b.oh[j] = 0u;
                b.c[j] = b.B[j] = 0.0;
                b.A[j] = 1.0;
            }
        }
        return b;
    }
};
template <int DC, int ALPHA>
__device__ __forceinline__ typename QuerySrcLat<DC, ALPHA>::Bound bind_src(const QuerySrcLat<DC, ALPHA>& s, int v) {
    return s.bind(v);
}

void fwd_query(int lattice, const Geo& g, int nvec, const QuerySrc& src, const ScaleSink& snk, void* work,
               const double2* tw, cudaStream_t s) {
    if (lattice && src.m >= 1 && src.m <= 31) {
        const bool a1 = src.si_alpha == 1;
        if (src.d <= 4) a1 ? fwd_impl(1, g, nvec, QuerySrcLat<4, 1>{src}, snk, work, tw, s)
                           : fwd_impl(1, g, nvec, QuerySrcLat<4, 2>{src}, snk, work, tw, s);
        else if (src.d <= 8) a1 ? fwd_impl(1, g, nvec, QuerySrcLat<8, 1>{src}, snk, work, tw, s)
                                : fwd_impl(1, g, nvec, QuerySrcLat<8, 2>{src}, snk, work, tw, s);
        else a1 ? fwd_impl(1, g, nvec, QuerySrcLat<16, 1>{src}, snk, work, tw, s)
                : fwd_impl(1, g, nvec, QuerySrcLat<16, 2>{src}, snk, work, tw, s);
        return;
    }
    fwd_impl(lattice, g, nvec, src, snk, work, tw, s);
}

int grad_blocks(int lattice, const Geo& g, bool split) {
    (void)lattice;
    if (split) return gen_blocks(1ll << g.m, GEN_EPT);
    if (!g.two) return 1;
    const int lc = g.cap - g.l1;
    return (1 << g.l2) >> lc;
}

template <class Snk>
static void inv_impl(int lattice, const Geo& g, int nvec, const void* in, const long long* in_off, long long cstride,
                     int nvpc, const Snk& snk, void* work, const double2* tw, cudaStream_t s) {
    const size_t es = lattice ? sizeof(double2) : sizeof(double);
    if (!g.two) {
        const size_t sm = size_t(padded_len(1 << g.lt)) * es;
        const int nt = nt_for(g.lt);
        if (lattice) {
            FM_NT_DISPATCH(nt, {
                auto k = k_inv_small_lat<NT, Snk>;
                set_smem(k, sm);
                ProfScope ps("inv_small_lat", s);
                k<<<nvec, NT, sm, s>>>(static_cast<const double2*>(in), in_off, cstride, nvpc, snk, g.m, tw);
            })
        } else {
            FM_NT_DISPATCH(nt, {
                auto k = k_inv_small_dig<NT, Snk>;
                set_smem(k, sm);
                ProfScope ps("inv_small_dig", s);
                k<<<nvec, NT, sm, s>>>(static_cast<const double*>(in), in_off, cstride, nvpc, snk, g.m);
            })
        }
        return;
    }
    const size_t sm = size_t(std::max((1 << (g.cap - g.l1)) * padded_len(1 << g.l1), padded_len(1 << g.l2))) * es;
    const long long vstride = 1ll << g.lt;
    const int lc = g.cap - g.l1;
    const int ncol_blk = (1 << g.l2) >> lc;
    const int nt = nt_for(g.cap);
    FM_NT_DISPATCH(nt, {
        if (lattice) {
            set_smem(k_inv_row_lat<NT>, sm);
            {
                ProfScope ps("inv_row_lat", s);
                k_inv_row_lat<NT><<<dim3(1 << g.l1, nvec), NT, sm, s>>>(static_cast<const double2*>(in), in_off, cstride,
                                                                        nvpc, static_cast<double2*>(work), vstride,
                                                                        g.l1, g.l2, g.m, tw);
            }
            auto kc = k_inv_col_lat<NT, Snk>;
            set_smem(kc, sm);
            ProfScope ps("inv_col_lat", s);
            kc<<<dim3(ncol_blk, nvec), NT, sm, s>>>(static_cast<const double2*>(work), vstride, snk, g.l1, g.l2, lc,
                                                    tw);
        } else {
            set_smem(k_inv_row_dig<NT>, sm);
            {
                ProfScope ps("inv_row_dig", s);
                k_inv_row_dig<NT><<<dim3(1 << g.l1, nvec), NT, sm, s>>>(static_cast<const double*>(in), in_off, cstride,
                                                                        nvpc, static_cast<double*>(work), vstride,
                                                                        g.l2);
            }
            auto kc = k_inv_col_dig<NT, Snk>;
            set_smem(kc, sm);
            ProfScope ps("inv_col_dig", s);
            kc<<<dim3(ncol_blk, nvec), NT, sm, s>>>(static_cast<const double*>(work), vstride, snk, g.l1, g.l2, lc);
        }
    })
}

void inv_grad(int lattice, const Geo& g, int nvec, const void* in, const long long* in_off, long long cstride,
              int nvpc, const GradSink& gs, void* work, void* genbuf, const double2* tw, cudaStream_t s) {
    if (genbuf) {  // split: inverse transform -> W buffer -> full-parallelism dot
        const long long n = 1ll << g.m;
        SinkStoreW snk{static_cast<double*>(genbuf), n, g.m};
        inv_impl(lattice, g, nvec, in, in_off, cstride, nvpc, snk, work, tw, s);
        ProfScope ps("gen_dot", s);
        FM_D_DISPATCH(gs.gen.sp.d, k_gen_dot<D><<<dim3(gs.nblk, nvec), GEN_NT, 0, s>>>(
                                       gs, static_cast<const double*>(genbuf), n))
        return;
    }
    const int d = gs.gen.sp.d;
    if (d <= 4) inv_impl(lattice, g, nvec, in, in_off, cstride, nvpc, SinkGradD<4>{gs, lattice, g.m}, work, tw, s);
    else if (d <= 8) inv_impl(lattice, g, nvec, in, in_off, cstride, nvpc, SinkGradD<8>{gs, lattice, g.m}, work, tw, s);
    else inv_impl(lattice, g, nvec, in, in_off, cstride, nvpc, SinkGradD<16>{gs, lattice, g.m}, work, tw, s);
}

void inv_coef(int lattice, const Geo& g, int nvec, const void* in, const long long* in_off, const CoefSink& cs,
              void* work, const double2* tw, cudaStream_t s) {
    SinkCoef snk{cs, lattice, g.m};
    inv_impl(lattice, g, nvec, in, in_off, 0, nvec, snk, work, tw, s);
}

// ============================================================================ per-frequency T x T solve
template <int T, bool CX>
__global__ void __launch_bounds__(256) k_solve_equal(SolveArgs a) {
    using S = Sc<CX>;
    using V = typename S::T;
    constexpr int P = T * (T + 1) / 2;
    const int c = blockIdx.y;
    const V* lam = static_cast<const V*>(a.lam) + c * a.cstride;
    const V* yh = static_cast<const V*>(a.yhat);
    double ld_acc = 0.0, q_acc = 0.0;
    int first_bad = INT_MAX;
    double imx[T], rex[T];
#pragma unroll
    for (int t = 0; t < T; ++t) imx[t] = rex[t] = 0.0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < a.nslots;
         p += (long long)gridDim.x * blockDim.x) {
        V A[P], r[T], ch[T], Ai[P];
#pragma unroll
        for (int q = 0; q < P; ++q) A[q] = lam[q * a.nslots + p];
#pragma unroll
        for (int t = 0; t < T; ++t) r[t] = yh[t * a.nslots + p];
        if constexpr (CX) {
            if (p == 0) {
                // packed slot 0: frequency 0 (.x) and Nyquist (.y), two real systems, weight 1 each;
                // tau = yhat(0)/sqrt(n) zeroes the frequency-0 residual (gp_core.cpp:67-88)
                double A0[P], AN[P], r0[T], rN[T], c0[T], cN[T], I0[P], IN[P], l0, lN, q0, qN;
#pragma unroll
                for (int q = 0; q < P; ++q) A0[q] = A[q].x, AN[q] = A[q].y;
#pragma unroll
                for (int t = 0; t < T; ++t) r0[t] = 0.0, rN[t] = r[t].y;
                const bool want = a.M || a.lam_inv;
                int st0 = ldl_solve<T, false>(A0, r0, want, l0, q0, c0, I0, imx, rex);
                int stN = 0;
                if (a.has_nyq) {
                    stN = ldl_solve<T, false>(AN, rN, want, lN, qN, cN, IN, imx, rex);
                } else {  // n == 1: no Nyquist frequency
                    lN = qN = 0.0;
#pragma unroll
                    for (int t = 0; t < T; ++t) cN[t] = 0.0;
#pragma unroll
                    for (int q = 0; q < P; ++q) IN[q] = 0.0;
                }
                if (st0 == 1 || stN == 1) first_bad = 0;
                ld_acc += l0 + lN;
                q_acc += q0 + qN;
                if (a.M) {
                    V* Mo = static_cast<V*>(a.M) + c * a.cstride;
                    int q = 0;
#pragma unroll
                    for (int x = 0; x < T; ++x)
#pragma unroll
                        for (int y = x; y < T; ++y, ++q)
                            Mo[q * a.nslots] = make_double2(I0[q] - c0[x] * c0[y], IN[q] - cN[x] * cN[y]);
                }
                if (a.lam_inv) {
                    V* Io = static_cast<V*>(a.lam_inv) + c * a.cstride;
#pragma unroll
                    for (int q = 0; q < P; ++q) Io[q * a.nslots] = make_double2(I0[q], IN[q]);
                }
                if (a.chat) {
                    V* Co = static_cast<V*>(a.chat) + c * (long long)T * a.nslots;
#pragma unroll
                    for (int t = 0; t < T; ++t) Co[t * a.nslots] = make_double2(c0[t], cN[t]);
                }
                continue;
            }
        } else {
            if (p == 0) {
#pragma unroll
                for (int t = 0; t < T; ++t) r[t] = 0.0;
            }
        }
        double ld, qd;
        const int st = ldl_solve<T, CX>(A, r, a.M || a.lam_inv, ld, qd, ch, Ai, imx, rex);
        if (st == 1 && p < first_bad) first_bad = int(p);
        const double w = CX ? 2.0 : 1.0;  // lattice slot k >= 1 stands for k and n - k
        ld_acc += w * ld;
        q_acc += w * qd;
        if (a.M) {
            V* Mo = static_cast<V*>(a.M) + c * a.cstride;
            int q = 0;
#pragma unroll
            for (int x = 0; x < T; ++x)
#pragma unroll
                for (int y = x; y < T; ++y, ++q) Mo[q * a.nslots + p] = S::sub(Ai[q], S::mulc(ch[x], ch[y]));
        }
        if (a.lam_inv) {
            V* Io = static_cast<V*>(a.lam_inv) + c * a.cstride;
#pragma unroll
            for (int q = 0; q < P; ++q) Io[q * a.nslots + p] = Ai[q];
        }
        if (a.chat) {
            V* Co = static_cast<V*>(a.chat) + c * (long long)T * a.nslots;
#pragma unroll
            for (int t = 0; t < T; ++t) Co[t * a.nslots + p] = ch[t];
        }
    }
    __shared__ double red[32];
    const double ls = block_sum<256>(ld_acc, red);
    const double qs = block_sum<256>(q_acc, red);
    if (threadIdx.x == 0) {
        a.partial[((size_t)c * a.nblk + blockIdx.x) * 2 + 0] = ls;
        a.partial[((size_t)c * a.nblk + blockIdx.x) * 2 + 1] = qs;
    }
    if (first_bad != INT_MAX) atomicMin(a.bad + c, first_bad);
    // per-stage maxima (non-negative doubles order like their bit patterns)
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
}

// Class-mode per-frequency solve (see SolveArgs): pairs sharing a shift offset share one raw
// spectrum; dNLL/dR_p is accumulated here by Parseval, sum_j W_p(j) q_o(j) =
// sum_k M_p(k) conj(qhat_o(k)) over all n frequencies (slot k >= 1 of the real FFT stands for k and
// n - k: weight 2, Re; slot 0 packs frequency 0 and Nyquist), so only the V class adjoints go
// through the inverse transform.
template <int T, bool CX>
__global__ void __launch_bounds__(256) k_solve_class(SolveArgs a) {
    using S = Sc<CX>;
    using Vt = typename S::T;
    constexpr int P = T * (T + 1) / 2;
    const int c = blockIdx.y;
    const Vt* spec = static_cast<const Vt*>(a.lam) + c * a.cstride;
    const Vt* yh = static_cast<const Vt*>(a.yhat);
    Vt* Zo = a.M ? static_cast<Vt*>(a.M) + c * a.cstride : nullptr;
    __shared__ double s_coef[P], s_xi[P], s_wR[P];
    __shared__ int s_cls[P];
    if (threadIdx.x < P) {
        const int q = threadIdx.x;
        s_coef[q] = a.coef[(size_t)c * P + q];
        s_xi[q] = a.xi[(size_t)c * P + q];
        s_wR[q] = (a.pair_a[q] == a.pair_b[q] ? 1.0 : 2.0) * a.Rpair[(size_t)c * P + q];
        s_cls[q] = a.pair_cls[q];
    }
    __syncthreads();
    double acc[2 + P];
#pragma unroll
    for (int q = 0; q < 2 + P; ++q) acc[q] = 0.0;
    int first_bad = INT_MAX;
    double imx[T], rex[T];
#pragma unroll
    for (int t = 0; t < T; ++t) imx[t] = rex[t] = 0.0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < a.nslots;
         p += (long long)gridDim.x * blockDim.x) {
        Vt H[P], A[P], r[T], ch[T], Ai[P];
#pragma unroll
        for (int q = 0; q < P; ++q) H[q] = spec[s_cls[q] * a.nslots + p];  // shared classes hit L1
#pragma unroll
        for (int t = 0; t < T; ++t) r[t] = yh[t * a.nslots + p];
        if constexpr (CX) {
            if (p == 0) {
                // packed slot 0: frequency 0 (.x) and Nyquist (.y), two real systems; tau zeroes
                // the frequency-0 residual (gp_core.cpp:67-88)
                double A0[P], AN[P], r0[T], rN[T], c0[T], cN[T], I0[P], IN[P], l0, lN, q0, qN;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    A0[q] = fma(s_coef[q], H[q].x, s_xi[q]);
                    AN[q] = fma(s_coef[q], H[q].y, s_xi[q]);
                }
#pragma unroll
                for (int t = 0; t < T; ++t) r0[t] = 0.0, rN[t] = r[t].y;
                const bool want = Zo != nullptr;
                int st0 = ldl_solve<T, false>(A0, r0, want, l0, q0, c0, I0, imx, rex);
                int stN = 0;
                if (a.has_nyq) {
                    stN = ldl_solve<T, false>(AN, rN, want, lN, qN, cN, IN, imx, rex);
                } else {  // n == 1: no Nyquist frequency
                    lN = qN = 0.0;
#pragma unroll
                    for (int t = 0; t < T; ++t) cN[t] = 0.0;
#pragma unroll
                    for (int q = 0; q < P; ++q) IN[q] = 0.0;
                }
                if (st0 == 1 || stN == 1) first_bad = 0;
                acc[0] += l0 + lN;
                acc[1] += q0 + qN;
                if (Zo) {
                    double2 M[P];
                    int q = 0;
#pragma unroll
                    for (int x = 0; x < T; ++x)
#pragma unroll
                        for (int y = x; y < T; ++y, ++q) M[q] = make_double2(I0[q] - c0[x] * c0[y], IN[q] - cN[x] * cN[y]);
#pragma unroll
                    for (int q2 = 0; q2 < P; ++q2) acc[2 + q2] += M[q2].x * H[q2].x + M[q2].y * H[q2].y;
#pragma unroll
                    for (int o = 0; o < P; ++o) {
                        if (o >= a.V) break;
                        double2 z = make_double2(0.0, 0.0);
#pragma unroll
                        for (int q2 = 0; q2 < P; ++q2)
                            if (s_cls[q2] == o) z = make_double2(fma(s_wR[q2], M[q2].x, z.x), fma(s_wR[q2], M[q2].y, z.y));
                        Zo[o * a.nslots] = z;
                    }
                }
                if (a.chat) {
                    Vt* Co = static_cast<Vt*>(a.chat) + c * (long long)T * a.nslots;
#pragma unroll
                    for (int t = 0; t < T; ++t) Co[t * a.nslots] = make_double2(c0[t], cN[t]);
                }
                continue;
            }
        } else {
            if (p == 0) {
#pragma unroll
                for (int t = 0; t < T; ++t) r[t] = 0.0;
            }
        }
#pragma unroll
        for (int q = 0; q < P; ++q) {
            if constexpr (CX) A[q] = make_double2(fma(s_coef[q], H[q].x, s_xi[q]), s_coef[q] * H[q].y);
            else A[q] = fma(s_coef[q], H[q], s_xi[q]);
        }
        double ld, qd;
        const int st = ldl_solve<T, CX>(A, r, Zo != nullptr, ld, qd, ch, Ai, imx, rex);
        if (st == 1 && p < first_bad) first_bad = int(p);
        const double w = CX ? 2.0 : 1.0;  // lattice slot k >= 1 stands for k and n - k
        acc[0] += w * ld;
        acc[1] += w * qd;
        if (Zo) {
            Vt M[P];
            int q = 0;
#pragma unroll
            for (int x = 0; x < T; ++x)
#pragma unroll
                for (int y = x; y < T; ++y, ++q) M[q] = S::sub(Ai[q], S::mulc(ch[x], ch[y]));
#pragma unroll
            for (int q2 = 0; q2 < P; ++q2) {
                if constexpr (CX) acc[2 + q2] += w * (M[q2].x * H[q2].x + M[q2].y * H[q2].y);  // Re(M conj H)
                else acc[2 + q2] += M[q2] * H[q2];
            }
#pragma unroll
            for (int o = 0; o < P; ++o) {
                if (o >= a.V) break;
                Vt z = S::zero();
#pragma unroll
                for (int q2 = 0; q2 < P; ++q2)
                    if (s_cls[q2] == o) z = S::add(z, S::scale(M[q2], s_wR[q2]));
                Zo[o * a.nslots + p] = z;
            }
        }
        if (a.chat) {
            Vt* Co = static_cast<Vt*>(a.chat) + c * (long long)T * a.nslots;
#pragma unroll
            for (int t = 0; t < T; ++t) Co[t * a.nslots + p] = ch[t];
        }
    }
    __shared__ double redv[8 * (2 + P)];
    block_sum_vec<256, 2 + P>(acc, redv);
    if (threadIdx.x == 0) {
        double* pp = a.partial + ((size_t)c * a.nblk + blockIdx.x) * (2 + P);
#pragma unroll
        for (int q = 0; q < 2 + P; ++q) pp[q] = acc[q];
    }
    if (first_bad != INT_MAX) atomicMin(a.bad + c, first_bad);
    if constexpr (CX) {
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
    }
}

template <int T>
static void solve_t(const SolveArgs& a, int ncand, cudaStream_t s) {
    dim3 grid(a.nblk, ncand);
    ProfScope ps("solve_equal", s);
    if (a.classes) {
        if (a.lattice) k_solve_class<T, true><<<grid, 256, 0, s>>>(a);
        else k_solve_class<T, false><<<grid, 256, 0, s>>>(a);
        return;
    }
    if (a.lattice) k_solve_equal<T, true><<<grid, 256, 0, s>>>(a);
    else k_solve_equal<T, false><<<grid, 256, 0, s>>>(a);
}

void solve_equal(const SolveArgs& a, int ncand, cudaStream_t s) {
    switch (a.T) {
        case 1: solve_t<1>(a, ncand, s); break;
        case 2: solve_t<2>(a, ncand, s); break;
        case 3: solve_t<3>(a, ncand, s); break;
        case 4: solve_t<4>(a, ncand, s); break;
        case 5: solve_t<5>(a, ncand, s); break;
        case 6: solve_t<6>(a, ncand, s); break;
        case 7: solve_t<7>(a, ncand, s); break;
        case 8: solve_t<8>(a, ncand, s); break;
    }
}

// ============================================================================ finalize
// Deterministic fixed-order reductions of the per-block partials into the per-candidate
// result record (NLL = r^T c + logdet, gp_core.cpp:207-211; gradient chain to R, eta, gamma).
__global__ void __launch_bounds__(256) k_finalize(FinalArgs a) { finalize_candidate<256>(a, blockIdx.x); }

void finalize(const FinalArgs& a, cudaStream_t s) {
    ProfScope ps("finalize", s);
    k_finalize<<<a.ncand, 256, 0, s>>>(a);
}

__global__ void __launch_bounds__(256) k_finalize_classes(ClassFinalArgs a) {
    const int c = blockIdx.x;
    if (!a.grad_partial) {  // no gradient: logdet / quad only
        FinalArgs f{};
        f.P = a.P;
        f.d = a.d;
        f.nblk_solve = a.nblk_solve;
        f.solve_partial = a.solve_partial;
        f.solve_stride = 2 + a.P;
        f.out = a.out;
        finalize_candidate<256>(f, c);
        return;
    }
    ClassSums t{};
    t.T = a.T;
    t.P = a.P;
    t.V = a.V;
    t.d = a.d;
    t.nrows = a.nblk_solve;
    t.nblk = a.nblk_grad;
    t.dstride = MAXD + 1;
    t.mid = a.solve_partial + (size_t)c * a.nblk_solve * (2 + a.P);
    t.dot = a.grad_partial + (size_t)c * a.V * a.nblk_grad * (MAXD + 1);
    t.pair_a = a.pair_a;
    t.pair_b = a.pair_b;
    t.Rpair = a.Rpair + (size_t)c * a.P;
    t.gamma = a.gamma[c];
    t.out = a.out + (size_t)c * NOUT;
    class_sums_out<256>(t);
}

void finalize_classes(const ClassFinalArgs& a, int ncand, cudaStream_t s) {
    ProfScope ps("finalize", s);
    k_finalize_classes<<<ncand, 256, 0, s>>>(a);
}

// ============================================================================ per-slot Hermitian apply
template <int T, bool CX>
__global__ void k_apply_herm(long long nslots, const void* opv, const void* inv, void* outv) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* op = static_cast<const V*>(opv);
    const V* in = static_cast<const V*>(inv);
    V* out = static_cast<V*>(outv);
    auto pidx = [](int a, int b) { return a * T - a * (a - 1) / 2 + (b - a); };
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < nslots;
         p += (long long)gridDim.x * blockDim.x) {
        V x[T];
#pragma unroll
        for (int t = 0; t < T; ++t) x[t] = in[t * nslots + p];
#pragma unroll
        for (int a = 0; a < T; ++a) {
            V acc = S::zero();
#pragma unroll
            for (int b = 0; b < T; ++b) {
                const V o = op[pidx(a < b ? a : b, a < b ? b : a) * nslots + p];
                V e;
                if constexpr (CX) {
                    if (p == 0) e = make_double2(o.x * x[b].x, o.y * x[b].y);  // packed real pair
                    else e = (a <= b) ? S::mul(o, x[b]) : S::mul(S::conj(o), x[b]);
                    acc = make_double2(acc.x + e.x, acc.y + e.y);
                } else {
                    acc += o * x[b];
                }
            }
            out[a * nslots + p] = acc;
        }
    }
}

void apply_hermitian(int lattice, int T, long long nslots, const void* op, const void* in, void* out,
                     cudaStream_t s) {
    const int blocks = int((nslots + 255) / 256 < 1184 ? (nslots + 255) / 256 : 1184);
    ProfScope ps("apply_hermitian", s);
#define FM_AH(TT)                                                                   \
    case TT:                                                                        \
        if (lattice) k_apply_herm<TT, true><<<blocks, 256, 0, s>>>(nslots, op, in, out); \
        else k_apply_herm<TT, false><<<blocks, 256, 0, s>>>(nslots, op, in, out);        \
        break;
    switch (T) {
        FM_AH(1) FM_AH(2) FM_AH(3) FM_AH(4) FM_AH(5) FM_AH(6) FM_AH(7) FM_AH(8)
    }
#undef FM_AH
}

}  // namespace fmtgp
