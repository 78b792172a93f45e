// Equal-n digital-net fit in three fused kernels — see digital.cuh.
#include <cstdlib>

#include "digital.cuh"

namespace fmtgp {

thread_local std::vector<DigLaunchRec>* dig_rec = nullptr;

// Column FWHT radix of K1 / K3 (wht_radix_cap): a radix-16 stage of a 2^10-element tile has 64 groups
// for 256 threads.  Measured on config 5 (256-candidate sweep, K1 / K3 totals): radix 16 5.76 / 9.14 ms,
// radix 8 (half the CTA busy) 5.42 / 12.0 ms, radix 4 (all of it) 6.96 / 13.9 ms — the idle threads'
// issue slots go to the SM's other CTAs, so K1 takes radix 8 and K3 stays at radix 16.

// hyperparameters of candidate c (kernel parameters when use_hv, else the device block)
template <int D>
__device__ __forceinline__ double hv_eta(const DigArgs& a, int c, int j) {
    return a.use_hv ? a.hv.eta[j] : __ldg(a.eta + size_t(c) * D + j);
}
__device__ __forceinline__ double hv_gamma(const DigArgs& a, int c) { return a.use_hv ? a.hv.gamma : __ldg(a.gamma + c); }

// FMTGP_TRACE: first-entry / last-exit globaltimer marks per kernel phase (slot: min or max)
__device__ __forceinline__ void dig_trace(unsigned long long* tr, int slot, bool is_min) {
    if (!tr || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (is_min) atomicMin(tr + slot, t);
    else atomicMax(tr + slot, t);
}

bool DigGeo::make(int m, int P, DigGeo& g, long long total_vecs, int d) {
    if (m < 1 || P < 1) return false;
    // row length: all P (= class count V) rows of one frequency block in <= 64 KB of smem
    int l2max = 0;
    while (l2max < 13 && (long long)P * (2ll << l2max) * 8 <= 65536) ++l2max;
    int l2 = std::min(l2max, (m + 1) / 2);
    l2 = std::max(l2, m - 11);  // column length <= 2^11
    if (l2 > l2max || l2 > m || l2 < 0) return false;
    g.m = m;
    g.l2 = l2;
    g.l1 = m - l2;
    // column tile: >= ~4 CTAs per SM over all vectors, 2^10..2^11 elements, <= 2^(l1 + l2)
    int tl = 11;
    if (total_vecs > 0 && ((total_vecs << m) >> tl) < 4 * 148) tl = 10;
    if (d > 4) tl = 10;  // kappa tile d * 2^tl doubles: keep >= 2 CTAs per SM (config 5: d = 10)
    if (const char* e = std::getenv("FMTGP_DIG_TL")) tl = std::max(8, std::min(11, std::atoi(e)));  // tuning
    tl = std::max(tl, g.l1);
    g.lc = std::min(tl - g.l1, l2);
    if (g.lc < 0) return false;
    g.nt_col = std::max(32, (1 << (g.l1 + g.lc)) / 4);  // 4 elements per thread in the load phases
    int need = (P << l2) / EPT;
    int nt = 256;
    while (nt < need && nt < 512) nt <<= 1;
    if (nt * EPT < (P << l2)) return false;
    g.nt_mid = nt;
    g.nblk_col = (1 << l2) >> g.lc;
    return true;
}

// ------------------------------------------------------------------ design-time kappa table
template <int D>
__global__ void __launch_bounds__(GEN_NT_DIG) k_kappa_table(GenSrc g, const uint64_t* ofs, long long n, double* kap) {
    __shared__ GenSmem<D> t;
    gen_smem_init<D>(t, g, 0, /*load_eta=*/false);
    const int o = blockIdx.y;
    uint64_t off[D];
#pragma unroll
    for (int j = 0; j < D; ++j) off[j] = ofs[size_t(o) * MAXD + j];
    __syncthreads();
    for (long long i = blockIdx.x * (long long)GEN_NT_DIG + threadIdx.x; i < n; i += (long long)gridDim.x * GEN_NT_DIG) {
        double kappa[D];
        kappa_d<D>(g, t, off, i, kappa);
#pragma unroll
        for (int j = 0; j < D; ++j) kap[(size_t(o) * D + j) * n + i] = kappa[j];
    }
}

void dig_kappa_table(const Spatial& sp, const PointGen& pg, const uint64_t* d_ofs, int nofs, long long n, double* kap,
                     cudaStream_t s) {
    GenSrc g{};
    g.sp = sp;
    g.pg = pg;
    const long long b = std::min<long long>((n + GEN_NT_DIG - 1) / GEN_NT_DIG, 2048);
    ProfScope ps("kappa_table", s);
    FM_D_DISPATCH(sp.d, k_kappa_table<D><<<dim3(unsigned(b), nofs), GEN_NT_DIG, 0, s>>>(g, d_ofs, n, kap))
}

// Design-time kappa tile (D rows of the CTA's C columns x N1) -> smem, asynchronously: 16-byte
// copies when a tile row holds >= 2 adjacent columns (kbuf must then be 16-byte aligned).
template <int NT, int D>
__device__ __forceinline__ void load_kappa_tile(double* kbuf, const double* kp, long long n, int l1, int l2, int lc,
                                                long long c0) {
    const int lt = l1 + lc;
    if (lc >= 1) {
        const int hl = lt - 1;
        for (int idx = threadIdx.x; idx < (D << hl); idx += NT) {
            const int j = idx >> hl, e = (idx & ((1 << hl) - 1)) << 1;
            const long long i = ((long long)(e >> lc) << l2) + c0 + (e & ((1 << lc) - 1));
            cp_async16(kbuf + (j << lt) + e, kp + size_t(j) * n + i);
        }
    } else {
        for (int idx = threadIdx.x; idx < (D << lt); idx += NT) {
            const int j = idx >> lt, e = idx & ((1 << lt) - 1);
            cp_async8(kbuf + (j << lt) + e, kp + size_t(j) * n + ((long long)e << l2) + c0);
        }
    }
}
__host__ __device__ constexpr int kbuf_offset(int C, int ld) { return (C * ld + 1) & ~1; }

// ------------------------------------------------------------------ K1: generator x column FWHT
template <int NT, int D>
__global__ void __launch_bounds__(NT, 3) k_dig_col_fwd(DigArgs a, int l1, int l2, int lc) {
    extern __shared__ __align__(16) double sm[];
    __shared__ GenSmem<D> tab;
    dig_trace(a.trace, 0, true);
    // candidate group: the CTA evaluates candidates [cb, ce) against one kappa tile (read once)
    const int o = blockIdx.y % a.V, cb = (blockIdx.y / a.V) * a.cpb, ce = min(a.nc, cb + a.cpb);
    const int C = 1 << lc, N1 = 1 << l1, ld = padded_len(N1);
    const long long c0 = (long long)blockIdx.x << lc, n = a.n;
    const double* kp = a.kap ? a.kap + size_t(o) * D * n : nullptr;
    const int tile = C << l1;
    double* kbuf = sm + kbuf_offset(C, ld);
    if (kp) {
        // design-time kappa tile -> smem with cp.async (no register staging)
        load_kappa_tile<NT, D>(kbuf, kp, n, l1, l2, lc, c0);
        cp_async_wait_all();
    }
    uint64_t off[D];
    if (!kp) {
#pragma unroll
        for (int j = 0; j < D; ++j) off[j] = __ldg(a.cofs + size_t(o) * MAXD + j);
    }
    const int rstep = NT >> lc;
    const bool lin = (NT & (C - 1)) == 0 && (rstep & 15) == 0;
    const int so0 = (int(threadIdx.x) & (C - 1)) * ld + sidx<true>(int(threadIdx.x) >> lc), sstep = rstep + (rstep >> 4);
    const long long go0 = ((long long)(int(threadIdx.x) >> lc) << l2) + c0 + (int(threadIdx.x) & (C - 1));
    const long long gstep = (long long)rstep << l2;
#pragma unroll 1
    for (int c = cb; c < ce; ++c) {
        double eta[D];
#pragma unroll
        for (int j = 0; j < D; ++j) eta[j] = hv_eta<D>(a, c, j);
        const double gam = hv_gamma(a, c);
        GenSrc g{};
        __syncthreads();  // previous candidate's store phase is done with sm / tab
        if (kp) {
            for (int e = threadIdx.x; e < tile; e += NT) {
                double kappa[D];
#pragma unroll
                for (int j = 0; j < D; ++j) kappa[j] = kbuf[j * tile + e];
                sm[(e & (C - 1)) * ld + sidx<true>(e >> lc)] = product_kernel_d<D, false>(kappa, eta, gam, nullptr);
            }
        } else {
            g.sp = a.sp;
            g.pg = a.pg;
            g.eta = a.eta;
            gen_smem_init<D>(tab, g, c);
            __syncthreads();
            for (int e = threadIdx.x; e < tile; e += NT) {
                const int j1 = e >> lc, cc = e & (C - 1);
                const long long i = ((long long)j1 << l2) + c0 + cc;
                double kappa[D];
                kappa_d<D>(g, tab, off, uint64_t(i), kappa);
                sm[cc * ld + sidx<true>(j1)] = product_kernel_d<D, false>(kappa, eta, gam, nullptr);
            }
        }
        if (c == cb) {
            pdl_trigger();
            // zero the per-fit flags once per fit (K2 / K3 run after this kernel)
            if (blockIdx.x == 0 && blockIdx.y == 0) {
                for (int t = threadIdx.x; t < a.nc; t += NT) a.bad[t] = 0x7f7f7f7f;
                for (int t = threadIdx.x; t < a.nc * MAXT * 2; t += NT) a.imre[t] = 0ull;
            }
        }
        __syncthreads();
        smem_wht<NT, true>(sm, l1, C, ld, wht_radix_cap<NT>(l1, C, 1));  // >= half of the CTA busy per stage
        double* out = a.Y + (size_t(c) * a.V + o) * n;
        if (lin) {  // affine offsets (see k_dig_col_inv's load_tile)
            const double* s0 = sm + so0;
            double* o0 = out + go0;
            for (int i = 0, e = threadIdx.x; e < tile; ++i, e += NT) o0[i * gstep] = s0[i * sstep];
        } else {
            for (int e = threadIdx.x; e < (C << l1); e += NT) {
                const int k1 = e >> lc, cc = e & (C - 1);
                out[((long long)k1 << l2) + c0 + cc] = sm[cc * ld + sidx<true>(k1)];
            }
        }
    }
    dig_trace(a.trace, 1, false);
    dig_trace(a.trace, 11, true);
}

// ------------------------------------------------------------------ K2: row FWHT + solve + inverse row FWHT
template <int NT, int T>
__global__ void __launch_bounds__(NT) k_dig_mid(DigArgs a, int l2) {
    constexpr int P = T * (T + 1) / 2;
    extern __shared__ __align__(16) double sm[];  // [V][padded N2]
    __shared__ double s_coef[P], s_xi[P], s_wR[P];
    __shared__ int s_cls[P];
    const int row = blockIdx.x, c = blockIdx.y, N2 = 1 << l2, lds = padded_len(N2), V = a.V;
    const long long n = a.n, base = (long long)row << l2;
    double* Yc = a.Y + size_t(c) * V * n;
    // prologue independent of K1 (overlaps its tail under programmatic dependent launch)
    if (threadIdx.x < P) {
        const int q = threadIdx.x;
        s_coef[q] = a.use_hv ? a.hv.coef[q] : __ldg(a.coef + size_t(c) * P + q);
        s_xi[q] = a.use_hv ? a.hv.xi[q] : __ldg(a.xi + size_t(c) * P + q);
        s_wR[q] = (a.pair_a[q] == a.pair_b[q] ? 1.0 : 2.0) * (a.use_hv ? a.hv.Rpair[q] : __ldg(a.Rpair + size_t(c) * P + q));
        s_cls[q] = a.pair_ofs[q];
    }
    constexpr int KPT = T <= 4 ? 2 : 1;  // frequencies per thread held in the yhat prefetch
    double rpre[KPT][T];
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int k2 = threadIdx.x + u * NT;
#pragma unroll
        for (int t = 0; t < T; ++t)
            rpre[u][t] = (k2 < N2 && base + k2 != 0) ? __ldg(a.yhat + size_t(t) * n + base + k2) : 0.0;
    }
    dig_trace(a.trace, 2, true);
    pdl_wait();
    dig_trace(a.trace, 3, true);
    pdl_trigger();
    for (int e = threadIdx.x; e < (V << l2); e += NT) {
        const int o = e >> l2, k2 = e & (N2 - 1);
        cp_async8(&sm[o * lds + sidx<true>(k2)], &Yc[size_t(o) * n + base + k2]);
    }
    cp_async_wait_all();
    __syncthreads();
    smem_wht<NT, true>(sm, l2, V, lds);
    double acc[2 + P], imx[T], rex[T];  // logdet, quad, sum_k M_p qhat_o (dR partials)
#pragma unroll
    for (int q = 0; q < 2 + P; ++q) acc[q] = 0.0;
#pragma unroll
    for (int t = 0; t < T; ++t) imx[t] = rex[t] = 0.0;
    int first_bad = 0x7f7f7f7f;
    double lpm = 1.0;  // running pivot product lpm * 2^lpe: one log per thread (ldl_core)
    int lpe = 0;
#pragma unroll 1
    for (int u = 0, k2 = threadIdx.x; k2 < N2; ++u, k2 += NT) {
        const long long k = base + k2;
        const int si = sidx<true>(k2);
        double A[P], r[T], ch[T], Ai[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            A[q] = fma(s_coef[q], sm[s_cls[q] * lds + si], s_xi[q]);  // lam = R_ab * H q + xi (fast_gram.cpp:82-85)
            if (a.lam_out) a.lam_out[(size_t(c) * P + q) * n + k] = A[q];
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
            double rv = 0.0;
#pragma unroll
            for (int w = 0; w < KPT; ++w)
                if (u == w) rv = rpre[w][t];
            r[t] = u < KPT ? rv : (k == 0 ? 0.0 : __ldg(a.yhat + size_t(t) * n + k));
        }
        double qd;
        const int st = ldl_core<T, false>(A, r, a.want_grad != 0, lpm, lpe, qd, ch, Ai, imx, rex);
        if (st == 1 && int(k) < first_bad) first_bad = int(k);
        acc[1] += qd;
        if (a.want_grad) {
            double Mq[P];
            int q = 0;
#pragma unroll
            for (int x = 0; x < T; ++x)
#pragma unroll
                for (int y = x; y < T; ++y, ++q) Mq[q] = Ai[q] - ch[x] * ch[y];  // M = dNLL/dLam
#pragma unroll
            for (int q2 = 0; q2 < P; ++q2) acc[2 + q2] = fma(Mq[q2], sm[s_cls[q2] * lds + si], acc[2 + q2]);
            for (int o = 0; o < V; ++o) sm[o * lds + si] = 0.0;  // this thread owns column k2 of every class
#pragma unroll
            for (int q2 = 0; q2 < P; ++q2) sm[s_cls[q2] * lds + si] += s_wR[q2] * Mq[q2];  // Z_o
        }
        if (a.chat_out && c == 0) {
#pragma unroll
            for (int t = 0; t < T; ++t) a.chat_out[size_t(t) * n + k] = ch[t];
        }
    }
    acc[0] = log_of(lpm, lpe);
    __shared__ double redv[(NT / 32) * (2 + P)];
    block_sum_vec<NT, 2 + P>(acc, redv);
    const int nrows = gridDim.x;
    if (threadIdx.x == 0) {
        double* pm = a.part_mid + (size_t(c) * nrows + row) * (2 + P);
#pragma unroll
        for (int q = 0; q < 2 + P; ++q) pm[q] = acc[q];
    }
    if (first_bad != 0x7f7f7f7f) atomicMin(a.bad + c, first_bad);
    // real spectra: the stage-global non-real test cannot fire, imre stays zeroed by K1
    if (!a.want_grad) return;
    __syncthreads();
    smem_wht<NT, true>(sm, l2, V, lds);  // inverse FWHT over the row bits (self-inverse up to scale)
    for (int e = threadIdx.x; e < (V << l2); e += NT) {
        const int o = e >> l2, k2 = e & (N2 - 1);
        Yc[size_t(o) * n + base + k2] = sm[o * lds + sidx<true>(k2)];
    }
    dig_trace(a.trace, 4, false);
    dig_trace(a.trace, 12, true);
}

// ------------------------------------------------------------------ K3: column FWHT -> W -> gradient dot
template <int NT, int D>
__global__ void __launch_bounds__(NT, 3) k_dig_col_inv(DigArgs a, int l1, int l2, int lc, int nrows) {
    extern __shared__ __align__(16) double sm[];
    __shared__ GenSmem<D> tab;
    __shared__ int s_last;
    // candidate group: the CTA evaluates candidates [cb, ce) against one kappa tile (read once)
    const int o = blockIdx.y % a.V, cb = (blockIdx.y / a.V) * a.cpb, ce = min(a.nc, cb + a.cpb);
    const int c = cb;  // the last-CTA tail (tail == 1) runs only with one candidate per CTA
    const int C = 1 << lc, N1 = 1 << l1, ld = padded_len(N1);
    const long long c0 = (long long)blockIdx.x << lc, n = a.n;
    const int tile = C << l1;
    double* kbuf = sm + kbuf_offset(C, ld);
    // the kappa tile does not depend on K2: it streams in while K2 finishes (PDL) and while the
    // column is loaded and transformed
    dig_trace(a.trace, 5, true);
    if (a.kap) load_kappa_tile<NT, D>(kbuf, a.kap + size_t(o) * D * n, n, l1, l2, lc, c0);
    // hyperparameters of the first candidate before the wait (they may live in mapped host memory)
    double eta_nx[D], gam_nx;
#pragma unroll
    for (int j = 0; j < D; ++j) eta_nx[j] = hv_eta<D>(a, cb, j);
    gam_nx = hv_gamma(a, cb);
    pdl_wait();
    dig_trace(a.trace, 6, true);
    if (a.tail != 1) pdl_trigger();  // separate finalize kernel: let its CTA become resident now
    uint64_t off[D];
    if (!a.kap) {
#pragma unroll
        for (int j = 0; j < D; ++j) off[j] = __ldg(a.cofs + size_t(o) * MAXD + j);
    }
    const double* kp = a.kap ? a.kap + size_t(o) * D * n : nullptr;
    const int nblk = gridDim.x;
    __shared__ double redv[(NT / 32) * D];
    // candidate groups double-buffer the column tile: candidate c + 1's tile streams in while c is
    // transformed and reduced (second buffer after the kappa tile)
    double* const tile1 = kbuf + (a.kap ? D * tile : 0) + 2;
    auto tile_of = [&](int k) { return (k & 1) ? tile1 : sm; };  // (no local pointer array: it would live in local memory)
    // element e_i = tid + i NT of a tile sits at row k1 = (tid >> lc) + i (NT >> lc), column tid & (C - 1):
    // when NT / C is a multiple of 16 both its padded smem offset and its global offset are affine in
    // i, and a candidate's tile load is one multiply-add pair per copy instead of the index math
    const int rstep = NT >> lc;
    const bool lin = (NT & (C - 1)) == 0 && (rstep & 15) == 0;
    const int so0 = (int(threadIdx.x) & (C - 1)) * ld + sidx<true>(int(threadIdx.x) >> lc), sstep = rstep + (rstep >> 4);
    const long long go0 = ((long long)(int(threadIdx.x) >> lc) << l2) + c0 + (int(threadIdx.x) & (C - 1));
    const long long gstep = (long long)rstep << l2;
    auto load_tile = [&](double* dst, int cand) {
        const double* x = a.Y + (size_t(cand) * a.V + o) * n;
        if (lin) {
            double* d0 = dst + so0;
            const double* x0 = x + go0;
            for (int i = 0, e = threadIdx.x; e < tile; ++i, e += NT) cp_async8(d0 + i * sstep, x0 + i * gstep);
        } else {
            for (int e = threadIdx.x; e < tile; e += NT) {
                const int k1 = e >> lc, cc = e & (C - 1);
                cp_async8(&dst[cc * ld + sidx<true>(k1)], &x[((long long)k1 << l2) + c0 + cc]);
            }
        }
    };
    load_tile(tile_of(0), cb);
    GenSrc g{};
    if (!kp) {  // XOR tables of the digital net (candidate-independent)
        g.sp = a.sp;
        g.pg = a.pg;
        g.eta = a.eta;
        gen_smem_init<D>(tab, g, cb, /*load_eta=*/false);
    }
#pragma unroll 1
    for (int cc2 = cb; cc2 < ce; ++cc2) {
        double* tb = tile_of(cc2 - cb);
        double eta[D];
#pragma unroll
        for (int j = 0; j < D; ++j) eta[j] = eta_nx[j];
        const double gam = gam_nx;
        if (cc2 + 1 < ce) {
#pragma unroll
            for (int j = 0; j < D; ++j) eta_nx[j] = hv_eta<D>(a, cc2 + 1, j);
            gam_nx = hv_gamma(a, cc2 + 1);
        }
        double acc[D];
#pragma unroll
        for (int j = 0; j < D; ++j) acc[j] = 0.0;
        cp_async_wait_all();  // this candidate's tile (and, first time, the kappa tile)
        __syncthreads();      // ... visible to all; the previous candidate is done with the other buffer
        if (cc2 + 1 < ce) load_tile(tile_of(cc2 + 1 - cb), cc2 + 1);
        smem_wht<NT, true>(tb, l1, C, ld);  // radix 16 (smaller radices measured slower here: 9.1 -> 12.0 / 13.9 ms)
        if (kp) {
            for (int e = threadIdx.x; e < tile; e += NT) {
                const double W = tb[(e & (C - 1)) * ld + sidx<true>(e >> lc)];  // W = H M, natural index
                double kappa[D], dq[D];
#pragma unroll
                for (int j = 0; j < D; ++j) kappa[j] = kbuf[j * tile + e];
                product_kernel_d<D, true>(kappa, eta, gam, dq);
#pragma unroll
                for (int j = 0; j < D; ++j) acc[j] = fma(W, dq[j], acc[j]);
            }
        } else {
            for (int e = threadIdx.x; e < tile; e += NT) {
                const int j1 = e >> lc, cc = e & (C - 1);
                const long long i = ((long long)j1 << l2) + c0 + cc;
                const double W = tb[cc * ld + sidx<true>(j1)];
                double kappa[D], dq[D];
                kappa_d<D>(g, tab, off, uint64_t(i), kappa);
                product_kernel_d<D, true>(kappa, eta, gam, dq);
#pragma unroll
                for (int j = 0; j < D; ++j) acc[j] = fma(W, dq[j], acc[j]);
            }
        }
        block_sum_vec<NT, D>(acc, redv);
        if (threadIdx.x == 0) {
            double* out = a.part_dot + ((size_t(cc2) * a.V + o) * nblk + blockIdx.x) * (MAXD + 1);
#pragma unroll
            for (int j = 0; j < D; ++j) out[j] = acc[j];
        }
    }
    dig_trace(a.trace, 7, false);
    dig_trace(a.trace, 13, true);
    if (a.tail != 1) return;  // k_dig_finalize reduces the partials
    // last-CTA reduction: one acq_rel ticket per candidate over its V * nblk CTAs (the release
    // publishes this CTA's partial, the last arrival's acquire sees all of them); fixed
    // summation order => deterministic
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ticket = atom_add_acq_rel_gpu(a.counter + c, 1u);
        s_last = ticket == unsigned(a.V * nblk) - 1;
        if (s_last) a.counter[c] = 0;  // self-reset for the next replay
    }
    __syncthreads();
    if (!s_last) return;
    dig_trace(a.trace, 8, false);
    // stage every partial into the (now free) dynamic smem with all copies in flight: the tail is
    // one L2 round trip instead of a chain of dependent ones
    const int S = 2 + a.P;
    double* st_mid = sm;                                 // [nrows][2 + P]
    double* st_dot = sm + ((nrows * S + 1) & ~1);        // [V][nblk][D]
    if (a.stage_tail) {
        const double* pm = a.part_mid + size_t(c) * nrows * S;
#pragma unroll 1
        for (int i = threadIdx.x; i < nrows * S; i += NT) cp_async8(st_mid + i, pm + i);
        const double* pc = a.part_dot + size_t(c) * a.V * nblk * (MAXD + 1);
#pragma unroll 1
        for (int i = threadIdx.x; i < a.V * nblk * D; i += NT) {
            const int r = i / D, j = i - r * D;
            cp_async8(st_dot + i, pc + size_t(r) * (MAXD + 1) + j);
        }
        cp_async_wait_all();
    }
    __syncthreads();
    dig_trace(a.trace, 9, false);
    ClassSums t{};
    t.T = a.T;
    t.P = a.P;
    t.V = a.V;
    t.d = D;
    t.nrows = nrows;
    t.nblk = nblk;
    t.dstride = a.stage_tail ? D : MAXD + 1;
    t.mid = a.stage_tail ? st_mid : a.part_mid + size_t(c) * nrows * S;
    t.dot = a.stage_tail ? st_dot : a.part_dot + size_t(c) * a.V * nblk * (MAXD + 1);
    t.pair_a = a.pair_a;
    t.pair_b = a.pair_b;
    t.Rpair = a.Rpair + size_t(c) * a.P;
    t.gamma = 0.0;  // unused by class_sums_out (dNLL/dgamma is formed on the host)
    t.out = (a.zc_res ? a.zc_res : a.out) + size_t(c) * NOUT;
    class_sums_out<NT>(t);
    if (a.zc_res)  // flags (K2's atomics, complete before this grid started) and tau words
        for (int i = a.res_flags_off + threadIdx.x; i < a.res_len; i += NT) a.zc_res[i] = a.res_dev[i];
    if (a.done_flag) {
        __syncthreads();  // every record word of this CTA is written ...
        if (threadIdx.x == 0) {
            __threadfence_system();  // ... and ordered before the completion word (cumulative fence)
            *a.done_flag = a.seq;
        }
    }
    __syncthreads();
    dig_trace(a.trace, 10, false);
}

// ------------------------------------------------------------------ finalize as its own kernel
// (DigArgs::tail != 1): one CTA per candidate; under programmatic dependent launch it is resident
// (prologue done) while K3 runs and reduces as soon as K3's partials are visible.
__global__ void __launch_bounds__(256) k_dig_finalize(DigArgs a, int nrows, int nblk) {
    const int c = blockIdx.x;
    ClassSums t{};
    t.T = a.T;
    t.P = a.P;
    t.V = a.V;
    t.d = a.d;
    t.nrows = nrows;
    t.nblk = nblk;
    t.dstride = MAXD + 1;
    t.mid = a.part_mid + size_t(c) * nrows * (2 + a.P);
    t.dot = a.part_dot + size_t(c) * a.V * nblk * (MAXD + 1);
    t.pair_a = a.pair_a;
    t.pair_b = a.pair_b;
    t.Rpair = a.Rpair + size_t(c) * a.P;
    t.gamma = 0.0;  // unused by class_sums_out (dNLL/dgamma is formed on the host)
    t.out = a.out + size_t(c) * NOUT;
    pdl_wait();
    class_sums_out<256>(t);
}

// ------------------------------------------------------------------ launcher
template <class K>
static void set_smem_dig(K kern, size_t bytes) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

template <int T>
static void mid_launch(const DigGeo& g, const DigArgs& a, size_t sm, cudaStream_t s) {
    const dim3 grid(1u << g.l1, a.nc);
    FM_NT_DISPATCH(g.nt_mid, {
        auto k = k_dig_mid<NT, T>;
        set_smem_dig(k, sm);
        ProfScope ps("dig_mid", s);
        CK_LAUNCH(launch_pdl(k, grid, dim3(NT), sm, s, true, a, g.l2));
        if (dig_rec) dig_rec->push_back({reinterpret_cast<const void*>(k), grid, dim3(NT), sm, a, {g.l2}, 1});
    })
}

void dig_fit(const DigGeo& g, const DigArgs& a_in, cudaStream_t s) {
    DigArgs a = a_in;
    const int C = 1 << g.lc;
    // K1/K3 dynamic smem: column tile (+ kappa tile); K3's last CTA reuses it to stage partials
    const size_t tile_words = size_t(kbuf_offset(C, padded_len(1 << g.l1))) + (a.kap ? size_t(a.d) << (g.l1 + g.lc) : 0) +
                              (a.cpb > 1 ? size_t(C) * padded_len(1 << g.l1) + 2 : 0);  // K3's second column tile
    const size_t stage_words = ((size_t(1 << g.l1) * (2 + a.P) + 1) & ~size_t(1)) + size_t(a.V) * g.nblk_col * a.d;
    // staging the partials for the last CTA's reduction is worth it only while it costs no
    // occupancy (config 5: 192 KB of partials vs a 99 KB tile -> 1 instead of 2 CTAs per SM)
    auto ctas = [](size_t words) { return int((227u * 1024u) / std::max<size_t>(words * sizeof(double), 1)); };
    const bool stage = ctas(std::max(tile_words, stage_words)) >= ctas(tile_words);
    a.stage_tail = stage ? 1 : 0;
    const size_t sm_col = (stage ? std::max(tile_words, stage_words) : tile_words) * sizeof(double);
    const dim3 gcol(g.nblk_col, a.V * ((a.nc + a.cpb - 1) / a.cpb));
    FM_D_DISPATCH(a.d, {
        FM_NT_DISPATCH(g.nt_col, {
            auto k1 = k_dig_col_fwd<NT, D>;
            set_smem_dig(k1, sm_col);
            ProfScope ps("dig_col_fwd", s);
            k1<<<gcol, NT, sm_col, s>>>(a, g.l1, g.l2, g.lc);
            if (dig_rec)
                dig_rec->push_back({reinterpret_cast<const void*>(k1), gcol, dim3(NT), sm_col, a, {g.l1, g.l2, g.lc}, 3});
        })
    })
    const size_t sm_mid = size_t(a.V) * padded_len(1 << g.l2) * sizeof(double);
    switch (a.T) {
        case 1: mid_launch<1>(g, a, sm_mid, s); break;
        case 2: mid_launch<2>(g, a, sm_mid, s); break;
        case 3: mid_launch<3>(g, a, sm_mid, s); break;
        case 4: mid_launch<4>(g, a, sm_mid, s); break;
        case 5: mid_launch<5>(g, a, sm_mid, s); break;
        case 6: mid_launch<6>(g, a, sm_mid, s); break;
        case 7: mid_launch<7>(g, a, sm_mid, s); break;
        default: mid_launch<8>(g, a, sm_mid, s); break;
    }
    if (!a.want_grad) return;
    const int nrows = 1 << g.l1;
    FM_D_DISPATCH(a.d, {
        FM_NT_DISPATCH(g.nt_col, {
            auto k3 = k_dig_col_inv<NT, D>;
            set_smem_dig(k3, sm_col);
            ProfScope ps("dig_col_inv", s);
            CK_LAUNCH(launch_pdl(k3, gcol, dim3(NT), sm_col, s, true, a, g.l1, g.l2, g.lc, nrows));
            if (dig_rec)
                dig_rec->push_back(
                    {reinterpret_cast<const void*>(k3), gcol, dim3(NT), sm_col, a, {g.l1, g.l2, g.lc, nrows}, 4});
        })
    })
    if (a.tail != 1) {
        ProfScope ps("dig_finalize", s);
        CK_LAUNCH(launch_pdl(k_dig_finalize, dim3(a.nc), dim3(256), 0, s, a.tail == 2, a, nrows, g.nblk_col));
        if (dig_rec)
            dig_rec->push_back({reinterpret_cast<const void*>(k_dig_finalize), dim3(a.nc), dim3(256), 0, a,
                                {nrows, g.nblk_col}, 2});
    }
}

}  // namespace fmtgp
