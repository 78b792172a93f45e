// Unequal-n LDL^H fold kernels — see fold.cuh.
#include "fold.cuh"
#include "kernels.cuh"

namespace fmtgp {

template <bool CX>
__device__ __forceinline__ typename Sc<CX>::T getv(const typename Sc<CX>::T* v, long long n, long long i) {
    if constexpr (CX) {
        if (n > 1 && i > n / 2) return cconj(v[n - i]);
    }
    return v[i];
}

template <bool CX>
__device__ __forceinline__ double half_weight(long long n, long long i) {
    if constexpr (CX) return (i == 0 || (n > 1 && i == n / 2)) ? 1.0 : 2.0;
    return 1.0;
}

__device__ __forceinline__ long long lat_pos(const VecMap& mp, long long k) {
    if (!mp.two) return k;
    return (k & ((1ll << mp.l1) - 1)) * (1ll << mp.l2) + (k >> mp.l1);
}

// ------------------------------------------------------------------ layout conversion
template <bool CX>
__global__ void k_s2n(const VecMap* maps, const void* slots_v, long long sstride, void* nat_v, long long nstride) {
    using V = typename Sc<CX>::T;
    const VecMap mp = maps[blockIdx.y];
    const V* slots = static_cast<const V*>(slots_v) + blockIdx.z * sstride + mp.soff;
    V* nat = static_cast<V*>(nat_v) + blockIdx.z * nstride + mp.noff;
    const long long n = 1ll << mp.m, H = fold_H(CX, n);
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < H; k += (long long)gridDim.x * blockDim.x) {
        if constexpr (CX) {
            if (k == 0) nat[0] = make_double2(slots[0].x, 0.0);
            else if (k == n / 2) nat[k] = make_double2(slots[0].y, 0.0);
            else nat[k] = slots[lat_pos(mp, k)];
        } else {
            nat[k] = slots[k];
        }
    }
}

template <bool CX>
__global__ void k_n2s(const VecMap* maps, const void* nat_v, long long nstride, void* slots_v, long long sstride) {
    using V = typename Sc<CX>::T;
    const VecMap mp = maps[blockIdx.y];
    V* slots = static_cast<V*>(slots_v) + blockIdx.z * sstride + mp.soff;
    const V* nat = static_cast<const V*>(nat_v) + blockIdx.z * nstride + mp.noff;
    const long long n = 1ll << mp.m, H = fold_H(CX, n);
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < H; k += (long long)gridDim.x * blockDim.x) {
        if constexpr (CX) {
            if (k == 0) slots[0] = make_double2(nat[0].x, n > 1 ? nat[n / 2].x : 0.0);
            else if (k != n / 2) slots[lat_pos(mp, k)] = nat[k];
        } else {
            slots[k] = nat[k];
        }
    }
}

static int blocks_for(long long work) {
    long long b = (work + 255) / 256;
    return int(b < 1 ? 1 : (b > 1184 ? 1184 : b));
}

void slots_to_nat(int lattice, int nvec, int nblk, const VecMap* maps, const void* slots, long long sstride,
                  void* nat, long long nstride, cudaStream_t s) {
    ProfScope ps("slots_to_nat", s);
    dim3 g(64, nvec, nblk);
    if (lattice) k_s2n<true><<<g, 256, 0, s>>>(maps, slots, sstride, nat, nstride);
    else k_s2n<false><<<g, 256, 0, s>>>(maps, slots, sstride, nat, nstride);
}

void nat_to_slots(int lattice, int nvec, int nblk, const VecMap* maps, const void* nat, long long nstride,
                  void* slots, long long sstride, cudaStream_t s) {
    ProfScope ps("nat_to_slots", s);
    dim3 g(64, nvec, nblk);
    if (lattice) k_n2s<true><<<g, 256, 0, s>>>(maps, nat, nstride, slots, sstride);
    else k_n2s<false><<<g, 256, 0, s>>>(maps, nat, nstride, slots, sstride);
}

// ------------------------------------------------------------------ factorisation
// Pivots of stage s: d_s = Re lam_ss (fast_gram.cpp:167-178 check_positive semantics).
template <bool CX>
__global__ void __launch_bounds__(256) k_pivot(FoldDims D, int s, const void* lam_v, double* partial, int nblk,
                                               int* bad, unsigned long long* imre) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lss = static_cast<const V*>(lam_v) + D.poff[D.pid[s][s]];
    const long long n = D.n[s], H = D.H[s];
    double acc = 0.0, imx = 0.0, rex = 0.0;
    int first = 0x7f7f7f7f;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < H; i += (long long)gridDim.x * 256) {
        const V v = lss[i];
        const double d = S::re(v);
        imx = fmax(imx, fabs(S::im(v)));
        rex = fmax(rex, d);
        if (!(d > 0.0)) {
            if (i < first) first = int(i);
            continue;
        }
        acc += half_weight<CX>(n, i) * log(d);
    }
    __shared__ double red[32];
    acc = block_sum<256>(acc, red);
    if (threadIdx.x == 0) partial[s * nblk + blockIdx.x] = acc;
    if (first != 0x7f7f7f7f) atomicMin(bad, first);
    // stage maxima for the non-real test |Im S| > 1e-8 max(1, max Re S) (fast_gram.cpp:167-172)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        imx = fmax(imx, __shfl_xor_sync(0xffffffffu, imx, o));
        rex = fmax(rex, __shfl_xor_sync(0xffffffffu, rex, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(imre + 2 * s, (unsigned long long)__double_as_longlong(imx));
        atomicMax(imre + 2 * s + 1, (unsigned long long)__double_as_longlong(rex));
    }
}

struct StagePairs {
    int np;
    int a[MAXP], b[MAXP];
};

template <bool CX>
__global__ void __launch_bounds__(256) k_fold_update(FoldDims D, int s, StagePairs sp, void* lam_v) {
    using S = Sc<CX>;
    using V = typename S::T;
    V* lam = static_cast<V*>(lam_v);
    const int a = sp.a[blockIdx.y], b = sp.b[blockIdx.y];
    const V* lsa = lam + D.poff[D.pid[s][a]];
    const V* lsb = lam + D.poff[D.pid[s][b]];
    const V* lss = lam + D.poff[D.pid[s][s]];
    V* lab = lam + D.poff[D.pid[a][b]];
    const long long nS = D.n[s], nA = D.n[a], HA = D.H[a];
    const long long reps = nS / nA;
    for (long long k = blockIdx.x * 256ll + threadIdx.x; k < HA; k += (long long)gridDim.x * 256) {
        V acc = S::zero();
        for (long long c = 0; c < reps; ++c) {
            const long long i = c * nA + k;
            const V x = getv<CX>(lsa, nS, i), y = getv<CX>(lsb, nS, i);
            const double d = S::re(getv<CX>(lss, nS, i));
            acc = S::add(acc, S::scale(S::mulc(y, x), 1.0 / d));  // conj(x) y / d
        }
        lab[k] = S::sub(lab[k], acc);
    }
}

void fold_factor(const FoldDims& D, void* lam, double* partial, int nblk, int* bad, unsigned long long* imre,
                 cudaStream_t s) {
    for (int st = 0; st < D.T; ++st) {
        {
            ProfScope ps("fold_pivot", s);
            if (D.lattice) k_pivot<true><<<nblk, 256, 0, s>>>(D, st, lam, partial, nblk, bad, imre);
            else k_pivot<false><<<nblk, 256, 0, s>>>(D, st, lam, partial, nblk, bad, imre);
        }
        if (st + 1 == D.T) break;
        StagePairs sp{};
        long long work = 0;
        for (int a = st + 1; a < D.T; ++a)
            for (int b = a; b < D.T; ++b) {
                sp.a[sp.np] = a;
                sp.b[sp.np] = b;
                ++sp.np;
                work = work > D.H[a] ? work : D.H[a];
            }
        ProfScope ps("fold_update", s);
        dim3 g(blocks_for(work), sp.np);
        if (D.lattice) k_fold_update<true><<<g, 256, 0, s>>>(D, st, sp, lam);
        else k_fold_update<false><<<g, 256, 0, s>>>(D, st, sp, lam);
    }
}

// ------------------------------------------------------------------ solves
template <bool CX>
__global__ void __launch_bounds__(256) k_fs_quad(FoldDims D, int s, const void* lam_v, const void* rhs_v,
                                                 double* qpart, int nblk) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lss = static_cast<const V*>(lam_v) + D.poff[D.pid[s][s]];
    const int r = blockIdx.y;
    const V* z = static_cast<const V*>(rhs_v) + r * D.tot_task + D.toff[s];
    const long long n = D.n[s], H = D.H[s];
    double acc = 0.0;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < H; i += (long long)gridDim.x * 256)
        acc += half_weight<CX>(n, i) * S::abs2(z[i]) / S::re(lss[i]);
    __shared__ double red[32];
    acc = block_sum<256>(acc, red);
    if (threadIdx.x == 0) qpart[((size_t)r * D.T + s) * nblk + blockIdx.x] = acc;
}

template <bool CX>
__global__ void __launch_bounds__(256) k_fs_update(FoldDims D, int s, const void* lam_v, void* rhs_v) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lam = static_cast<const V*>(lam_v);
    const int a = s + 1 + blockIdx.y, r = blockIdx.z;
    V* rhs = static_cast<V*>(rhs_v) + r * D.tot_task;
    const V* lsa = lam + D.poff[D.pid[s][a]];
    const V* lss = lam + D.poff[D.pid[s][s]];
    const V* zs = rhs + D.toff[s];
    V* ra = rhs + D.toff[a];
    const long long nS = D.n[s], nA = D.n[a], HA = D.H[a], reps = nS / nA;
    for (long long k = blockIdx.x * 256ll + threadIdx.x; k < HA; k += (long long)gridDim.x * 256) {
        V acc = S::zero();
        for (long long c = 0; c < reps; ++c) {
            const long long i = c * nA + k;
            acc = S::add(acc, S::scale(S::mulc(getv<CX>(zs, nS, i), getv<CX>(lsa, nS, i)),
                                       1.0 / S::re(getv<CX>(lss, nS, i))));
        }
        ra[k] = S::sub(ra[k], acc);
    }
}

template <bool CX>
__global__ void __launch_bounds__(256) k_bs(FoldDims D, int s, const void* lam_v, void* rhs_v) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lam = static_cast<const V*>(lam_v);
    const int r = blockIdx.y;
    V* rhs = static_cast<V*>(rhs_v) + r * D.tot_task;
    const V* lss = lam + D.poff[D.pid[s][s]];
    V* zs = rhs + D.toff[s];
    const long long HS = D.H[s];
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < HS; i += (long long)gridDim.x * 256) {
        V acc = zs[i];
        for (int a = s + 1; a < D.T; ++a) {
            const V* lsa = lam + D.poff[D.pid[s][a]];
            const long long nA = D.n[a];
            acc = S::sub(acc, S::mul(lsa[i], getv<CX>(rhs + D.toff[a], nA, i % nA)));
        }
        zs[i] = S::scale(acc, 1.0 / S::re(lss[i]));
    }
}

void fold_solve(const FoldDims& D, const void* lam, void* rhs, int nrhs, double* qpart, int nblk, bool back,
                cudaStream_t s) {
    for (int st = 0; st < D.T; ++st) {
        if (qpart) {
            ProfScope ps("fold_fs_quad", s);
            dim3 g(nblk, nrhs);
            if (D.lattice) k_fs_quad<true><<<g, 256, 0, s>>>(D, st, lam, rhs, qpart, nblk);
            else k_fs_quad<false><<<g, 256, 0, s>>>(D, st, lam, rhs, qpart, nblk);
        }
        if (st + 1 < D.T) {
            ProfScope ps("fold_fs_update", s);
            dim3 g(blocks_for(D.H[st + 1]), D.T - st - 1, nrhs);
            if (D.lattice) k_fs_update<true><<<g, 256, 0, s>>>(D, st, lam, rhs);
            else k_fs_update<false><<<g, 256, 0, s>>>(D, st, lam, rhs);
        }
    }
    if (!back) return;
    for (int st = D.T - 1; st >= 0; --st) {
        ProfScope ps("fold_bs", s);
        dim3 g(blocks_for(D.H[st]), nrhs);
        if (D.lattice) k_bs<true><<<g, 256, 0, s>>>(D, st, lam, rhs);
        else k_bs<false><<<g, 256, 0, s>>>(D, st, lam, rhs);
    }
}

// cross[q] partials = sum_s sum_i w_i Re(conj(z_q) z_{q+nq}) / d_s over the forward-substituted
// right-hand sides q and q + nq (posterior covariance k(x)^T K^-1 k(x') = zx^H D^-1 zx')
template <bool CX>
__global__ void __launch_bounds__(256) k_fs_cross(FoldDims D, const void* lam_v, const void* rhs_v, int nq,
                                                  double* part, int nblk) {
    using S = Sc<CX>;
    using V = typename S::T;
    const int q = blockIdx.y;
    const V* za = static_cast<const V*>(rhs_v) + size_t(q) * D.tot_task;
    const V* zb = static_cast<const V*>(rhs_v) + size_t(q + nq) * D.tot_task;
    double acc = 0.0;
    for (int s = 0; s < D.T; ++s) {
        const V* lss = static_cast<const V*>(lam_v) + D.poff[D.pid[s][s]];
        const long long n = D.n[s], H = D.H[s], o = D.toff[s];
        for (long long i = blockIdx.x * 256ll + threadIdx.x; i < H; i += (long long)gridDim.x * 256) {
            const V a = za[o + i], b = zb[o + i];
            double re;
            if constexpr (CX) re = a.x * b.x + a.y * b.y;
            else re = a * b;
            acc += half_weight<CX>(n, i) * re / S::re(lss[i]);
        }
    }
    __shared__ double red[32];
    acc = block_sum<256>(acc, red);
    if (threadIdx.x == 0) part[size_t(q) * nblk + blockIdx.x] = acc;
}

void fold_cross_quad(const FoldDims& D, const void* lam, const void* rhs, int nq, double* part, int nblk,
                     cudaStream_t s) {
    ProfScope ps("fold_fs_cross", s);
    dim3 g(nblk, nq);
    if (D.lattice) k_fs_cross<true><<<g, 256, 0, s>>>(D, lam, rhs, nq, part, nblk);
    else k_fs_cross<false><<<g, 256, 0, s>>>(D, lam, rhs, nq, part, nblk);
}

// ------------------------------------------------------------------ selected inversion (trace of Lam^-1)
// Lam = U^H D U with U_{(s,i),(a, i mod n_a)} = lam_sa[i] / d_s[i] (the fold's factor).  Z = Lam^-1
// restricted to the SPECTRUM'S OWN pattern — z_ab[i] = Z_{(a,i),(b, i mod n_b)}, a <= b, the layout
// of lam — satisfies (Takahashi: Z = D^-1 U^-H + (I - U) Z), for s = T-1 .. 0:
//   z_sb[i] = -sum_{a>s} lam_sa[i] / d_s[i] * Z_{(a, i mod n_a),(b, i mod n_b)}   (b > s)
//   z_ss[i] = (1 - sum_{a>s} Re(lam_sa[i] conj(z_sa[i]))) / d_s[i]
// and every Z entry on the right lies on the pattern again (transposed when n_a < n_b), so the
// recursion closes in the spectrum's storage: trace(Lam^-1) = sum_s sum_i Re z_ss[i] without
// Algorithm 1's r x r grid (fast_gram.cpp:151-263, 301-309).  Lattice vectors keep their Hermitian
// natural half (Z inherits the symmetry of the real-data spectra).
template <bool CX>
__device__ __forceinline__ typename Sc<CX>::T zget(const FoldDims& D, const typename Sc<CX>::T* z, int a, long long p,
                                                   int b, long long q) {
    using S = Sc<CX>;
    if (a <= b) return getv<CX>(z + D.poff[D.pid[a][b]], D.n[a], p);
    return S::conj(getv<CX>(z + D.poff[D.pid[b][a]], D.n[b], q));
}

template <bool CX>
__global__ void __launch_bounds__(256) k_selinv_off(FoldDims D, int s, const void* lam_v, void* z_v) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lam = static_cast<const V*>(lam_v);
    V* z = static_cast<V*>(z_v);
    const int b = s + 1 + blockIdx.y;
    V* zsb = z + D.poff[D.pid[s][b]];
    const V* lss = lam + D.poff[D.pid[s][s]];
    const long long H = D.H[s], nb = D.n[b];
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < H; i += (long long)gridDim.x * 256) {
        V acc = S::zero();
        for (int a = s + 1; a < D.T; ++a)
            acc = S::add(acc, S::mul(lam[D.poff[D.pid[s][a]] + i], zget<CX>(D, z, a, i % D.n[a], b, i % nb)));
        zsb[i] = S::scale(acc, -1.0 / S::re(lss[i]));
    }
}

template <bool CX>
__global__ void __launch_bounds__(256) k_selinv_diag(FoldDims D, int s, const void* lam_v, void* z_v, double* part,
                                                     int nblk) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lam = static_cast<const V*>(lam_v);
    V* z = static_cast<V*>(z_v);
    V* zss = z + D.poff[D.pid[s][s]];
    const V* lss = lam + D.poff[D.pid[s][s]];
    const long long n = D.n[s], H = D.H[s];
    double tr = 0.0;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < H; i += (long long)gridDim.x * 256) {
        double acc = 0.0;
        for (int a = s + 1; a < D.T; ++a) {
            const V l = lam[D.poff[D.pid[s][a]] + i], w = z[D.poff[D.pid[s][a]] + i];
            acc += S::re(S::mulc(l, w));  // Re(l conj(w))
        }
        const double v = (1.0 - acc) / S::re(lss[i]);
        if constexpr (CX) zss[i] = make_double2(v, 0.0);
        else zss[i] = v;
        tr += half_weight<CX>(n, i) * v;
    }
    __shared__ double red[32];
    tr = block_sum<256>(tr, red);
    if (threadIdx.x == 0) part[s * nblk + blockIdx.x] = tr;
}

void fold_selinv_trace(const FoldDims& D, const void* lam, void* z, double* part, int nblk, cudaStream_t s) {
    ProfScope ps("fold_selinv", s);
    for (int st = D.T - 1; st >= 0; --st) {
        if (st + 1 < D.T) {
            dim3 g(blocks_for(D.H[st]), D.T - st - 1);
            if (D.lattice) k_selinv_off<true><<<g, 256, 0, s>>>(D, st, lam, z);
            else k_selinv_off<false><<<g, 256, 0, s>>>(D, st, lam, z);
        }
        if (D.lattice) k_selinv_diag<true><<<nblk, 256, 0, s>>>(D, st, lam, z, part, nblk);
        else k_selinv_diag<false><<<nblk, 256, 0, s>>>(D, st, lam, z, part, nblk);
    }
}

// Gradient adjoint on the pattern: M_ab[i] = Z_ab[i] - chat_a[i] conj(chat_b[i mod n_b]), in place
// over z (M = Lam^-1 - chat chat^H, the same M the equal-n solves form per frequency)
template <bool CX>
__global__ void __launch_bounds__(256) k_adjoint(FoldDims D, void* z_v, const void* chat_v) {
    using S = Sc<CX>;
    using V = typename S::T;
    int a = 0, b = 0;
    for (int q = blockIdx.y;; ++a) {  // pair blockIdx.y -> (a <= b), row by row
        if (q < D.T - a) {
            b = a + q;
            break;
        }
        q -= D.T - a;
    }
    V* z = static_cast<V*>(z_v) + D.poff[D.pid[a][b]];
    const V* ca = static_cast<const V*>(chat_v) + D.toff[a];
    const V* cb = static_cast<const V*>(chat_v) + D.toff[b];
    const long long H = D.H[a], nb = D.n[b];
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < H; i += (long long)gridDim.x * 256)
        z[i] = S::sub(z[i], S::mulc(ca[i], getv<CX>(cb, nb, i % nb)));
}

void fold_adjoint(const FoldDims& D, void* z, const void* chat, cudaStream_t s) {
    ProfScope ps("fold_adjoint", s);
    long long work = 0;
    for (int t = 0; t < D.T; ++t) work = work > D.H[t] ? work : D.H[t];
    dim3 g(blocks_for(work), D.T * (D.T + 1) / 2);
    if (D.lattice) k_adjoint<true><<<g, 256, 0, s>>>(D, z, chat);
    else k_adjoint<false><<<g, 256, 0, s>>>(D, z, chat);
}

// ------------------------------------------------------------------ Gram apply (gram_matvec)
template <bool CX>
__global__ void __launch_bounds__(256) k_gram_nat(FoldDims D, const void* lam_v, const void* v_v, void* out_v) {
    using S = Sc<CX>;
    using V = typename S::T;
    const V* lam = static_cast<const V*>(lam_v);
    const V* v = static_cast<const V*>(v_v);
    V* out = static_cast<V*>(out_v);
    const int a = blockIdx.y;
    const long long nA = D.n[a], HA = D.H[a];
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < HA; i += (long long)gridDim.x * 256) {
        V acc = S::mul(lam[D.poff[D.pid[a][a]] + i], v[D.toff[a] + i]);
        for (int b = 0; b < D.T; ++b) {
            if (b == a) continue;
            const long long nB = D.n[b];
            if (b > a) {  // tall block (a, b): lam_ab[i] v_b[i mod n_b]
                acc = S::add(acc, S::mul(lam[D.poff[D.pid[a][b]] + i], getv<CX>(v + D.toff[b], nB, i % nB)));
            } else {  // wide block: adjoint of the tall (b, a)
                const V* lba = lam + D.poff[D.pid[b][a]];
                for (long long c = 0; c < nB / nA; ++c) {
                    const long long j = c * nA + i;
                    acc = S::add(acc, S::mulc(getv<CX>(v + D.toff[b], nB, j), getv<CX>(lba, nB, j)));
                }
            }
        }
        out[D.toff[a] + i] = acc;
    }
}

void fold_gram_apply(const FoldDims& D, const void* lam, const void* v, void* out, cudaStream_t s) {
    long long work = 0;
    for (int t = 0; t < D.T; ++t) work = work > D.H[t] ? work : D.H[t];
    ProfScope ps("fold_gram", s);
    dim3 g(blocks_for(work), D.T);
    if (D.lattice) k_gram_nat<true><<<g, 256, 0, s>>>(D, lam, v, out);
    else k_gram_nat<false><<<g, 256, 0, s>>>(D, lam, v, out);
}

}  // namespace fmtgp
