// In-place mixed-radix FFT building blocks for the fused lattice kernels (lattice.cu).
//
// A vector of N = 2^LOG complex values (compile-time LOG >= 5) is transformed in shared memory
// by Gentleman-Sande decimation in frequency (DIF, forward) and its exact mirror, decimation in
// time (DIT, inverse).  LOG = 4 A16 + log2(R_last):
//   * A16 radix-16 stages s = 0 .. A16-1 with stride M_s = 2^(LOG - 4(s+1)) (block 16 M_s):
//       DIF: x[b 16M + j1 + M j2] (j2 natural) -> 16-point DFT -> * w_{16M}^(j1 k2) -> position
//            b 16M + j1 + M k2;
//       DIT: the inverse of that map (conjugate twiddle before the conjugate DFT);
//   * one tail stage of radix R_last = 2^(LOG mod 4) (or 16 when LOG mod 4 == 0) with M = 1,
//     twiddle-free.
// Every stage reads and writes the same 16 positions of its group, so a stage needs ONE
// barrier (the Stockham kernels of transform.cuh need two), and the first / last stage of a
// transform can be fused with whatever produces / consumes the data in registers.  The DIF
// output is in digit-reversed order: ip_freq(p) is the frequency held at position p, ip_pos its
// inverse; the DIT input is expected in that same order and its output is natural.
// Unnormalised, like transform.cuh: DIF computes sum_j x_j e^(-2 pi i jk/N), DIT the conjugate
// kernel.  Smem addressing is the padded sidx<true> (1 pad per 16 elements): radix-16 stages
// and the contiguous 16-position tail groups are bank-conflict free, and because a group's
// base has its low bits below M, sidx(base + r M) = sidx(base) + r M + (r M >> 4): with LOG a
// template parameter every smem access of a stage is an immediate offset from one pointer.
#pragma once

#include "transform.cuh"

namespace fmtgp {

template <int LOG>
struct Ip {
    static_assert(LOG >= 5 && LOG <= 13, "in-place FFT length");
    static constexpr int RL = (LOG & 3) ? (LOG & 3) : 4;  // log2 R_last
    static constexpr int A16 = (LOG - RL) >> 2;           // radix-16 stages before the tail
    // frequency held at DIF output position p: digit s of k (base 16, s < A16) sits at position
    // weight 2^(LOG - 4(s+1)); the tail digit (base R_last) at weight 1
    static __device__ __forceinline__ int freq(int p) {
        int k = (p & ((1 << RL) - 1)) << (4 * A16);
#pragma unroll
        for (int s = 0; s < A16; ++s) k |= ((p >> (LOG - 4 * (s + 1))) & 15) << (4 * s);
        return k;
    }
    static __device__ __forceinline__ int pos(int k) {
        int p = k >> (4 * A16);
#pragma unroll
        for (int s = 0; s < A16; ++s) p |= ((k >> (4 * s)) & 15) << (LOG - 4 * (s + 1));
        return p;
    }
    // frequency bits of the low 4 position bits: freq(p0 + lo) = freq(p0) | freq_lo(lo) for p0 a
    // multiple of 16 (the tail digit, then the low bits of radix-16 digit A16-1 at weight R_last)
    static __host__ __device__ constexpr int freq_lo(int lo) {
        return ((lo & ((1 << RL) - 1)) << (4 * A16)) | ((lo >> RL) << (4 * (A16 - 1)));
    }
};

// smem offset of element r of a group with stride M = 2^ML relative to sidx(base)
template <int ML>
__host__ __device__ constexpr int ip_off(int r) {
    return (r << ML) + ((r << ML) >> 4);
}
// exp(-2 pi i t / 2^L), L <= 13: one table read
__device__ __forceinline__ double2 tw_small(const double2* __restrict__ tab, uint32_t t, int L) {
    return __ldg(tab + (size_t(L) << TW_BASE_LOG) + (t & ((1u << L) - 1u)));
}

// w_{2^L}^(j1 k2) for k2 = 1..15 from four table reads (k2 = 1, 4, 8, 12) and at most three
// products in between (the scheme of fft_stage_body).  Loads first: callers issue this before
// their data loads so the table latency overlaps them.
struct Tw16 {
    double2 w1, w4, w8, w12;
    __device__ __forceinline__ void load(const double2* __restrict__ tw, int j1, int L) {
        w1 = tw_small(tw, uint32_t(j1), L);
        w4 = tw_small(tw, uint32_t(4 * j1), L);
        w8 = tw_small(tw, uint32_t(8 * j1), L);
        w12 = tw_small(tw, uint32_t(12 * j1), L);
    }
    // f(k2, w) for k2 = 1..15 in natural order, w = w^(j1 k2)
    template <class F>
    __device__ __forceinline__ void each(F&& f) const {
        double2 cur = w1;
#pragma unroll
        for (int k2 = 1; k2 < 16; ++k2) {
            if (k2 == 1) cur = w1;
            else if (k2 == 4) cur = w4;
            else if (k2 == 8) cur = w8;
            else if (k2 == 12) cur = w12;
            else cur = cmul(cur, w1);
            f(k2, cur);
        }
    }
};

// Stage-0 twiddles of a row transform merged with a common factor b (the per-thread base of the
// four-step twiddle): f(k2, b w^(j1 k2)) for k2 = 0..15, from b, b w^4, b w^8, b w^12 and w:
// 12 products per use, and the base never has to be multiplied into the 16 inputs.
struct Tw16B {
    double2 b0, b4, b8, b12, w1;
    __device__ __forceinline__ void load(const double2* __restrict__ tw, int j1, int L, double2 base) {
        w1 = tw_small(tw, uint32_t(j1), L);
        b0 = base;
        b4 = cmul(base, tw_small(tw, uint32_t(4 * j1), L));
        b8 = cmul(base, tw_small(tw, uint32_t(8 * j1), L));
        b12 = cmul(base, tw_small(tw, uint32_t(12 * j1), L));
    }
    template <class F>
    __device__ __forceinline__ void each0(F&& f) const {
        double2 cur = b0;
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
            if (k2 == 0) cur = b0;
            else if (k2 == 4) cur = b4;
            else if (k2 == 8) cur = b8;
            else if (k2 == 12) cur = b12;
            else cur = cmul(cur, w1);
            f(k2, cur);
        }
    }
};

// Stride-2 stage (ML = 1): j1 is 0 or 1, so the twiddles are 1 or the constants w_32^k2 — selected
// per lane (FSEL, off the fp64 pipe) instead of 4 table reads and 11 products (ip_stage<..., C1>).
// Measured on config 4: L1 -1 %, L3 +2 % (it spills more), so only the forward column kernel uses it.
struct Tw16C1 {
    int j1;
    template <class F>
    __device__ __forceinline__ void each(F&& f) const {
        constexpr double C32[16] = {1.0,
                                    0.9807852804032304491261822,
                                    0.9238795325112867561281832,
                                    0.8314696123025452370787884,
                                    0.7071067811865475244008444,
                                    0.5555702330196022247428308,
                                    0.38268343236508977172846,
                                    0.1950903220161282678482849,
                                    0.0,
                                    -0.1950903220161282678482849,
                                    -0.38268343236508977172846,
                                    -0.5555702330196022247428308,
                                    -0.7071067811865475244008444,
                                    -0.8314696123025452370787884,
                                    -0.9238795325112867561281832,
                                    -0.9807852804032304491261822};
        constexpr double S32[16] = {0.0,
                                    0.1950903220161282678482849,
                                    0.38268343236508977172846,
                                    0.5555702330196022247428308,
                                    0.7071067811865475244008444,
                                    0.8314696123025452370787884,
                                    0.9238795325112867561281832,
                                    0.9807852804032304491261822,
                                    1.0,
                                    0.9807852804032304491261822,
                                    0.9238795325112867561281832,
                                    0.8314696123025452370787884,
                                    0.7071067811865475244008444,
                                    0.5555702330196022247428308,
                                    0.38268343236508977172846,
                                    0.1950903220161282678482849};
#pragma unroll
        for (int k2 = 1; k2 < 16; ++k2) f(k2, make_double2(j1 ? C32[k2] : 1.0, j1 ? -S32[k2] : 0.0));
    }
};

// The same 15 twiddles read from a shared-memory table [k2 - 1][j1] (lanes of a warp read
// consecutive j1: conflict-free, immediate offsets): no products, no global loads.  Used by the
// middle stages whose stride is small (few distinct j1), see IpTw below.
template <int ML>
struct Tw16S {
    const double2* p;  // table + j1
    template <class F>
    __device__ __forceinline__ void each(F&& f) const {
#pragma unroll
        for (int k2 = 1; k2 < 16; ++k2) f(k2, p[(k2 - 1) << ML]);
    }
};

// DIF radix-16 group in registers: v[j2] natural in; out v[r] = Y[brev4(r)] * w^(j1 brev4(r)).
template <class TW>
__device__ __forceinline__ void dif16_regs(double2 (&v)[16], const TW& t) {
    reg_dft<16>(v, -1);
    t.each([&](int k2, double2 w) { v[brev_c<16>(k2)] = cmul(v[brev_c<16>(k2)], w); });
}
// DIT radix-16 group: v[k2] natural in; untwiddle, conjugate DFT; out v[r] = y[brev4(r)].
template <class TW>
__device__ __forceinline__ void dit16_regs(double2 (&v)[16], const TW& t) {
    t.each([&](int k2, double2 w) { v[k2] = cmulc(v[k2], w); });
    reg_dft<16>(v, +1);
}

// Every stage after DIF stage 0 (and every DIT stage before the last) works inside blocks of
// N/16 positions, and group gi of a stage lies in block gi >> (LOG - 8) — the block of chunk gi
// of the tail stage too.  Thread tid handles the groups gi = tid + j NT, so the 2^(LOG-8) <= 32
// threads that touch a block are lanes of ONE warp (LOG <= 13): those stages need __syncwarp,
// not a CTA barrier (WL = warp-local), and the warps of a CTA drift apart instead of running
// every stage in lock step.
template <bool WL>
__device__ __forceinline__ void ip_sync() {
    if constexpr (WL) __syncwarp();
    else __syncthreads();
}

// Shared-memory twiddle tables of the middle stages (stage s >= 1, stride 2^ML, ML = LOG - 4(s+1)):
// 15 2^ML entries per stage, kept for the stages with ML <= LAT_STW_MAXML.  A kernel declares
// `__shared__ double2 stw[IpTw<LOG>::N]`, fills it once (ip_tw_fill, then a CTA barrier) and
// passes it to ip_mid_stages<..., STW = true>.  Measured on config 4: the row kernel (L2) gains
// 1.5 %; the column kernels (L1, L3) spill with it and lose 3 - 20 %, so they keep Tw16.
#ifndef LAT_STW_MAXML
#define LAT_STW_MAXML 5
#endif
template <int LOG>
struct IpTw {
    static constexpr int A = Ip<LOG>::A16;
    static constexpr int ml(int s) { return LOG - 4 * (s + 1); }
    static constexpr bool on(int s) { return s >= 1 && s < A && ml(s) <= LAT_STW_MAXML; }
    static constexpr int n(int s) { return on(s) ? (15 << ml(s)) : 0; }
    static constexpr int off(int s) { return s <= 1 ? 0 : n(1); }  // stages 1, 2 only (LOG <= 13)
    static constexpr int N = n(1) + n(2) > 0 ? n(1) + n(2) : 1;
};
template <int NT, int LOG>
__device__ __forceinline__ void ip_tw_fill(double2* stw, const double2* __restrict__ tw) {
#pragma unroll
    for (int s = 1; s <= 2; ++s) {
        if (!IpTw<LOG>::on(s)) continue;
        const int ML = IpTw<LOG>::ml(s);
        for (int e = threadIdx.x; e < (15 << ML); e += NT) {
            const int k2 = (e >> ML) + 1, j1 = e & ((1 << ML) - 1);
            stw[IpTw<LOG>::off(s) + e] = tw_small(tw, uint32_t(j1 * k2), ML + 4);
        }
    }
}

// One middle radix-16 stage s over nvec vectors (stride ld), then a barrier (WL: warp barrier).
template <int NT, int LOG, int S_, bool DIT, bool WL = false, bool STW = false, bool C1 = false>
__device__ __forceinline__ void ip_stage(double2* sm, int nvec, int ld, const double2* __restrict__ tw,
                                         const double2* stw) {
    constexpr int ML = LOG - 4 * (S_ + 1);
    constexpr int GPV = LOG - 4;  // log2 groups per vector
    const int total = nvec << GPV;
#pragma unroll 1
    for (int gi = threadIdx.x; gi < total; gi += NT) {
        const int vec = gi >> GPV, q = gi & ((1 << GPV) - 1);
        const int j1 = q & ((1 << ML) - 1);
        const int base = ((q >> ML) << (ML + 4)) + j1;
        double2* x = sm + vec * ld + sidx<true>(base);
        double2 v[16];
        auto body = [&](const auto& t) {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = x[ip_off<ML>(r)];
            if (DIT) dit16_regs(v, t);
            else dif16_regs(v, t);
#pragma unroll
            for (int r = 0; r < 16; ++r) x[ip_off<ML>(brev_c<16>(r))] = v[r];
        };
        if constexpr (STW && IpTw<LOG>::on(S_)) {  // the kernel passes its filled table
            body(Tw16S<ML>{stw + IpTw<LOG>::off(S_) + j1});
        } else if constexpr (ML == 1 && C1) {
            body(Tw16C1{j1});
        } else {
            Tw16 t;
            t.load(tw, j1, ML + 4);
            body(t);
        }
    }
    ip_sync<WL>();
}

// Middle radix-16 stages 1 .. A16-1 (stage 0 is fused by the kernels): DIF ascending, DIT descending.
// WL: warp barriers between them; the DIT form ends with a CTA barrier anyway (stage 0 reads
// across blocks), unless LAST_WL (the caller synchronises the CTA itself).
template <int NT, int LOG, bool DIT, bool WL = false, bool STW = false, bool C1 = false>
__device__ __forceinline__ void ip_mid_stages(double2* sm, int nvec, int ld, const double2* __restrict__ tw,
                                              const double2* stw = nullptr) {
    static_assert(!WL || LOG <= 13, "warp-local stages need blocks of <= 32 groups");
    constexpr int A = Ip<LOG>::A16;
    if constexpr (!DIT) {
        if constexpr (A > 1) ip_stage<NT, LOG, 1, false, WL, STW, C1>(sm, nvec, ld, tw, stw);
        if constexpr (A > 2) ip_stage<NT, LOG, 2, false, WL, STW, C1>(sm, nvec, ld, tw, stw);
    } else {
        if constexpr (A > 2) ip_stage<NT, LOG, 2, true, WL, STW, C1>(sm, nvec, ld, tw, stw);
        if constexpr (A > 1) ip_stage<NT, LOG, 1, true, false, STW, C1>(sm, nvec, ld, tw, stw);
    }
}

// Tail stage (M = 1, radix R = 2^RL, twiddle-free) on 16 contiguous positions held in v:
// DIF: v natural -> v[c R + r] = Y_c[brev_R(r)]; DIT: v[c R + k2] natural -> y_c[brev_R(r)].
template <int LOG>
__device__ __forceinline__ void tail_regs(double2 (&v)[16], int dir) {
    constexpr int R = 1 << Ip<LOG>::RL;
#pragma unroll
    for (int c = 0; c < 16 / R; ++c) reg_dft<R>(v + c * R, dir);
}
// position offset (within the 16) of output element i of tail_regs
template <int LOG>
__host__ __device__ constexpr int tail_out_pos(int i) {
    constexpr int RL = Ip<LOG>::RL;
    constexpr int R = 1 << RL;
    int r = i & (R - 1), b = 0;
    for (int k = 0; k < RL; ++k) b |= ((r >> k) & 1) << (RL - 1 - k);
    return (i & ~(R - 1)) + b;
}

// Tail stage over whole smem vectors: thread owns 16 contiguous positions (conflict-free).
template <int NT, int LOG, bool WL = false>
__device__ __forceinline__ void ip_tail_stage(double2* sm, int nvec, int ld, int dir) {
    constexpr int CPV = LOG - 4;
    const int total = nvec << CPV;
#pragma unroll 1
    for (int gi = threadIdx.x; gi < total; gi += NT) {
        const int vec = gi >> CPV, p0 = (gi & ((1 << CPV) - 1)) << 4;
        double2* x = sm + vec * ld + sidx<true>(p0);
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = x[r];
        tail_regs<LOG>(v, dir);
#pragma unroll
        for (int r = 0; r < 16; ++r) x[tail_out_pos<LOG>(r)] = v[r];
    }
    ip_sync<WL>();
}

}  // namespace fmtgp
