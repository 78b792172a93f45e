// In-place mixed-radix FFT building blocks for the fused lattice kernels (lattice.cu).
//
// A vector of N = 2^LOG complex values (LOG >= 5) is transformed in shared memory by
// Gentleman-Sande decimation in frequency (DIF, forward) and its exact mirror, decimation in
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
// with M >= 2 and the contiguous 16-position tail groups are bank-conflict free.
#pragma once

#include "transform.cuh"

namespace fmtgp {

struct IpGeo {
    int log;   // N = 2^log
    int a16;   // radix-16 stages before the tail
    int rl;    // log2 R_last (4 when log is a multiple of 4)
    __host__ __device__ static IpGeo of(int log) {
        IpGeo g;
        g.log = log;
        g.rl = (log & 3) ? (log & 3) : 4;
        g.a16 = (log - g.rl) >> 2;
        return g;
    }
};

// frequency held at DIF output position p: digit s of k (base 16, s < a16) sits at position
// weight 2^(log - 4(s+1)); the tail digit (base R_last) at weight 1.
__device__ __forceinline__ int ip_freq(int p, IpGeo g) {
    int k = (p & ((1 << g.rl) - 1)) << (4 * g.a16);
#pragma unroll
    for (int s = 0; s < 3; ++s)
        if (s < g.a16) k |= ((p >> (g.log - 4 * (s + 1))) & 15) << (4 * s);
    return k;
}
__device__ __forceinline__ int ip_pos(int k, IpGeo g) {
    int p = k >> (4 * g.a16);
#pragma unroll
    for (int s = 0; s < 3; ++s)
        if (s < g.a16) p |= ((k >> (4 * s)) & 15) << (g.log - 4 * (s + 1));
    return p;
}

// frequency bits of the low 4 position bits: ip_freq(p0 + lo) = ip_freq(p0) | ip_freq_lo(lo) for p0 a
// multiple of 16 (the tail digit, then the low bits of radix-16 digit a16-1 at position weight R_last)
__device__ __forceinline__ int ip_freq_lo(int lo, IpGeo g) {
    return ((lo & ((1 << g.rl) - 1)) << (4 * g.a16)) | ((lo >> g.rl) << (4 * (g.a16 - 1)));
}

// w_{2^L}^(j1 k2) for k2 = 1..15 from four table reads (k2 = 1, 4, 8, 12) and at most three
// products in between (the scheme of fft_stage_body).  Loads first: callers issue this before
// their data loads so the table latency overlaps them.
struct Tw16 {
    double2 w1, w4, w8, w12;
    __device__ __forceinline__ void load(const double2* __restrict__ tw, int j1, int L) {
        w1 = twiddle(tw, uint64_t(j1), L);
        w4 = twiddle(tw, uint64_t(4 * j1), L);
        w8 = twiddle(tw, uint64_t(8 * j1), L);
        w12 = twiddle(tw, uint64_t(12 * j1), L);
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

// DIF radix-16 group in registers: v[j2] natural in; out v[r] = Y[brev4(r)] * w^(j1 brev4(r)).
__device__ __forceinline__ void dif16_regs(double2 (&v)[16], const Tw16& t) {
    reg_dft<16>(v, -1);
    t.each([&](int k2, double2 w) { v[brev_c<16>(k2)] = cmul(v[brev_c<16>(k2)], w); });
}
// DIT radix-16 group: v[k2] natural in; untwiddle, conjugate DFT; out v[r] = y[brev4(r)].
__device__ __forceinline__ void dit16_regs(double2 (&v)[16], const Tw16& t) {
    t.each([&](int k2, double2 w) { v[k2] = cmulc(v[k2], w); });
    reg_dft<16>(v, +1);
}

// Middle radix-16 stages [s0, s1) of nvec vectors (stride ld) on one group per thread per
// vector-slot; each stage ends with a barrier.  DIF runs s ascending, DIT descending.
template <int NT, bool DIT>
__device__ __forceinline__ void ip_mid_stages(double2* sm, IpGeo g, int s0, int s1, int nvec, int ld,
                                              const double2* __restrict__ tw) {
    constexpr auto S = sidx<true>;
    const int gpv_log = g.log - 4;
    const int total = nvec << gpv_log;
#pragma unroll 1
    for (int i = 0; i < s1 - s0; ++i) {
        const int s = DIT ? s1 - 1 - i : s0 + i;
        const int M_log = g.log - 4 * (s + 1);
#pragma unroll 1
        for (int gi = threadIdx.x; gi < total; gi += NT) {
            const int vec = gi >> gpv_log, q = gi & ((1 << gpv_log) - 1);
            const int j1 = q & ((1 << M_log) - 1);
            const int base = ((q >> M_log) << (M_log + 4)) + j1;
            double2* x = sm + vec * ld;
            Tw16 t;
            t.load(tw, j1, M_log + 4);
            double2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = x[S(base + (r << M_log))];
            if (DIT) dit16_regs(v, t);
            else dif16_regs(v, t);
#pragma unroll
            for (int r = 0; r < 16; ++r) x[S(base + (brev_c<16>(r) << M_log))] = v[r];
        }
        __syncthreads();
    }
}

// Tail stage (M = 1, radix R = 2^rl, twiddle-free) on 16 contiguous positions held in v:
// DIF: v natural -> v[c R + r] = Y_c[brev_R(r)]; DIT: v[c R + k2] natural -> y_c[brev_R(r)].
template <int R>
__device__ __forceinline__ void tail_regs_r(double2 (&v)[16], int dir) {
#pragma unroll
    for (int c = 0; c < 16 / R; ++c) reg_dft<R>(v + c * R, dir);
}
__device__ __forceinline__ void tail_regs(double2 (&v)[16], int rl, int dir) {
    switch (rl) {
        case 1: tail_regs_r<2>(v, dir); break;
        case 2: tail_regs_r<4>(v, dir); break;
        case 3: tail_regs_r<8>(v, dir); break;
        default: tail_regs_r<16>(v, dir); break;
    }
}
// position offset (within the 16) of output element i of tail_regs
__device__ __forceinline__ int tail_out_pos(int i, int rl) {
    const int r = i & ((1 << rl) - 1);
    return (i & ~((1 << rl) - 1)) + int(__brev(unsigned(r)) >> (32 - rl));
}

// Tail stage over whole smem vectors: thread owns 16 contiguous positions (conflict-free).
template <int NT>
__device__ __forceinline__ void ip_tail_stage(double2* sm, IpGeo g, int nvec, int ld, int dir) {
    constexpr auto S = sidx<true>;
    const int cpv_log = g.log - 4;
    const int total = nvec << cpv_log;
#pragma unroll 1
    for (int gi = threadIdx.x; gi < total; gi += NT) {
        const int vec = gi >> cpv_log, p0 = (gi & ((1 << cpv_log) - 1)) << 4;
        double2* x = sm + vec * ld;
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = x[S(p0 + r)];
        tail_regs(v, g.rl, dir);
#pragma unroll
        for (int r = 0; r < 16; ++r) x[S(p0 + tail_out_pos(r, g.rl))] = v[r];
    }
    __syncthreads();
}

}  // namespace fmtgp
