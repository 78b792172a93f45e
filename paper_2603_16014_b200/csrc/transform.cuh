// Shared-memory fast transforms (fp64), the B200 replacement of the reference's
// scalar radix-2 loops (/root/reference/proj/src/transforms.cpp:19-100).
//
//  * FFT: Stockham autosort, radix 16/8/4/2 butterflies in registers, natural order in
//    and out, one smem round trip per stage.  Unnormalised; dir = -1 computes
//    sum_j a_j e^{-2 pi i jk/N}, dir = +1 the conjugate kernel.
//  * FWHT: radix-16 Hadamard groups over 4-bit slices, in place, natural order.
//
// Every thread holds EPT = 16 complex (or 16 real) values per stage, so a CTA of NT
// threads transforms NT*16 elements; batches of vectors share the CTA.
#pragma once

#include "common.cuh"

namespace fmtgp {

constexpr int EPT = 16;

// Bank-conflict-free smem addressing: one pad element after every 16 (a radix-16 group's
// stride-1 stage would otherwise put 32 lanes 128 B apart, i.e. on one bank).
template <bool PADDED>
__device__ __forceinline__ int sidx(int i) {
    return PADDED ? i + (i >> 4) : i;
}
__host__ __device__ constexpr int padded_len(int n) { return n + (n >> 4) + 1; }

// In-register DFT of R points (natural order in, bit-reversed order out), dir = -1 / +1.
template <int R>
__device__ __forceinline__ void reg_dft(double2* v, int dir) {
    // cos / sin (2 pi t / 16), t = 0..15
    constexpr double C16[16] = {1.0,
                                0.92387953251128675613,
                                0.70710678118654752440,
                                0.38268343236508977173,
                                0.0,
                                -0.38268343236508977173,
                                -0.70710678118654752440,
                                -0.92387953251128675613,
                                -1.0,
                                -0.92387953251128675613,
                                -0.70710678118654752440,
                                -0.38268343236508977173,
                                0.0,
                                0.38268343236508977173,
                                0.70710678118654752440,
                                0.92387953251128675613};
    constexpr double S16[16] = {0.0,
                                0.38268343236508977173,
                                0.70710678118654752440,
                                0.92387953251128675613,
                                1.0,
                                0.92387953251128675613,
                                0.70710678118654752440,
                                0.38268343236508977173,
                                0.0,
                                -0.38268343236508977173,
                                -0.70710678118654752440,
                                -0.92387953251128675613,
                                -1.0,
                                -0.92387953251128675613,
                                -0.70710678118654752440,
                                -0.38268343236508977173};
    // radix-2 decimation in frequency, output bit-reversed
#pragma unroll
    for (int len = R; len >= 2; len >>= 1) {
        const int half = len >> 1;
#pragma unroll
        for (int i = 0; i < R; i += len)
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 a = v[i + j], b = v[i + j + half];
                v[i + j] = cadd(a, b);
                double2 d = csub(a, b);
                const int t = j * (16 / len);  // angle 2 pi j / len in sixteenths
                if (t == 0) {
                } else if (t == 4) {  // multiply by exp(dir * i pi/2) = dir * i
                    d = dir < 0 ? make_double2(d.y, -d.x) : make_double2(-d.y, d.x);
                } else {
                    const double2 w = make_double2(C16[t], dir < 0 ? -S16[t] : S16[t]);
                    d = cmul(d, w);
                }
                v[i + j + half] = d;
            }
    }
    // output left in bit-reversed order: v[r] = X[bitrev_R(r)]; callers index accordingly
}

template <int R>
__host__ __device__ constexpr int brev_c(int k) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1, k >>= 1) r = (r << 1) | (k & 1);
    return r;
}

template <int R>
__device__ __forceinline__ void reg_wht(double* v) {
#pragma unroll
    for (int len = 2; len <= R; len <<= 1) {
        const int half = len >> 1;
#pragma unroll
        for (int i = 0; i < R; i += len)
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double a = v[i + j], b = v[i + j + half];
                v[i + j] = a + b;
                v[i + j + half] = a - b;
            }
    }
}

// One Stockham stage of radix R over nvec vectors of length 2^logN (vector q at
// buf + q * vstride).  Ns = 2^ns_log is the size of the already-combined sub-DFTs.
// Tail stages (R < 16) hold G = 16/R groups per thread; kept out of line so their register
// allocation does not stack on top of the radix-16 stages inlined in the same kernel.
template <int NT, int R, int RL, bool PADDED = false>
__device__ __forceinline__ void fft_stage_body(double2* buf, int logN, int ns_log, int nvec, int vstride, int dir,
                                          const double2* __restrict__ tw) {
    constexpr int G = EPT / R;
    const int gpv_log = logN - RL;
    const int gpv = 1 << gpv_log;
    const int total = gpv * nvec;
    double2 v[G][R];
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int gi = threadIdx.x + q * NT;
        if (gi < total) {
            const int vec = gi >> gpv_log, j = gi & (gpv - 1);
            const double2* x = buf + vec * vstride;
            const int k = j & ((1 << ns_log) - 1);
#pragma unroll
            for (int r = 0; r < R; ++r) v[q][r] = x[sidx<PADDED>(j + (r << gpv_log))];
            if (ns_log > 0) {
                // w^r for r < R: table reads at r = 1, 4, 8, 12 and at most three products by w in
                // between (4 loads instead of R-1 — those loads were this loop's long-scoreboard
                // stalls; error a few ulp; 12 live registers, no spill at NT = 512).
                double2 w1 = make_double2(1.0, 0.0), cur = w1;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    if (r == 1 || (r & 3) == 0) {
                        cur = twiddle(tw, uint64_t(r) * uint64_t(k), ns_log + RL);
                        if (dir > 0) cur.y = -cur.y;
                        if (r == 1) w1 = cur;
                    } else {
                        cur = cmul(cur, w1);
                    }
                    v[q][r] = cmul(v[q][r], cur);
                }
            }
            reg_dft<R>(v[q], dir);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int gi = threadIdx.x + q * NT;
        if (gi < total) {
            const int vec = gi >> gpv_log, j = gi & (gpv - 1);
            double2* x = buf + vec * vstride;
            const int k = j & ((1 << ns_log) - 1);
            const int o = ((j >> ns_log) << (ns_log + RL)) + k;
#pragma unroll
            for (int r = 0; r < R; ++r) x[sidx<PADDED>(o + (brev_c<R>(r) << ns_log))] = v[q][r];
        }
    }
    __syncthreads();
}

template <int NT, int R, int RL, bool PADDED>
__device__ __noinline__ void fft_stage_tail(double2* buf, int logN, int ns_log, int nvec, int vstride, int dir,
                                            const double2* __restrict__ tw) {
    fft_stage_body<NT, R, RL, PADDED>(buf, logN, ns_log, nvec, vstride, dir, tw);
}

template <int NT, int R, int RL, bool PADDED = false>
__device__ __forceinline__ void fft_stage(double2* buf, int logN, int ns_log, int nvec, int vstride, int dir,
                                          const double2* __restrict__ tw) {
    if constexpr (R == 16) fft_stage_body<NT, R, RL, PADDED>(buf, logN, ns_log, nvec, vstride, dir, tw);
    else fft_stage_tail<NT, R, RL, PADDED>(buf, logN, ns_log, nvec, vstride, dir, tw);
}

// Full unnormalised DFT of nvec vectors of length 2^logN in smem (natural order).
// Caller must __syncthreads() before (data in place); returns synchronised.
// Stages from `done` on (the first `done` radix-2 levels already applied, e.g. fused into a
// kernel's load phase: x[2j] = a_j + a_{j+N/2}, x[2j+1] = a_j - a_{j+N/2}, the twiddle-free
// Stockham radix-2 stage with ns_log = 0).
template <int NT, bool PADDED = false>
__device__ void smem_fft_from(double2* buf, int logN, int done, int nvec, int vstride, int dir,
                              const double2* __restrict__ tw) {
    while (done < logN) {
        const int left = logN - done;
        if (left >= 4) {
            fft_stage<NT, 16, 4, PADDED>(buf, logN, done, nvec, vstride, dir, tw);
            done += 4;
        } else if (left == 3) {
            fft_stage<NT, 8, 3, PADDED>(buf, logN, done, nvec, vstride, dir, tw);
            done += 3;
        } else if (left == 2) {
            fft_stage<NT, 4, 2, PADDED>(buf, logN, done, nvec, vstride, dir, tw);
            done += 2;
        } else {
            fft_stage<NT, 2, 1, PADDED>(buf, logN, done, nvec, vstride, dir, tw);
            done += 1;
        }
    }
}

template <int NT, bool PADDED = false>
__device__ void smem_fft(double2* buf, int logN, int nvec, int vstride, int dir, const double2* __restrict__ tw) {
    smem_fft_from<NT, PADDED>(buf, logN, 0, nvec, vstride, dir, tw);
}

template <int NT, int R, int RL, bool PADDED = false>
__device__ __forceinline__ void wht_stage(double* buf, int logN, int s, int nvec, int vstride) {
    constexpr int G = EPT / R;
    const int gpv_log = logN - RL;
    const int gpv = 1 << gpv_log;
    const int total = gpv * nvec;
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int gi = threadIdx.x + q * NT;
        if (gi < total) {
            const int vec = gi >> gpv_log, j = gi & (gpv - 1);
            double* x = buf + vec * vstride;
            const int lo = j & ((1 << s) - 1), hi = j >> s;
            const int base = (hi << (s + RL)) | lo;
            double v[R];
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = x[sidx<PADDED>(base + (r << s))];
            reg_wht<R>(v);
#pragma unroll
            for (int r = 0; r < R; ++r) x[sidx<PADDED>(base + (r << s))] = v[r];
        }
    }
    __syncthreads();
}

// Largest radix (log2, 1..4) whose stages still give at least `share` of the NT threads a group.
template <int NT>
__device__ __forceinline__ int wht_radix_cap(int logN, int nvec, int share_log) {
    const int elems = nvec << logN;
    int cap = 4;
    while (cap > 1 && (elems >> cap) < (NT >> share_log)) --cap;
    return cap;
}

// Unnormalised Walsh-Hadamard transform of nvec vectors of length 2^logN in smem.
// `cap` bounds the radix of a stage (log2): a radix-16 stage has 2^logN nvec / 16 groups, one per
// thread, so small tiles leave most of the CTA waiting at the stage's barrier (wht_radix_cap).
template <int NT, bool PADDED = false>
__device__ void smem_wht(double* buf, int logN, int nvec, int vstride, int cap = 4) {
    int done = 0;
    while (done < logN) {
        const int left = min(logN - done, cap);
        if (left >= 4) {
            wht_stage<NT, 16, 4, PADDED>(buf, logN, done, nvec, vstride);
            done += 4;
        } else if (left == 3) {
            wht_stage<NT, 8, 3, PADDED>(buf, logN, done, nvec, vstride);
            done += 3;
        } else if (left == 2) {
            wht_stage<NT, 4, 2, PADDED>(buf, logN, done, nvec, vstride);
            done += 2;
        } else {
            wht_stage<NT, 2, 1, PADDED>(buf, logN, done, nvec, vstride);
            done += 1;
        }
    }
}

}  // namespace fmtgp
