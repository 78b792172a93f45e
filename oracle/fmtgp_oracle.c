/* CPU restatement of the reference fast-MTGP hot path — see fmtgp_oracle.h.
 * TEST INFRASTRUCTURE ONLY (checker / CPU baseline); never linked into the product. */
#include "fmtgp_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

static _Thread_local char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

#define MASK53 ((((uint64_t)1) << 53) - 1)

/* ---------------------------------------------------------------- rng.hpp:14-47 */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}
uint64_t orc_rand_u64(uint64_t seed, uint64_t stream, uint64_t counter) {
    const uint64_t golden = 0x9E3779B97F4A7C15ULL;
    const uint64_t sub = mix64(seed + golden * (stream + 1));
    return mix64(sub + golden * (counter + 1));
}
static double uniform01(uint64_t seed, uint64_t stream, uint64_t c) {
    return (double)(orc_rand_u64(seed, stream, c) >> 11) * 0x1p-53;
}
double orc_normal(uint64_t seed, uint64_t stream, uint64_t k) {
    double u1 = uniform01(seed, stream, 2 * k);
    const double u2 = uniform01(seed, stream, 2 * k + 1);
    if (u1 <= 0.0) u1 = 0x1p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}

/* ---------------------------------------------------------------- transforms.cpp:10-100 */
uint64_t orc_bit_reverse(uint64_t i, int m) {
    uint64_t r = 0;
    for (int k = 0; k < m; ++k) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}
static int log2_exact(size_t n, int* m) {
    if (n == 0 || (n & (n - 1))) return fail(1, "length must be a power of two");
    *m = 0;
    while (((size_t)1 << *m) < n) ++*m;
    return 0;
}
/* transforms.cpp:19-30: in-place radix-2, scaled 2^{-m/2} */
int orc_fwht(double* a, size_t n) {
    int m;
    if (log2_exact(n, &m)) return 1;
    for (size_t len = 1; len < n; len <<= 1)
        for (size_t i = 0; i < n; i += 2 * len)
            for (size_t j = i; j < i + len; ++j) {
                const double u = a[j], v = a[j + len];
                a[j] = u + v;
                a[j + len] = u - v;
            }
    const double scale = pow(0.5, 0.5 * m);
    for (size_t i = 0; i < n; ++i) a[i] *= scale;
    return 0;
}
static cplx tw(size_t j, int m) { /* transforms.cpp:39-54: exp(-2 pi i j / 2^m) */
    const double ang = -6.283185307179586476925287 * (double)j / (double)((size_t)1 << m);
    return cos(ang) + I * sin(ang);
}
/* transforms.cpp:58-77: DIT butterflies on natural-order input = DFT(bitrev a), unitary */
static int fft_bitrev_c(cplx* a, size_t n) {
    int m;
    if (log2_exact(n, &m)) return 1;
    if (n == 1) return 0;
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1, stride = n / len;
        for (size_t i = 0; i < n; i += len)
            for (size_t j = 0; j < half; ++j) {
                const cplx v = a[i + j + half] * tw(j * stride, m);
                const cplx u = a[i + j];
                a[i + j] = u + v;
                a[i + j + half] = u - v;
            }
    }
    const double scale = pow(0.5, 0.5 * m);
    for (size_t i = 0; i < n; ++i) a[i] *= scale;
    return 0;
}
/* transforms.cpp:81-100: DIF with conjugated twiddles = bitrev(IDFT a) */
static int fft_bitrev_inv_c(cplx* a, size_t n) {
    int m;
    if (log2_exact(n, &m)) return 1;
    if (n == 1) return 0;
    for (size_t len = n; len >= 2; len >>= 1) {
        const size_t half = len >> 1, stride = n / len;
        for (size_t i = 0; i < n; i += len)
            for (size_t j = 0; j < half; ++j) {
                const cplx u = a[i + j];
                const cplx v = a[i + j + half];
                a[i + j] = u + v;
                a[i + j + half] = (u - v) * conj(tw(j * stride, m));
            }
    }
    const double scale = pow(0.5, 0.5 * m);
    for (size_t i = 0; i < n; ++i) a[i] *= scale;
    return 0;
}
int orc_fft_bitrev(double* a, size_t n) { return fft_bitrev_c((cplx*)a, n); }
int orc_fft_bitrev_inv(double* a, size_t n) { return fft_bitrev_inv_c((cplx*)a, n); }

/* ---------------------------------------------------------------- kernels.cpp:25-103 */
double orc_si_bernoulli_1d(double x, double xp, int alpha) {
    const double diff = x - xp;
    const double u1 = diff - floor(diff);
    const double u2 = -diff - floor(-diff);
    double u = u1 < u2 ? u1 : u2;
    if (u >= 1.0) u = 0.0;
    const double pi2 = 9.869604401089358618834491;
    if (alpha == 1) return 2.0 * pi2 * (u * (u - 1.0) + 1.0 / 6.0);
    if (alpha == 2) {
        const double b4 = ((u - 2.0) * u + 1.0) * u * u - 1.0 / 30.0;
        return -(2.0 / 3.0) * pi2 * pi2 * b4;
    }
    return NAN;
}
static uint64_t frac_to_bits(double x) { return (uint64_t)(x * 0x1p53); } /* ld_sequences.cpp:55-58 */

double orc_dsi_order_1d(int alpha, double x, double xp) {
    const uint64_t w = frac_to_bits(x) ^ frac_to_bits(xp);
    if (w == 0) {
        switch (alpha) {
            case 1: return 1.0;
            case 2: return 1.5;
            case 3: return 25.0 / 18.0;
            case 4: return 407.0 / 294.0;
        }
        return NAN;
    }
    const int beta = 53 - (64 - __builtin_clzll(w)) + 1;
    const double u = (double)w * 0x1p-53;
    const double t1 = ldexp(1.0, -beta);
    switch (alpha) {
        case 1: return 1.0 - 3.0 * t1;
        case 2: return -1.0 - beta * u + 2.5 * (1.0 - t1);
        case 3: {
            const double t2 = t1 * t1;
            return -1.0 + beta * u * u - 5.0 * (1.0 - t1) * u + (43.0 / 18.0) * (1.0 - t2);
        }
        case 4: {
            const double t2 = t1 * t1, t3 = t2 * t1;
            double x3 = 0.0; /* kernels.cpp:69-75: set bits from the lowest up */
            uint64_t rem = w;
            while (rem) {
                const int a = 53 - __builtin_ctzll(rem);
                x3 += ldexp(1.0, -3 * a);
                rem &= rem - 1;
            }
            return -1.0 - (2.0 / 3.0) * beta * u * u * u + 5.0 * (1.0 - t1) * u * u - (43.0 / 9.0) * (1.0 - t2) * u +
                   (701.0 / 294.0) * (1.0 - t3) - beta * x3 / 3.0;
        }
    }
    return NAN;
}

typedef struct {
    const OrcDesign* dz;
    const OrcHyper* h;
    int L, d, lattice;
    size_t n[8], off[9], N;
    double* X; /* [N][d] materialised points (LdDesign::X) */
    double R[64];
} Ctx;

/* SpatialKernel::operator() (kernels.cpp:91-103) */
static double spatial(const Ctx* c, const double* x, const double* xp) {
    double prod = c->h->gamma;
    for (int j = 0; j < c->d; ++j) {
        double base;
        if (c->lattice) {
            base = orc_si_bernoulli_1d(x[j], xp[j], c->h->si_alpha);
        } else {
            base = 0.0; /* dsi_walsh_1d: zero weights skipped (kernels.cpp:84-89) */
            for (int a = 1; a <= 4; ++a)
                if (c->h->b[a - 1] != 0.0) base += c->h->b[a - 1] * orc_dsi_order_1d(a, x[j], xp[j]);
        }
        prod *= 1.0 + c->h->eta[j] * base;
    }
    return prod;
}

/* lattice_points / digital_net_points (ld_sequences.cpp:31-87) */
static void points(const OrcDesign* dz, int l, size_t count, double* out) {
    int mgen = 0;
    if (dz->kind == 0)
        while (((uint64_t)1 << mgen) < dz->n_max) ++mgen;
    for (size_t r = 0; r < count; ++r)
        for (int j = 0; j < dz->d; ++j) {
            const uint64_t sh = dz->shift_bits[l * dz->d + j];
            uint64_t bits;
            if (dz->kind == 0) {
                const uint64_t k = orc_bit_reverse(r, mgen);
                const uint64_t frac = ((k * dz->g[j]) & (dz->n_max - 1)) << (53 - mgen);
                bits = (frac + sh) & MASK53;
            } else {
                bits = sh;
                uint64_t rem = r;
                for (int p = 0; rem; ++p, rem >>= 1)
                    if (rem & 1) bits ^= dz->columns[(size_t)j * dz->m_cols + p];
            }
            out[r * dz->d + j] = (double)bits * 0x1p-53;
        }
}

static int ctx_init(Ctx* c, const OrcDesign* dz, const OrcHyper* h) {
    memset(c, 0, sizeof *c);
    c->dz = dz;
    c->h = h;
    c->L = dz->L;
    c->d = dz->d;
    c->lattice = dz->kind == 0;
    c->off[0] = 0;
    for (int l = 0; l < c->L; ++l) {
        c->n[l] = (size_t)1 << dz->m[l];
        c->off[l + 1] = c->off[l] + c->n[l];
        if (l && dz->m[l] > dz->m[l - 1]) return fail(1, "build_spectrum: task sizes must be descending");
    }
    c->N = c->off[c->L];
    c->X = malloc(sizeof(double) * c->N * c->d);
    for (int l = 0; l < c->L; ++l) points(dz, l, c->n[l], c->X + c->off[l] * c->d);
    /* task_gram R = B B^T + diag(t) (kernels.cpp:124-135) */
    for (int a = 0; a < c->L; ++a) {
        if (!(h->t[a] > 0.0)) return fail(1, "task_gram: non-positive diagonal entry");
        for (int b = 0; b < c->L; ++b) {
            double s = 0.0;
            for (int k = 0; k < h->s; ++k) s += h->B[a * h->s + k] * h->B[b * h->s + k];
            c->R[a * c->L + b] = s + (a == b ? h->t[a] : 0.0);
        }
    }
    return 0;
}
static void ctx_free(Ctx* c) { free(c->X); }

static void fwd(cplx* v, size_t n, int lattice) { /* fast_gram.cpp:12-20 */
    if (lattice) {
        fft_bitrev_c(v, n);
        return;
    }
    double* re = malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) re[i] = creal(v[i]);
    orc_fwht(re, n);
    for (size_t i = 0; i < n; ++i) v[i] = re[i];
    free(re);
}
static void inv(cplx* v, size_t n, int lattice) { /* fast_gram.cpp:22-31 */
    if (lattice) {
        fft_bitrev_inv_c(v, n);
        return;
    }
    fwd(v, n, 0);
}
static int pair_index(int L, int l, int lp) { return l * L - l * (l - 1) / 2 + (lp - l); }

/* build_spectrum (fast_gram.cpp:42-89) */
static cplx** spectrum(const Ctx* c) {
    const int L = c->L;
    cplx** lam = calloc((size_t)L * (L + 1) / 2, sizeof(cplx*));
    for (int l = 0; l < L; ++l)
        for (int lp = l; lp < L; ++lp) {
            const size_t nl = c->n[l];
            cplx* col = malloc(sizeof(cplx) * nl);
            const double* x0 = c->X + c->off[lp] * c->d;
            for (size_t i = 0; i < nl; ++i)
                col[i] = c->R[l * L + lp] * spatial(c, c->X + (c->off[l] + i) * c->d, x0);
            fwd(col, nl, c->lattice);
            const double scale = sqrt((double)c->n[lp]);
            for (size_t i = 0; i < nl; ++i) col[i] *= scale;
            if (l == lp)
                for (size_t i = 0; i < nl; ++i) col[i] += c->h->xi[l];
            lam[pair_index(L, l, lp)] = col;
        }
    return lam;
}
static void free_spectrum(cplx** lam, int L) {
    for (int p = 0; p < L * (L + 1) / 2; ++p) free(lam[p]);
    free(lam);
}

int orc_build_spectrum(const OrcDesign* dz, const OrcHyper* h, double* re, double* im) {
    Ctx c;
    if (ctx_init(&c, dz, h)) return 1;
    cplx** lam = spectrum(&c);
    size_t o = 0;
    for (int l = 0; l < c.L; ++l)
        for (int lp = l; lp < c.L; ++lp) {
            const cplx* v = lam[pair_index(c.L, l, lp)];
            for (size_t i = 0; i < c.n[l]; ++i, ++o) {
                re[o] = creal(v[i]);
                im[o] = cimag(v[i]);
            }
        }
    free_spectrum(lam, c.L);
    ctx_free(&c);
    return 0;
}

/* invert_and_logdet (Algorithm 1, fast_gram.cpp:151-263): grid of r x r diagonal blocks */
typedef struct {
    size_t r, base;
    cplx** grid; /* [r*r], NULL = structural zero, each length `base` */
    double logdet;
} Inv;

static int check_positive(cplx* s, size_t n, double* logdet) { /* fast_gram.cpp:167-178 */
    double remax = 0.0;
    for (size_t k = 0; k < n; ++k) remax = fmax(remax, fabs(creal(s[k])));
    for (size_t k = 0; k < n; ++k) {
        if (fabs(cimag(s[k])) > 1e-8 * fmax(1.0, remax)) return fail(1, "invert_and_logdet: non-real Schur complement");
        if (!(creal(s[k]) > 0.0)) return fail(2, "non-positive Schur entry");
        *logdet += log(creal(s[k]));
        s[k] = creal(s[k]);
    }
    return 0;
}

static int invert(const Ctx* c, cplx** lam, Inv* out) {
    const int L = c->L;
    size_t r = 0;
    cplx** A = NULL;
    out->logdet = 0.0;
    for (int l = 0; l < L; ++l) {
        const size_t nl = c->n[l];
        if (l == 0) {
            cplx* s = malloc(sizeof(cplx) * nl);
            memcpy(s, lam[pair_index(L, 0, 0)], sizeof(cplx) * nl);
            int st = check_positive(s, nl, &out->logdet);
            if (st) {
                free(s);
                return st;
            }
            for (size_t k = 0; k < nl; ++k) s[k] = 1.0 / s[k];
            A = calloc(1, sizeof(cplx*));
            A[0] = s;
            r = 1;
            continue;
        }
        const size_t f = c->n[l - 1] / nl; /* refine granularity (fast_gram.cpp:190-206) */
        if (f > 1) {
            const size_t rn = r * f;
            cplx** ref = calloc(rn * rn, sizeof(cplx*));
            for (size_t i = 0; i < r; ++i)
                for (size_t j = 0; j < r; ++j) {
                    cplx* blk = A[i * r + j];
                    if (!blk) continue;
                    for (size_t a = 0; a < f; ++a) {
                        cplx* v = malloc(sizeof(cplx) * nl);
                        memcpy(v, blk + a * nl, sizeof(cplx) * nl);
                        ref[(i * f + a) * rn + (j * f + a)] = v;
                    }
                    free(blk);
                }
            free(A);
            A = ref;
            r = rn;
        }
        /* stage columns B_i (fast_gram.cpp:137-149) */
        const cplx** B = calloc(r, sizeof(cplx*));
        for (int lp = 0; lp < l; ++lp) {
            const cplx* v = lam[pair_index(L, lp, l)];
            const size_t first = c->off[lp] / nl;
            for (size_t cc = 0; cc * nl < c->n[lp]; ++cc) B[first + cc] = v + cc * nl;
        }
        cplx* Lcol = calloc(r * nl, sizeof(cplx));
        for (size_t i = 0; i < r; ++i)
            for (size_t j = 0; j < r; ++j) {
                const cplx* blk = A[i * r + j];
                if (!blk) continue;
                for (size_t k = 0; k < nl; ++k) Lcol[i * nl + k] += blk[k] * B[j][k];
            }
        cplx* S = malloc(sizeof(cplx) * nl);
        memcpy(S, lam[pair_index(L, l, l)], sizeof(cplx) * nl);
        for (size_t i = 0; i < r; ++i)
            for (size_t k = 0; k < nl; ++k) S[k] -= conj(B[i][k]) * Lcol[i * nl + k];
        int st = check_positive(S, nl, &out->logdet);
        if (st) {
            free(S);
            free(Lcol);
            free(B);
            for (size_t q = 0; q < r * r; ++q) free(A[q]);
            free(A);
            return st;
        }
        const size_t rn = r + 1;
        cplx** grown = calloc(rn * rn, sizeof(cplx*));
        for (size_t i = 0; i < r; ++i) {
            for (size_t j = 0; j < r; ++j) {
                cplx* blk = A[i * r + j];
                if (!blk) blk = calloc(nl, sizeof(cplx));
                for (size_t k = 0; k < nl; ++k) {
                    const cplx H = Lcol[i * nl + k] / creal(S[k]);
                    blk[k] += H * conj(Lcol[j * nl + k]);
                }
                grown[i * rn + j] = blk;
            }
            cplx* right = malloc(sizeof(cplx) * nl);
            cplx* bottom = malloc(sizeof(cplx) * nl);
            for (size_t k = 0; k < nl; ++k) {
                const cplx H = Lcol[i * nl + k] / creal(S[k]);
                right[k] = -H;
                bottom[k] = -conj(H);
            }
            grown[i * rn + r] = right;
            grown[r * rn + i] = bottom;
        }
        cplx* corner = malloc(sizeof(cplx) * nl);
        for (size_t k = 0; k < nl; ++k) corner[k] = 1.0 / creal(S[k]);
        grown[r * rn + r] = corner;
        free(A);
        free(S);
        free(Lcol);
        free(B);
        A = grown;
        r = rn;
    }
    out->r = r;
    out->base = c->n[L - 1];
    out->grid = A;
    return 0;
}
static void free_inv(Inv* v) {
    for (size_t q = 0; q < v->r * v->r; ++q) free(v->grid[q]);
    free(v->grid);
}

/* solve (fast_gram.cpp:265-299) */
static int solve(const Ctx* c, const Inv* iv, const double* y, double* out) {
    cplx* z = malloc(sizeof(cplx) * c->N);
    for (int l = 0; l < c->L; ++l) {
        for (size_t k = 0; k < c->n[l]; ++k) z[c->off[l] + k] = y[c->off[l] + k];
        fwd(z + c->off[l], c->n[l], c->lattice);
    }
    cplx* w = calloc(c->N, sizeof(cplx));
    for (size_t i = 0; i < iv->r; ++i)
        for (size_t j = 0; j < iv->r; ++j) {
            const cplx* blk = iv->grid[i * iv->r + j];
            if (!blk) continue;
            for (size_t k = 0; k < iv->base; ++k) w[i * iv->base + k] += blk[k] * z[j * iv->base + k];
        }
    int st = 0;
    for (int l = 0; l < c->L; ++l) {
        inv(w + c->off[l], c->n[l], c->lattice);
        double lim = 0.0, lre = 0.0;
        for (size_t k = 0; k < c->n[l]; ++k) {
            lim = fmax(lim, fabs(cimag(w[c->off[l] + k])));
            lre = fmax(lre, fabs(creal(w[c->off[l] + k])));
            out[c->off[l] + k] = creal(w[c->off[l] + k]);
        }
        /* ORC_RESIDUE_GUARD=0 (tests only): keep the real projection where the reference's guard
         * would throw — BASELINE config 3 at full size, SURVEY.md §8c caveat 1 */
        const char* g = getenv("ORC_RESIDUE_GUARD");
        if (lim > 1e-8 * fmax(1.0, lre) && !(g && g[0] == '0')) st = fail(1, "solve: abnormal imaginary residue");
    }
    free(z);
    free(w);
    return st;
}

/* gram_matvec (fast_gram.cpp:91-131) */
static void matvec(const Ctx* c, cplx** lam, const double* y, double* out) {
    const int L = c->L;
    cplx* z = malloc(sizeof(cplx) * c->N);
    cplx* o = calloc(c->N, sizeof(cplx));
    for (int l = 0; l < L; ++l) {
        for (size_t k = 0; k < c->n[l]; ++k) z[c->off[l] + k] = y[c->off[l] + k];
        fwd(z + c->off[l], c->n[l], c->lattice);
    }
    for (int l = 0; l < L; ++l)
        for (int lp = l; lp < L; ++lp) {
            const cplx* v = lam[pair_index(L, l, lp)];
            const size_t nl = c->n[l], nlp = c->n[lp];
            if (l == lp) {
                for (size_t k = 0; k < nl; ++k) o[c->off[l] + k] += v[k] * z[c->off[l] + k];
                continue;
            }
            for (size_t cc = 0; cc * nlp < nl; ++cc)
                for (size_t k = 0; k < nlp; ++k) {
                    const size_t row = cc * nlp + k;
                    o[c->off[l] + row] += v[row] * z[c->off[lp] + k];
                    o[c->off[lp] + k] += conj(v[row]) * z[c->off[l] + row];
                }
        }
    for (int l = 0; l < L; ++l) {
        inv(o + c->off[l], c->n[l], c->lattice);
        for (size_t k = 0; k < c->n[l]; ++k) out[c->off[l] + k] = creal(o[c->off[l] + k]);
    }
    free(z);
    free(o);
}

static void extract_pi(const Ctx* c, const Inv* iv, double* Pi) { /* fast_gram.cpp:311-335 */
    for (int l = 0; l < c->L; ++l)
        for (int lp = 0; lp < c->L; ++lp) {
            const cplx* blk = iv->grid[(c->off[l] / iv->base) * iv->r + c->off[lp] / iv->base];
            Pi[l * c->L + lp] = blk ? sqrt((double)c->n[l] * (double)c->n[lp]) * creal(blk[0]) : 0.0;
        }
}

static void small_solve(int n, double* A, double* b) { /* Gaussian elimination, partial pivoting */
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (fabs(A[i * n + k]) > fabs(A[p * n + k])) p = i;
        for (int j = 0; j < n; ++j) {
            double t = A[k * n + j];
            A[k * n + j] = A[p * n + j];
            A[p * n + j] = t;
        }
        double t = b[k];
        b[k] = b[p];
        b[p] = t;
        for (int i = k + 1; i < n; ++i) {
            const double f = A[i * n + k] / A[k * n + k];
            for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
            b[i] -= f * b[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < n; ++k) s -= A[i * n + k] * b[k];
        b[i] = s / A[i * n + i];
    }
}

int orc_invert_solve(const OrcDesign* dz, const OrcHyper* h, const double* b, double* x, double* kb, double* logdet,
                     double* trace, double* Pi) {
    Ctx c;
    if (ctx_init(&c, dz, h)) return 1;
    cplx** lam = spectrum(&c);
    Inv iv;
    int st = invert(&c, lam, &iv);
    if (st) {
        free_spectrum(lam, c.L);
        ctx_free(&c);
        return st;
    }
    *logdet = iv.logdet;
    if (x) st = solve(&c, &iv, b, x);
    if (kb) matvec(&c, lam, b, kb);
    if (trace) { /* trace_inverse (fast_gram.cpp:301-309) */
        double tr = 0.0;
        for (size_t i = 0; i < iv.r; ++i)
            if (iv.grid[i * iv.r + i])
                for (size_t k = 0; k < iv.base; ++k) tr += creal(iv.grid[i * iv.r + i][k]);
        *trace = tr;
    }
    if (Pi) extract_pi(&c, &iv, Pi);
    free_inv(&iv);
    free_spectrum(lam, c.L);
    ctx_free(&c);
    return st;
}

/* refresh + loss_value NMLL (gp_core.cpp:67-141, 197-211); no noise escalation */
static int fit_core(Ctx* c, const double* y, OrcFit* out, double* cvec, Inv* keep) {
    cplx** lam = spectrum(c);
    Inv iv;
    int st = invert(c, lam, &iv);
    free_spectrum(lam, c->L);
    if (st) return st;
    const int L = c->L;
    double tau[8];
    if (L == 1) {
        double mean = 0.0;
        for (size_t i = 0; i < c->N; ++i) mean += y[i];
        tau[0] = mean / (double)c->N;
    } else {
        double* w = malloc(sizeof(double) * c->N);
        st = solve(c, &iv, y, w);
        double Pi[64], rhs[8];
        extract_pi(c, &iv, Pi);
        for (int l = 0; l < L; ++l) {
            rhs[l] = 0.0;
            for (size_t k = c->off[l]; k < c->off[l + 1]; ++k) rhs[l] += w[k];
        }
        small_solve(L, Pi, rhs);
        for (int l = 0; l < L; ++l) tau[l] = rhs[l];
        free(w);
    }
    double* r = malloc(sizeof(double) * c->N);
    for (int l = 0; l < L; ++l)
        for (size_t k = c->off[l]; k < c->off[l + 1]; ++k) r[k] = y[k] - tau[l];
    double* cc = cvec ? cvec : malloc(sizeof(double) * c->N);
    if (!st) st = solve(c, &iv, r, cc);
    double quad = 0.0;
    for (size_t i = 0; i < c->N; ++i) quad += r[i] * cc[i];
    out->quad = quad;
    out->logdet = iv.logdet;
    out->nll = quad + iv.logdet;
    for (int l = 0; l < L; ++l) out->tau[l] = tau[l];
    free(r);
    if (!cvec) free(cc);
    if (keep) *keep = iv;
    else free_inv(&iv);
    return st;
}

int orc_fit(const OrcDesign* dz, const OrcHyper* h, const double* y, OrcFit* out, double* c_out) {
    Ctx c;
    if (ctx_init(&c, dz, h)) return 1;
    int st = fit_core(&c, y, out, c_out, NULL);
    ctx_free(&c);
    return st;
}

/* posterior_mean_batch / kernel_against_data (gp_core.cpp:386-421) */
int orc_posterior_mean(const OrcDesign* dz, const OrcHyper* h, const double* y, int task, const double* X,
                       size_t count, double* out) {
    Ctx c;
    if (ctx_init(&c, dz, h)) return 1;
    OrcFit f;
    double* cv = malloc(sizeof(double) * c.N);
    int st = fit_core(&c, y, &f, cv, NULL);
    if (!st)
        for (size_t q = 0; q < count; ++q) {
            double acc = 0.0;
            for (int lp = 0; lp < c.L; ++lp)
                for (size_t i = 0; i < c.n[lp]; ++i)
                    acc += c.R[task * c.L + lp] * spatial(&c, X + q * c.d, c.X + (c.off[lp] + i) * c.d) *
                           cv[c.off[lp] + i];
            out[q] = f.tau[task] + acc;
        }
    free(cv);
    ctx_free(&c);
    return st;
}

/* posterior_cov with x = x' (gp_core.cpp:423-445): one full solve per query */
int orc_posterior_var(const OrcDesign* dz, const OrcHyper* h, const double* y, int task, const double* X,
                      size_t count, double* out) {
    Ctx c;
    if (ctx_init(&c, dz, h)) return 1;
    OrcFit f;
    Inv iv;
    int st = fit_core(&c, y, &f, NULL, &iv);
    if (st) {
        ctx_free(&c);
        return st;
    }
    double* k = malloc(sizeof(double) * c.N);
    double* w = malloc(sizeof(double) * c.N);
    for (size_t q = 0; q < count && !st; ++q) {
        const double* x = X + q * c.d;
        for (int j = 0; j < c.L; ++j)
            for (size_t i = 0; i < c.n[j]; ++i)
                k[c.off[j] + i] = c.R[task * c.L + j] * spatial(&c, x, c.X + (c.off[j] + i) * c.d);
        st = solve(&c, &iv, k, w);
        double acc = 0.0;
        for (size_t i = 0; i < c.N; ++i) acc += k[i] * w[i];
        out[q] = c.R[task * c.L + task] * spatial(&c, x, x) - acc;
    }
    free(k);
    free(w);
    free_inv(&iv);
    ctx_free(&c);
    return st;
}

/* multitask_cubature (cubature.cpp:52-75), internal order */
int orc_cubature(const OrcDesign* dz, const OrcHyper* h, const double* y, double* mu, double* Sigma) {
    Ctx c;
    if (ctx_init(&c, dz, h)) return 1;
    OrcFit f;
    Inv iv;
    double* cv = malloc(sizeof(double) * c.N);
    int st = fit_core(&c, y, &f, cv, &iv);
    if (!st) {
        const int L = c.L;
        const double g = h->gamma;
        double etc[8], Pi[64], RP[64];
        for (int l = 0; l < L; ++l) {
            etc[l] = 0.0;
            for (size_t k = c.off[l]; k < c.off[l + 1]; ++k) etc[l] += cv[k];
        }
        extract_pi(&c, &iv, Pi);
        for (int a = 0; a < L; ++a) {
            double s = 0.0;
            for (int b = 0; b < L; ++b) s += c.R[a * L + b] * etc[b];
            mu[a] = f.tau[a] + g * s;
        }
        for (int a = 0; a < L; ++a)
            for (int b = 0; b < L; ++b) {
                double s = 0.0;
                for (int k = 0; k < L; ++k) s += c.R[a * L + k] * Pi[k * L + b];
                RP[a * L + b] = s;
            }
        for (int a = 0; a < L; ++a)
            for (int b = 0; b < L; ++b) {
                double s = 0.0;
                for (int k = 0; k < L; ++k) s += RP[a * L + k] * c.R[k * L + b];
                Sigma[a * L + b] = g * c.R[a * L + b] - g * g * s;
            }
        for (int a = 0; a < L; ++a)
            for (int b = a + 1; b < L; ++b)
                Sigma[a * L + b] = Sigma[b * L + a] = 0.5 * (Sigma[a * L + b] + Sigma[b * L + a]);
        for (int a = 0; a < L; ++a)
            if (Sigma[a * L + a] < 0.0 && Sigma[a * L + a] > -1e-12) Sigma[a * L + a] = 0.0;
        free_inv(&iv);
    }
    free(cv);
    ctx_free(&c);
    return st;
}

int orc_design_points(const OrcDesign* dz, double* out) {
    size_t off = 0;
    for (int l = 0; l < dz->L; ++l) {
        const size_t n = (size_t)1 << dz->m[l];
        points(dz, l, n, out + off * dz->d);
        off += n;
    }
    return 0;
}
