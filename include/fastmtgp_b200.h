/* fastmtgp-b200 — C ABI of the B200 fast multitask-GP fit path (sm_100a, fp64).
 *
 * Drop-in boundary for the reference's structured-Gram seam
 * (/root/reference/proj/include/fastmtgp/fast_gram.hpp:34-70) and for the model-level
 * hot path it serves (gp_core.hpp:46-83).  Plain pointers and sizes only; host arrays
 * are owned by the caller, device memory by the model handle.  Every entry point
 * returns an fmtgp status code; fmtgp_last_error() holds the thread-local message.
 *
 * Conventions:
 *   - task-indexed inputs/outputs are in INTERNAL order (descending n, stable), exactly
 *     what fast_gram.hpp's functions take (R_internal, xi_internal; gp_core.cpp:19-32);
 *   - observation / coefficient vectors are length N = sum n_l, task blocks in internal
 *     order, points of a task in the design's natural (radical-inverse) order;
 *   - pair (l, lp), l <= lp, enumerated row by row (fast_gram.cpp:35-40).
 */
#ifndef FASTMTGP_B200_H
#define FASTMTGP_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FMTGP_API __attribute__((visibility("default")))
#else
#define FMTGP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (common.hpp:16-22 exception mapping) */
#define FMTGP_OK 0
#define FMTGP_ERR_INVALID 1         /* FastMtgpError: bad sizes / arguments               */
#define FMTGP_ERR_SCHUR 2           /* SchurBreakdown: non-positive Schur pivot (retryable) */
#define FMTGP_ERR_NONREAL 3         /* FastMtgpError: non-real Schur complement / residue  */
#define FMTGP_ERR_CUDA 4            /* CUDA runtime failure                               */
#define FMTGP_ERR_OOM 5             /* device allocation failed                           */
#define FMTGP_ERR_UNSUPPORTED 6     /* valid input outside what this build implements     */

#define FMTGP_MAX_D 16
#define FMTGP_MAX_T 8

/* Design: LdDesign (ld_sequences.hpp:56-77) without materialised points — the kernels
 * regenerate every coordinate from the generator.  Layout identical to the oracle's
 * RefDesign (oracle/ref_capi.cpp). */
typedef struct fmtgp_design {
    int kind;                  /* 0: shifted rank-1 lattice (SI kernel), 1: digital net (DSI) */
    int d;                     /* dimension, <= FMTGP_MAX_D                                   */
    int L;                     /* tasks, <= FMTGP_MAX_T                                       */
    const int* m;              /* [L] log2 sizes, internal (descending) order                  */
    const uint64_t* g;         /* lattice: generating vector [d], g[0] == 1                    */
    uint64_t n_max;            /* lattice: power of two >= 2^m[0]                              */
    const uint64_t* columns;   /* digital: [d * m_cols] 53-bit msb-aligned direction numbers   */
    int m_cols;                /* digital: columns per dimension, >= m[0]                      */
    const uint64_t* shift_bits;/* [L * d] 53-bit per-task shifts (internal order)             */
} fmtgp_design;

/* Hyperparams (kernels.hpp:21-31), task-indexed fields in INTERNAL order. */
typedef struct fmtgp_hyper {
    double gamma;
    const double* eta;   /* [d] */
    int si_alpha;        /* lattice: 1 -> B2, 2 -> B4 */
    double b[4];         /* digital: Walsh order weights */
    const double* B;     /* [L * s] row-major task factor, R = B B^T + diag(t) */
    int s;
    const double* t;     /* [L] > 0 */
    const double* xi;    /* [L] >= 0 nugget */
} fmtgp_hyper;

/* SpatialKernel (kernels.hpp:53-66) for the explicit-R seam entry point. */
typedef struct fmtgp_spatial {
    double gamma;
    const double* eta;   /* [d] */
    int si_alpha;
    double b[4];
} fmtgp_spatial;

/* One NLL evaluation: loss_value (gp_core.cpp:197-227) plus the analytic gradient that
 * replaces the reference's central finite differences (gp_core.cpp:341-351). */
typedef struct fmtgp_result {
    double nll;                 /* (y - E tau)^T K^-1 (y - E tau) + log|K| (no 1/2, no N log 2pi) */
    double logdet;
    double quad;
    double dgamma;              /* dNLL/dgamma                                          */
    double deta[FMTGP_MAX_D];   /* dNLL/deta_j                                          */
    double dR[FMTGP_MAX_T * FMTGP_MAX_T]; /* symmetric G: dNLL = sum_ab G_ab dR_ab (L x L, stride L) */
    double dB[FMTGP_MAX_T * FMTGP_MAX_T]; /* dNLL/dB = 2 G B   (L x s, row-major)       */
    double dt[FMTGP_MAX_T];     /* dNLL/dt_l = G_ll                                     */
    double tau[FMTGP_MAX_T];    /* closed-form NMLL prior means (internal order)        */
    double xi_scale;            /* nugget escalation factor applied (10^attempts)       */
    int escalations;            /* SchurBreakdown retries used (gp_core.cpp:98-127)     */
    int status;                 /* FMTGP_OK or the per-candidate failure code           */
} fmtgp_result;

typedef struct fmtgp_model* fmtgp_model_t;

FMTGP_API const char* fmtgp_last_error(void);
FMTGP_API int fmtgp_abi_version(void);

/* ---- model: device-resident design, observations and workspace ------------------- */
FMTGP_API int fmtgp_model_create(const fmtgp_design* design, int device, int max_candidates, fmtgp_model_t* out);
FMTGP_API int fmtgp_model_destroy(fmtgp_model_t model);
/* y: host [N] (internal order).  Uploads, computes yhat = blockdiag(V̄) y once (cached,
 * BASELINE config 5 "FWHT of y computed once") and the closed-form tau. */
FMTGP_API int fmtgp_model_set_y(fmtgp_model_t model, const double* y);
/* same from a device pointer (no host round trip) */
FMTGP_API int fmtgp_model_set_y_device(fmtgp_model_t model, const double* y_dev);
/* benchmark observations on the device (bench.cpp:84-101, problems.cpp): y = problem(level
 * user_of_internal[l] + 1, x_{l,i}) + noise * N(0,1) (rng::normal(seed, 0x401 + user, i)) at the
 * model's own design points, then the same yhat / tau as set_y.  problem: "rosenbrock" (d 2, 3
 * fidelities), "ackley" (4, 2), "borehole" (8, 2), "elliptic" (16, 3).  y_host [N] optional. */
FMTGP_API int fmtgp_model_problem_y(fmtgp_model_t model, const char* problem, const int* user_of_internal,
                                    double noise, uint64_t seed, double* y_host);
/* the same problems at arbitrary points, on the device (eval_batch, problems.cpp:145-154): out[i] =
 * problem(level, X[i*d .. i*d+d-1]); X host [count][d] with the problem's d, out host [count].
 * The held-out truth of the benchmark's l2 error (bench.cpp:159-170). */
FMTGP_API int fmtgp_problem_eval(const char* problem, int level, const double* X, uint64_t count, double* out,
                                 int device);
/* stream the model's work is ordered on (cudaStream_t as void*) */
FMTGP_API void* fmtgp_model_stream(fmtgp_model_t model);

/* ---- fast_gram.hpp seam ------------------------------------------------------------ */
/* build_spectrum (fast_gram.cpp:42-89): Lam_{l,lp} for the hyperparameters. */
FMTGP_API int fmtgp_build_spectrum(fmtgp_model_t model, const fmtgp_hyper* h);
/* build_spectrum with the reference's exact argument list (fast_gram.hpp:34-36):
 * R_internal [L * L] row-major task Gram, spatial kernel, xi_internal [L]. */
FMTGP_API int fmtgp_build_spectrum_R(fmtgp_model_t model, const double* R_internal, const fmtgp_spatial* spatial,
                                     const double* xi_internal);
/* copy pair (l <= lp) back in natural frequency order, length n_l (tests / small N) */
FMTGP_API int fmtgp_spectrum_read(fmtgp_model_t model, int l, int lp, double* re, double* im);
/* invert_and_logdet (fast_gram.cpp:151-263): factorises the current spectrum.
 * FMTGP_ERR_SCHUR on a non-positive pivot, FMTGP_ERR_NONREAL on a non-real one. */
FMTGP_API int fmtgp_invert_and_logdet(fmtgp_model_t model, double* logdet);
/* solve (fast_gram.cpp:265-299): x = K^-1 b, host arrays [N] */
FMTGP_API int fmtgp_solve(fmtgp_model_t model, const double* b, double* x);
/* gram_matvec (fast_gram.cpp:91-131): out = K b */
FMTGP_API int fmtgp_gram_matvec(fmtgp_model_t model, const double* b, double* out);
/* extract_pi_h (fast_gram.cpp:311-335): Pi = E^T K^-1 E, [L * L] row-major */
FMTGP_API int fmtgp_extract_pi(fmtgp_model_t model, double* Pi);
/* H of extract_pi_h (fast_gram.cpp:311-335, fast_gram.hpp:64-68): H_lk = sqrt(n_l) (Lam^-1)_{N_{l-1}, k n_L},
 * [L * r] row-major complex (re / im), r = N / n_{L-1} (equal n: r = L) */
FMTGP_API int fmtgp_extract_h(fmtgp_model_t model, double* H_re, double* H_im);
/* frequencies [k0, k0 + count) of pair (l <= lp) in natural order (fmtgp_spectrum_read for a range) */
FMTGP_API int fmtgp_spectrum_read_range(fmtgp_model_t model, int l, int lp, int64_t k0, int64_t count, double* re,
                                        double* im);
/* trace_inverse (fast_gram.cpp:301-309); unequal n by selected inversion of the fold */
FMTGP_API int fmtgp_trace_inverse(fmtgp_model_t model, double* tr);

/* ---- gp_core hot path -------------------------------------------------------------- */
/* refresh + loss_value (NMLL) [+ analytic gradient] with SchurBreakdown noise escalation
 * (xi x10, at most 6 retries; zero xi -> 1e-12 * scale, gp_core.cpp:98-127). */
FMTGP_API int fmtgp_nll(fmtgp_model_t model, const fmtgp_hyper* h, int want_grad, fmtgp_result* out);
/* ncand independent hyperparameter candidates in one sweep (BASELINE config 5); each
 * result carries its own status / escalation count. */
FMTGP_API int fmtgp_nll_batch(fmtgp_model_t model, int ncand, const fmtgp_hyper* h, int want_grad, fmtgp_result* out);
/* coefficients c = K^-1 (y - E tau) of the last fmtgp_nll call (GpModel::c), host [N] */
FMTGP_API int fmtgp_coefficients(fmtgp_model_t model, double* c);

/* ---- fit: the reference's iRprop- loop (gp_core.cpp:317-382) driven by the analytic gradient --
 * Parameter vector theta (ParamPack, gp_core.cpp:243-304): [log gamma, log eta[d], B[L*s] (row-major),
 * log t[L], and for digital designs log b[4]].  One NLL+gradient evaluation per step instead of the
 * reference's 2*P_theta+1 loss evaluations; iRprop- constants 0.1 / 1.2 / 0.5 / [1e-6, 1].
 * loss_trace[k] = best loss after step k; theta_best receives the best parameters; the model is
 * left refreshed at them (coefficients / posterior / cubature follow). */
typedef struct fmtgp_fit_report {
    int steps;
    int n_params;
    int escalations;            /* noise escalations of the final refresh              */
    double final_loss;          /* best loss                                            */
    double tau[FMTGP_MAX_T];    /* prior means at the best parameters (internal order)  */
} fmtgp_fit_report;
/* GCV loss (loss_value(model, LossKind::gcv), gp_core.cpp:213-226): ||c||^2 / (tr K^-1)^2 with the
 * reference's escalation, c = K^-1 (y - E tau_GCV); unequal n through H and the selected-inversion
 * trace.  num / tr optional. */
FMTGP_API int fmtgp_gcv(fmtgp_model_t model, const fmtgp_hyper* h, double* loss, double* num, double* tr);
FMTGP_API int fmtgp_fit_param_count(fmtgp_model_t model, int s, int* n_params);
FMTGP_API int fmtgp_fit(fmtgp_model_t model, const fmtgp_hyper* init, int steps, double* theta_best,
                        double* loss_trace, double* step_seconds, fmtgp_fit_report* report);
/* posterior_mean_batch (gp_core.cpp:409-421) for the last fmtgp_nll hyperparameters:
 * X host [count * d], task internal index */
FMTGP_API int fmtgp_posterior_mean(fmtgp_model_t model, int task, const double* X, int64_t count, double* out);
/* posterior variance K((t,x),(t,x)) - k^T K^-1 k (posterior_cov, gp_core.cpp:423-445, x = x') */
FMTGP_API int fmtgp_posterior_var(fmtgp_model_t model, int task, const double* X, int64_t count, double* out);
/* posterior_cov (gp_core.cpp:423-445) for count pairs: out[i] = K((task,X[i]),(task2,Xp[i])) - k^T K^-1 k'
 * (both kernel columns folded forward on the device; X, Xp host [count * d]) */
FMTGP_API int fmtgp_posterior_cov(fmtgp_model_t model, int task, const double* X, int task2, const double* Xp,
                                  int64_t count, double* out);
/* multitask_cubature (cubature.cpp:52-75): mu [L], Sigma [L * L] (internal order) */
FMTGP_API int fmtgp_cubature(fmtgp_model_t model, double* mu, double* Sigma);

/* ---- frequency-sharded lattice fit over `world` ranks -----------------
 * No reference counterpart (the reference is single-process): the config-4 extension.  Each rank
 * holds a model of the full design (y replicated, fmtgp_model_set_y) and runs three phases on
 * its stream; between them the caller moves the exchange blocks with an all-to-all of equal
 * chunks (world blocks of exchange_elems / world complex values, block h goes to rank h):
 *   begin(Y)  generator x column FFT of this rank's column blocks into Y
 *   all-to-all Y -> Y2
 *   mid(Y2)   row FFT + per-frequency solve + inverse row FFT of this rank's row clusters, in place
 *   all-to-all Y2 -> Y3
 *   end(Y3)   inverse column FFT + gradient dot; rec = [NOUT sums | first bad slot | non-real maxima]
 * The caller combines the ranks' records (sum the first NOUT entries in rank order, min of the
 * bad slot, max of the maxima) and calls finish for the fmtgp_result (status SCHUR -> escalate
 * xi_scale x10 as fmtgp_nll does, gp_core.cpp:98-127). */
#define FMTGP_SHARD_REC_LEN (4 + FMTGP_MAX_D + FMTGP_MAX_T * FMTGP_MAX_T + 1 + 2 * FMTGP_MAX_T)
FMTGP_API int fmtgp_shard_setup(fmtgp_model_t model, int rank, int world, int64_t* exchange_elems);
FMTGP_API int fmtgp_shard_begin(fmtgp_model_t model, const fmtgp_hyper* h, int want_grad, double xi_scale,
                                void* Y);
FMTGP_API int fmtgp_shard_mid(fmtgp_model_t model, void* Y2);
FMTGP_API int fmtgp_shard_end(fmtgp_model_t model, const void* Y3, double* rec);
FMTGP_API int fmtgp_shard_finish(fmtgp_model_t model, const fmtgp_hyper* h, const double* rec, int want_grad,
                                 double xi_scale, int escalations, fmtgp_result* out);
/* Pipelined exchange: split each all-to-all into `chunks` (a power of two dividing the rank's
 * column blocks and row pairs; 1 = the unchunked phases above).  Chunk k is the contiguous range
 * [k, k+1) * exchange_elems / chunks of every buffer (itself `world` equal blocks), so
 *   for k: begin_chunk(k) -> Y;   all-to-all of chunk k, Y -> Y2   (overlaps begin_chunk(k+1))
 *   for k: mid_chunk(Y2, Y, k);   all-to-all of chunk k, Y -> Y3   (overlaps mid_chunk(k+1))
 *   end(Y3)
 * begin_chunk(0) stages the hyperparameters; every mid_chunk needs all forward chunks received,
 * and writes Y (free once the forward exchange is done) — never Y2 in place. */
FMTGP_API int fmtgp_shard_chunks(fmtgp_model_t model, int chunks);
FMTGP_API int fmtgp_shard_begin_chunk(fmtgp_model_t model, const fmtgp_hyper* h, int want_grad, double xi_scale,
                                      void* Y, int chunk);
FMTGP_API int fmtgp_shard_mid_chunk(fmtgp_model_t model, void* Y2, void* Yout, int chunk);

/* ---- measurement: per-kernel CUDA-event timing on the model's stream ---------------- */
/* iters fmtgp_nll calls from a C loop, each bracketed by CUDA events on the model's stream after an
 * optional L2 flush of flush_bytes (outside the events): ms[iters] device ms per call, wall_us the
 * mean host wall time per call */
FMTGP_API int fmtgp_bench_nll(fmtgp_model_t model, const fmtgp_hyper* h, int want_grad, int iters,
                              size_t flush_bytes, double* ms, double* wall_us);
FMTGP_API int fmtgp_profile_enable(fmtgp_model_t model, int on);  /* also resets the tallies */
/* idx-th kernel name seen since enable, its summed device ms and launch count;
 * FMTGP_ERR_INVALID past the last entry */
FMTGP_API int fmtgp_profile_read(fmtgp_model_t model, int idx, char* name, int name_len, double* total_ms,
                                 int* launches);

#ifdef __cplusplus
}
#endif
#endif /* FASTMTGP_B200_H */
