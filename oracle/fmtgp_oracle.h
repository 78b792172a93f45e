/* CPU restatement of the reference fast-MTGP hot path (TEST INFRASTRUCTURE).
 *
 * Plain C11 port of /root/reference/proj/src/{transforms,kernels,ld_sequences,fast_gram,
 * gp_core,cubature}.cpp restricted to the north-star path; each function cites the
 * reference lines it follows.  Used only by tests/ (checker), __graft_entry__.smoke()
 * and bench.py's cpu_baseline fallback when oracle/_ref is unavailable.  Pinned against
 * the reference's own known-answer tests (tests/test_oracle_kats.py) and against golden
 * vectors produced by the reference library itself (tests/golden/, tools/make_golden.py).
 */
#ifndef FMTGP_ORACLE_H
#define FMTGP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* identical layout to fmtgp_design / RefDesign */
typedef struct OrcDesign {
    int kind, d, L;
    const int* m;
    const uint64_t* g;
    uint64_t n_max;
    const uint64_t* columns;
    int m_cols;
    const uint64_t* shift_bits;
} OrcDesign;

typedef struct OrcHyper {
    double gamma;
    const double* eta;
    int si_alpha;
    double b[4];
    const double* B;
    int s;
    const double* t;
    const double* xi;
} OrcHyper;

typedef struct OrcFit {
    double nll, logdet, quad;
    double tau[8];
} OrcFit;

/* status: 0 ok, 1 FastMtgpError, 2 SchurBreakdown */
const char* orc_last_error(void);
uint64_t orc_rand_u64(uint64_t seed, uint64_t stream, uint64_t counter);
double orc_normal(uint64_t seed, uint64_t stream, uint64_t k);
uint64_t orc_bit_reverse(uint64_t i, int m);
int orc_fwht(double* a, size_t n);
int orc_fft_bitrev(double* a_interleaved, size_t n);
int orc_fft_bitrev_inv(double* a_interleaved, size_t n);
double orc_si_bernoulli_1d(double x, double xp, int alpha);
double orc_dsi_order_1d(int alpha, double x, double xp);
int orc_design_points(const OrcDesign* dz, double* out);
int orc_build_spectrum(const OrcDesign* dz, const OrcHyper* h, double* re, double* im);
int orc_invert_solve(const OrcDesign* dz, const OrcHyper* h, const double* b, double* x, double* kb, double* logdet,
                     double* trace, double* Pi);
int orc_fit(const OrcDesign* dz, const OrcHyper* h, const double* y, OrcFit* out, double* c);
int orc_posterior_mean(const OrcDesign* dz, const OrcHyper* h, const double* y, int task, const double* X,
                       size_t count, double* out);
int orc_posterior_var(const OrcDesign* dz, const OrcHyper* h, const double* y, int task, const double* X,
                      size_t count, double* out);
int orc_cubature(const OrcDesign* dz, const OrcHyper* h, const double* y, double* mu, double* Sigma);

#ifdef __cplusplus
}
#endif
#endif
