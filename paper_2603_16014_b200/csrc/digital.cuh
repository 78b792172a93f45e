// Equal-n digital-net (DSI / FWHT) fit in three fused kernels — the configuration-2/5 hot path.
//
//   K1 k_dig_col_fwd : generator q_o(i) (design-time kappa table or on the fly) x column FWHT,
//                      one vector per pair-offset CLASS o (pairs with equal Delta_a ^ Delta_b share
//                      q — all diagonal pairs do), not per pair
//   K2 k_dig_mid     : row FWHT of every class + spectrum epilogue per pair (R, xi) + per-frequency
//                      T x T LDL^H solve (logdet, quad, M = Lam^-1 - chat chat^H) + dR partials
//                      sum_k M_p qhat_o (Parseval) + Z_o = sum_{p in o} w_p R_p M_p + inverse row FWHT
//   K3 k_dig_col_inv : inverse column FWHT -> H Z_o -> dot with dq_o/deta -> partials,
//                      last CTA reduces everything into the result record (class_sums_out)
//
// n = N1 * N2 (natural index i = j1 * N2 + j2); FWHT over the two bit groups commutes, and the
// spectrum index after both passes is natural, so K2 owns the frequencies {k1 * N2 + k2}: all
// pairs of one frequency meet in one CTA and the solve needs no extra HBM round trip — the
// fused four-step of SURVEY.md §8d (8n(6P+T) bytes instead of 8n(8P+T)).
#pragma once

#include <vector>

#include "kernels.cuh"

namespace fmtgp {

struct DigGeo {
    int m, l1, l2;   // n = 2^m = 2^l1 (columns) * 2^l2 (rows)
    int lc;          // log2 columns per K1/K3 CTA (tile = 2^(l1 + lc) <= 2^11)
    int nt_col, nt_mid;
    int nblk_col;    // K1/K3 CTAs per vector
    static bool make(int m, int V, DigGeo& g, long long total_vecs = 0, int d = 0);  // V rows per K2 CTA
};

// Hyperparameter values carried in the kernel parameters (one candidate): no H2D copy node in
// the fit's graph; the captured kernel nodes are re-parameterised per fit (dig_graph_update).
struct DigHyperVals {
    double eta[MAXD];
    double gamma;
    double coef[MAXP], xi[MAXP], Rpair[MAXP];
};

struct DigArgs {
    int T, P, d, nc;
    int V;                    // distinct pair-offset classes (transforms run per class)
    long long n;
    Spatial sp;
    PointGen pg;
    const uint64_t* cofs;     // [V][MAXD] class offsets
    const double* kap;        // design-time table [V][d][n] (nullptr: evaluate on the fly)
    const int* pair_ofs;      // [P] pair -> class
    const double* eta;        // [nc][d]
    const double* gamma;      // [nc]
    const double* coef;       // [nc][P]  R_ab
    const double* xi;         // [nc][P]
    const double* Rpair;      // [nc][P]
    const int* pair_a;
    const int* pair_b;
    const double* yhat;       // [T][n]
    double* Y;                // [nc][V][n] intermediate (column pass out, row pass in/out)
    double* lam_out;          // [nc][P][n] spectrum (nullptr: skip)
    double* chat_out;         // [T][n] chat of candidate 0 (nullptr: skip)
    double* part_mid;         // [nc][nrows][2 + P]  logdet, quad, sum_k M_p qhat_o (class_sums_out)
    double* part_dot;         // [nc][V][nblk_col][MAXD+1]
    int* bad;                 // [nc] first failing slot, 0x7f7f7f7f none
    unsigned long long* imre; // [nc][MAXT][2]
    unsigned int* counter;    // [nc + nc*V] last-CTA tickets (self-resetting)
    double* vec_sum;          // [nc][V][MAXD+1] per-class gradient sums
    double* out;              // [nc][NOUT]
    int want_grad;
    unsigned long long* trace = nullptr;  // FMTGP_TRACE diagnostics: globaltimer marks (see dig_trace)
    // zero-copy result record (tail == 1): the last CTA writes the record straight into the
    // mapped pinned host block and copies the flags / tau words after it (no D2H copy node)
    double* zc_res = nullptr;     // mapped host result block (device alias), nullptr: off
    const double* res_dev = nullptr;  // the device result block (flags / tau source)
    int res_flags_off = 0, res_len = 0;  // doubles before the flags / whole block
    // completion word in mapped host memory: after the record (system fence) the last CTA stores
    // `seq`, and the host returns as soon as it sees it instead of waiting for the graph to retire
    volatile unsigned long long* done_flag = nullptr;
    unsigned long long seq = 0;
    int cpb = 1;
    int use_hv = 0;           // hyperparameters from hv (candidate 0) instead of the pointers
    DigHyperVals hv;              // candidates per K1/K3 CTA (the kappa tile is read once per CTA)
    int tail = 1;             // 1: last CTA of K3 reduces; 0: separate finalize kernel; 2: same, PDL-launched
    int stage_tail = 1;       // the last CTA stages the partials in smem (when they fit in the column tile)
};

// design-time kappa table: kap[o][j][i] = dsi_walsh(z_i ^ off_o[j], b)
void dig_kappa_table(const Spatial& sp, const PointGen& pg, const uint64_t* d_ofs /*[nofs][MAXD]*/, int nofs,
                     long long n, double* kap, cudaStream_t s);
void dig_fit(const DigGeo& g, const DigArgs& a, cudaStream_t s);

// Launch records of dig_fit (set `dig_rec` before a stream capture): the kernels all take DigArgs
// first, so a captured graph can be re-parameterised with new hyperparameter values.
struct DigLaunchRec {
    const void* func;
    dim3 grid, block;
    size_t smem;
    DigArgs a;
    int ints[4];
    int nints;
};
extern thread_local std::vector<DigLaunchRec>* dig_rec;

}  // namespace fmtgp
