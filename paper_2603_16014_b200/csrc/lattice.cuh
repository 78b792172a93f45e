// Equal-n rank-1-lattice (SI / real FFT) fit in three fused kernels — the configuration-4 hot path.
//
//   L1 k_lat_col_fwd : generator q_o(2j), q_o(2j+1) on the fly (32-bit lattice arithmetic, exact)
//                      packed as z(j) = q(2j) + i q(2j+1) x column FFT x four-step twiddle, one
//                      vector per pair-offset CLASS o (all diagonal pairs share offset 0)
//   L2 k_lat_mid     : 2-CTA cluster owning the Hermitian partner rows (r, N1 - r): row FFT of every
//                      class, real-FFT post-processing of each frequency PAIR (k, N' - k) by one
//                      thread (own + partner smem over DSMEM), per-frequency T x T LDL^H solve
//                      (logdet, quad, M = Lam^-1 - chat chat^H, Parseval dR partials, class adjoints
//                      Z_o), inverse pre-processing written back in place, inverse row FFT
//   L3 k_lat_col_inv : inverse column FFT -> W -> dot with dq_o/deta (generator on the fly) ->
//                      partials; the last CTA reduces everything into the result record
//
// The arithmetic per frequency is k_solve_class's (kernels.cu) and the transforms are the
// generic two-pass ones (passes.cuh) — what changes is that the spectra, the adjoints and the
// solve never make an HBM round trip between them: per fit the path moves 8n'(V (2 + 2) + T)
// bytes (n' = n/2 complex slots) instead of the generic path's 8n'(V (6 + 2) + 2T + ...).
// Reference: fast_gram.cpp:42-89 (build_spectrum), :151-263 (invert_and_logdet, equal n),
// gp_core.cpp:92-141 + 197-227 (refresh / loss_value), gradient as in DESIGN.md §4.
#pragma once

#include "kernels.cuh"

namespace fmtgp {

struct LatGeo {
    int m, lt;       // n = 2^m real points, n' = 2^lt = n/2 complex slots
    int l1, l2;      // n' = N1 (rows of L2) * N2 (row length); slot of frequency k1 + N1 k2 = k1 N2 + k2
    int lc;          // log2 columns per L1/L3 CTA (tile 2^(l1 + lc) <= 2^13)
    int nblk_col;    // L1/L3 CTAs per vector
    static bool make(int m, int V, int T, int d, LatGeo& g);
    // the generic-kernel geometry with the same slot layout (yhat, coefficients, seam calls)
    Geo slot_geo() const;
};

// L3 grid cap (one gradient-dot slot per candidate x class and CTA; model.cu sizes part_dot for it)
constexpr int LAT_MAX_INV_GRID = 256;

struct LatArgs {
    int T, P, V, d, nc, m;
    long long half;           // n' slots per vector
    int si_alpha;
    const uint64_t* g;        // [d] generating vector
    const uint64_t* cofs;     // [V][MAXD] class offsets (53-bit, Delta_a - Delta_b)
    const int* pair_ofs;      // [P] pair -> class
    const double* eta;        // [nc][d]
    const double* gamma;      // [nc]
    const double* coef;       // [nc][P]  R_ab
    const double* xi;         // [nc][P]
    const double* Rpair;      // [nc][P]
    const int* pair_a;
    const int* pair_b;
    const double2* yhat;      // [T][n'] slot layout
    const double2* yperm;     // [T][n'] yhat with each row in DIF position order (lat_perm_yhat)
    double2* Y;               // [nc][V][n'] intermediate
    double* part_mid;         // [nc][N1][2 + P]
    double* part_dot;         // [nc][V][max(nblk_col, L3 grid)][MAXD + 1]
    int* bad;                 // [nc]
    unsigned long long* imre; // [nc][MAXT][2]
    unsigned int* counter;    // [0]: L3 last-CTA ticket (self-resetting)
    double* out;              // [nc][NOUT]
    const double2* tw;
    int want_grad;
    int distinct;             // pair_ofs is the all-shifts-distinct map (cls_distinct in lattice.cu)
    int next_pf = 0;          // L2 prefetch of the next wave's rows (bit 0 yhat, bit 1 exchange rows): measured
                              // slower, and the early lines are evicted before use (+1.2 GB DRAM): off
    // ---- frequency sharding over G ranks (G = 1: one GPU).  Rank g owns the
    // column blocks [g ncb, (g+1) ncb) of L1 / L3 (WC = N2 / G columns) and the row clusters
    // [g QP, (g+1) QP) of L2 (R = 2 QP rows: cluster q = rows {q, N1 - q}, or {0, N1/2} for q = 0).
    // (nrank = G, rank = g.)  The intermediate is stored in exchange blocks Y[h][o][i][jl]: h = the rank that owns the row
    // (i its local index 2 (q - h QP) + side) and jl the column local to its column owner, so
    // that "rows of h x my columns" is one contiguous block — the all-to-all's send unit.  L1
    // writes Y, the all-to-all moves the blocks to their row owners, L2 works in place, a second
    // all-to-all returns them to the column owners (Cbuf) for L3.  G = 1: Cbuf == Y.
    int nrank = 1, rank = 0;
    int QP = 0, R = 0, WC = 0, ncb = 0;
    int lwc = 0, lqp = 0;     // log2 WC, log2 QP (world sizes are powers of two): no integer division
    const double2* Cbuf = nullptr;
    // ---- pipelined exchange (K = 2^lkc chunks; K = 1: the layout above).  The forward blocks are
    // stored column-chunked, Y[kc][h][o][i][jl - kc WC/K] (chunk kc = local columns [kc WC/K,
    // (kc+1) WC/K)), the return blocks row-chunked, [kr][h][o][i - kr R/K][jl] (rows [kr R/K,
    // (kr+1) R/K)): chunk k of every rank's buffer is one contiguous all-to-all of G equal blocks.
    // L1 launches per column chunk and L2 per row chunk (`chunk`; -1 = all), so chunk k's exchange
    // runs under chunk k+1's kernel.  L2 writes Yout (the return send buffer; nullptr = in place).
    int lkc = 0, lg = 0;      // log2 K, log2 nrank
    int chunk = -1;
    double2* Yout = nullptr;
};

void lat_fit(const LatGeo& g, const LatArgs& a, cudaStream_t s);
// yperm[t][row][p] = yhat[t][row][ip_freq(p)] (ipfft.cuh): the row order L2's solve walks in
void lat_perm_yhat(const LatGeo& g, int T, long long half, const void* yhat, void* yperm, cudaStream_t s);
// one phase of it (1: L1, 2: L2, 3: L3 when want_grad) — the sharded fit interleaves all-to-alls
void lat_phase(const LatGeo& g, const LatArgs& a, int phase, cudaStream_t s);

}  // namespace fmtgp
