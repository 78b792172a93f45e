// Unequal-n block recursion as a stage-wise LDL^H "fold".
//
// Reference: invert_and_logdet builds the dense r x r grid of Lam^-1 (Algorithm 1,
// /root/reference/proj/src/fast_gram.cpp:151-263), O(N^2/n_L) storage.
// Same pivots (the diagonal Schur complements S of each stage, hence the same logdet),
// factored instead of inverted: stage s eliminates task s (largest first) and updates
//   lam_ab[k] -= sum_c conj(lam_sa[c n_a + k]) lam_sb[c n_a + k] / d_s[c n_a + k],  s < a <= b,
// in place, so storage stays the spectrum's own sum_l (T-l+1) n_l entries.  Solves are
// forward / back substitution through the same strided folds.
//
// Layout ("natural half"): lattice vectors are Hermitian spectra of real columns, stored
// for frequencies k in [0, n/2] (n/2+1 complex); index i > n/2 reads conj(v[n-i]).
// Digital vectors are real, stored in full (n entries).
#pragma once

#include "passes.cuh"

namespace fmtgp {

struct VecMap {          // one vector: slot layout <-> natural layout
    long long soff, noff;  // slot offset, natural offset
    int m, two, l1, l2;
};

struct FoldDims {
    int T, lattice;
    long long n[MAXT];
    long long H[MAXT];      // stored (natural) length of a vector of task length n[t]
    long long poff[MAXP];   // natural offset of pair (a <= b), row by row
    long long toff[MAXT];   // natural offset of task t in a right-hand-side block
    long long tot_pair, tot_task;
    int pid[MAXT][MAXT];
};

__host__ __device__ inline long long fold_H(int lattice, long long n) { return lattice ? (n > 1 ? n / 2 + 1 : 1) : n; }

// slot layout -> natural layout for nvec vectors (maps[v]); vector v of candidate/query block
// `blk` lives at slots + blk * sstride + soff, nat + blk * nstride + noff
void slots_to_nat(int lattice, int nvec, int nblk, const VecMap* maps, const void* slots, long long sstride,
                  void* nat, long long nstride, cudaStream_t s);
void nat_to_slots(int lattice, int nvec, int nblk, const VecMap* maps, const void* nat, long long nstride,
                  void* slots, long long sstride, cudaStream_t s);

// factor in place; per-stage pivot partials: partial[s][blk] (logdet), bad[0] first failing
// natural index (0x7f7f7f7f none), imre[s] = (max |Im Lam_ss|, max pivot) as double bits
void fold_factor(const FoldDims& D, void* lam, double* partial, int nblk, int* bad, unsigned long long* imre,
                 cudaStream_t s);
// nrhs right-hand sides [nrhs][tot_task] in place: forward substitution (+ quad partials
// qpart[r][s][blk]) and optionally back substitution (-> Lam^-1 rhs)
void fold_solve(const FoldDims& D, const void* lam, void* rhs, int nrhs, double* qpart, int nblk, bool back,
                cudaStream_t s);
// part[q][blk]: sum over stages of w Re(conj(z_q) z_{q+nq}) / d of forward-substituted rhs (covariances)
void fold_cross_quad(const FoldDims& D, const void* lam, const void* rhs, int nq, double* part, int nblk,
                     cudaStream_t s);
// trace(Lam^-1) by selected inversion on the factor's own pattern: z (tot_pair entries) receives
// Z = Lam^-1 on that pattern, part[s][blk] the per-stage partial traces
void fold_selinv_trace(const FoldDims& D, const void* lam, void* z, double* part, int nblk, cudaStream_t s);
// z <- z - chat chat^H on the pattern (z from fold_selinv_trace, chat natural [tot_task])
void fold_adjoint(const FoldDims& D, void* z, const void* chat, cudaStream_t s);
// out = Lam v (unfolded spectrum, natural layout), one right-hand side
void fold_gram_apply(const FoldDims& D, const void* lam, const void* v, void* out, cudaStream_t s);

}  // namespace fmtgp
