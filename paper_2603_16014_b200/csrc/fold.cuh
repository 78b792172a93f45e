// Unequal-n block recursion as a stage-wise LDL^H "fold".
//
// Reference: invert_and_logdet builds the dense r x r grid of Lam^-1 (Algorithm 1,
// /root/reference/proj/src/fast_gram.cpp:151-263), O(N^2/n_L) storage.
// Same pivots (the diagonal Schur complements S of each stage, so the same logdet),
// factored instead of inverted: stage s eliminates task s (largest first) and updates
//   lam_ab[k] -= sum_c conj(lam_sa[c n_a + k]) lam_sb[c n_a + k] / d_s[c n_a + k],  s < a <= b,
// in place, so storage stays the spectrum's own sum_l (T-l+1) n_l entries.  Solves are
// forward / back substitution through the same strided folds.
//
// Layout ("natural half"): lattice vectors are Hermitian spectra of real columns, stored
// for frequencies k in [0, n/2] (n/2+1 complex); index i > n/2 reads conj(v[n-i]).
// Digital vectors are real, stored in full (n entries).
#pragma once

#include "common.cuh"

namespace fmtgp {

struct FoldDims {
    int T, P, lattice;
    long long n[MAXT];
    long long H[MAXT];        // stored length per task-length vector
    long long poff[MAXP];     // pair (a<=b) natural offsets
    long long toff[MAXT];     // task natural offsets (right-hand-side layout)
    long long tot_pair, tot_task;
    int pid[MAXT][MAXT];      // pair id of (a<=b)
};

// spectra slot layout (transform output) <-> natural half layout, per vector
void slots_to_nat(int lattice, int m, const Geo_* geo_unused, int nvec, const void* slots, const long long* soff,
                  void* nat, const long long* noff, cudaStream_t s);

}  // namespace fmtgp
