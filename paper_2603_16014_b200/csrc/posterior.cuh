#pragma once

#include "common.cuh"

namespace fmtgp {

struct PostArgs {
    int lattice, d, T, task, si_alpha, mgen, m_cols;
    uint64_t n_max;
    const uint64_t* g;       // device [d]
    const uint64_t* cols;    // device [d * m_cols]
    const uint64_t* shifts;  // device [T * d]
    double b[4];
    const double* eta;       // device [d]
    const double* R;         // device [T * T] internal
    double gamma, tau;
    long long n[MAXT], off[MAXT];
    const double* c;         // device [N] coefficients
    const double* X;         // device [count * d]
    long long count;
    double* out;             // device [count]
    double* part;            // device [nsplit][count] partial sums (workspace)
    int nsplit;              // training-point chunks (grid.y)
    long long chunk;         // global training indices per chunk (multiple of the tile)
};

// grid shape for `count` queries over N training points: >= ~4 CTAs per SM
void posterior_split(long long count, long long N, int& nsplit, long long& chunk);

void posterior_mean(const PostArgs& a, cudaStream_t s);

}  // namespace fmtgp
