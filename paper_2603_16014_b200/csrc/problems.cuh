// Benchmark observations on the device (problems.cu): the reference's multi-fidelity test problems
// at the design points, with the benchmark's observation noise (bench.cpp:84-101).
#pragma once

#include "common.cuh"

namespace fmtgp {

struct ProblemDesign {  // what problem_y needs of a model's design (internal task order)
    int d, T, lattice, mgen, m_cols;
    uint64_t n_max;
    const uint64_t* g;       // device
    const uint64_t* cols;    // device
    const uint64_t* shifts;  // device [T][d]
    long long off[MAXT + 1];
};

// problem index (0 rosenbrock, 1 ackley, 2 borehole, 3 elliptic) and its d / fidelity count; -1 unknown
int problem_index(const char* name, int* d, int* levels);
// y[i] (device, length off[T]) = problem(level user[l] + 1, x_{l,i}) + noise N(0,1) from
// rng::normal(seed, 0x401 + user[l], i)
void problem_y(int problem, const ProblemDesign& pd, const int* user, double noise, uint64_t seed, double* y,
               cudaStream_t s);
// out[i] (device) = problem(level, X[i*d ..]) for X device [count][d] (eval_batch, problems.cpp:145-154)
void problem_eval(int problem, int level, int d, const double* X, uint64_t count, double* out, cudaStream_t s);

}  // namespace fmtgp
