// Kernel declarations shared by kernels.cu (device code) and model.cu (host orchestration).
#pragma once

#include "passes.cuh"

namespace fmtgp {

// ---------------------------------------------------------------- optional per-launch timing
// When a model enables profiling, every kernel launch is bracketed by CUDA events on its
// stream (bench.py's live roofline denominators).  Off by default: zero overhead.
struct Profiler {
    virtual void begin(const char* name, cudaStream_t s) = 0;
    virtual void end(cudaStream_t s) = 0;
    virtual ~Profiler() = default;
};
extern thread_local Profiler* g_prof;
struct ProfScope {
    cudaStream_t s;
    ProfScope(const char* name, cudaStream_t st) : s(st) {
        if (g_prof) g_prof->begin(name, s);
    }
    ~ProfScope() {
        if (g_prof) g_prof->end(s);
    }
};

// ---------------------------------------------------------------- launch helpers
void init_twiddles(double2* tab, cudaStream_t s);

// forward transforms of nvec vectors of log2-length m into slot arrays
// genbuf != nullptr selects the split mode (separate full-parallelism generator kernel)
void fwd_gen(int lattice, const Geo& g, int nvec, const GenSrc& src, const SpecSink& snk, void* work, void* genbuf,
             const double2* tw, cudaStream_t s);
void fwd_array(int lattice, const Geo& g, int nvec, const ArraySrc& src, const ScaleSink& snk, void* work,
               const double2* tw, cudaStream_t s);
void fwd_query(int lattice, const Geo& g, int nvec, const QuerySrc& src, const ScaleSink& snk, void* work,
               const double2* tw, cudaStream_t s);

// inverse transforms of slot arrays (vector v at in + in_off[v]) into a sink
void inv_grad(int lattice, const Geo& g, int nvec, const void* in, const long long* in_off, long long cstride,
              int nvpc, const GradSink& snk, void* work, void* genbuf, const double2* tw, cudaStream_t s);
void inv_coef(int lattice, const Geo& g, int nvec, const void* in, const long long* in_off, const CoefSink& snk,
              void* work, const double2* tw, cudaStream_t s);
int grad_blocks(int lattice, const Geo& g, bool split);

// ---------------------------------------------------------------- equal-n per-frequency solve
struct SolveArgs {
    int T, P, lattice;
    long long nslots;       // slots per vector
    int has_nyq;            // lattice n >= 2: slot 0 also carries the Nyquist frequency
    long long cstride;      // slots per candidate in lam / M
    const void* lam;        // [ncand][P][nslots]
    const void* yhat;       // [T][nslots]   (shared by candidates)
    void* M;                // [ncand][P][nslots]  M = Lam^-1 - chat chat^H  (nullptr: skip)
    void* lam_inv;          // [ncand][P][nslots]  Lam^-1 upper (nullptr: skip)
    void* chat;             // [ncand][T][nslots]  (nullptr: skip)
    double* partial;        // [ncand][nblk][2] (logdet, quad)
    int* bad;               // [ncand] first failing slot (0x7f7f7f7f if none)
    unsigned long long* imre;  // [ncand][MAXT][2] per-stage max |Im Lam_ss|, max pivot (double bits)
    int nblk;
};
void solve_equal(const SolveArgs& a, int ncand, cudaStream_t s);

struct FinalArgs {
    int T, P, d, ncand;
    int nblk_solve, nblk_grad;
    const double* solve_partial;  // [ncand][nblk_solve][2]
    const double* grad_partial;   // [ncand][P][nblk_grad][MAXD+1] (nullptr: no gradient)
    const double* Rpair;          // [ncand][P]
    const double* gamma;          // [ncand]
    const int* pair_a;            // [P]
    const int* pair_b;            // [P]
    double* out;                  // [ncand][NOUT]
};
// per-candidate output record
constexpr int OUT_LOGDET = 0, OUT_QUAD = 1, OUT_NLL = 2, OUT_DGAMMA = 3, OUT_DETA = 4;
constexpr int OUT_DR = OUT_DETA + MAXD;             // [MAXT*MAXT] symmetric dNLL/dR (G with G_ab = G_ba = 1/2 dR_pair)
constexpr int NOUT = OUT_DR + MAXT * MAXT;
void finalize(const FinalArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- per-slot matvec (solve / gram apply)
// out_a = sum_b Op_ab(k) in_b(k) with Op Hermitian given by upper pairs (equal n)
void apply_hermitian(int lattice, int T, long long nslots, const void* op_upper, const void* in, void* out,
                     cudaStream_t s);

}  // namespace fmtgp
