// Kernel declarations shared by kernels.cu (device code) and model.cu (host orchestration).
#pragma once

#include "passes.cuh"

namespace fmtgp {

// compile-time dispatch helpers (threads per CTA, spatial dimension)
#define FM_NT_CASE(V, ...)     \
    case V: {                  \
        constexpr int NT = V;  \
        __VA_ARGS__;           \
    } break;
#define FM_NT_DISPATCH(nt, ...)                                                                      \
    switch (nt) {                                                                                    \
        FM_NT_CASE(32, __VA_ARGS__) FM_NT_CASE(64, __VA_ARGS__) FM_NT_CASE(128, __VA_ARGS__)         \
        FM_NT_CASE(256, __VA_ARGS__) default : {                                                      \
            constexpr int NT = 512;                                                                  \
            __VA_ARGS__;                                                                             \
        }                                                                                            \
        break;                                                                                       \
    }

#define FM_D_DISPATCH(d, ...)                                                                          \
    switch (d) {                                                                                       \
        FM_D_CASE(1, __VA_ARGS__) FM_D_CASE(2, __VA_ARGS__) FM_D_CASE(3, __VA_ARGS__)                  \
        FM_D_CASE(4, __VA_ARGS__) FM_D_CASE(5, __VA_ARGS__) FM_D_CASE(6, __VA_ARGS__)                  \
        FM_D_CASE(7, __VA_ARGS__) FM_D_CASE(8, __VA_ARGS__) FM_D_CASE(9, __VA_ARGS__)                  \
        FM_D_CASE(10, __VA_ARGS__) FM_D_CASE(11, __VA_ARGS__) FM_D_CASE(12, __VA_ARGS__)               \
        FM_D_CASE(13, __VA_ARGS__) FM_D_CASE(14, __VA_ARGS__) FM_D_CASE(15, __VA_ARGS__)               \
        FM_D_CASE(16, __VA_ARGS__) default : break;                                                    \
    }
#define FM_D_CASE(V, ...)    \
    case V: {                \
        constexpr int D = V; \
        __VA_ARGS__;         \
    } break;

constexpr int GEN_NT_DIG = 256;

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
    // class mode (nll path): lam holds the raw spectra of the V offset classes [ncand][V][nslots];
    // lambda_p = coef_p * lam[cls_p] + xi_p is formed in registers, M receives the class adjoints
    // Z_o = sum_{p in o} w_p R_p M_p, partial records are [2 + P] (logdet, quad, sum_k M_p qhat)
    int classes = 0, V = 0;
    const int* pair_cls = nullptr;  // [P]
    const double* coef = nullptr;   // [ncand][P]
    const double* xi = nullptr;     // [ncand][P]
    const double* Rpair = nullptr;  // [ncand][P]
    const int* pair_a = nullptr;
    const int* pair_b = nullptr;
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
    int solve_stride = 2;         // doubles per solve partial record (logdet, quad, ...)
};
// partials may come from other CTAs of the same kernel (last-CTA finalize): L2 loads (__ldcg)
// per-candidate output record
constexpr int OUT_LOGDET = 0, OUT_QUAD = 1, OUT_NLL = 2, OUT_DGAMMA = 3, OUT_DETA = 4;
constexpr int OUT_DR = OUT_DETA + MAXD;             // [MAXT*MAXT] symmetric dNLL/dR (G with G_ab = G_ba = 1/2 dR_pair)
constexpr int NOUT = OUT_DR + MAXT * MAXT;
void finalize(const FinalArgs& a, cudaStream_t s);

template <int NT>
__device__ void finalize_candidate(const FinalArgs& a, int c) {
    double* out = a.out + (size_t)c * NOUT;
    __shared__ double red[32];
    __shared__ double S[MAXP][MAXD + 1];
    const int d = a.d, P = a.P;
    double ld = 0.0, q = 0.0;
    for (int b = threadIdx.x; b < a.nblk_solve; b += NT) {
        ld += __ldcg(a.solve_partial + ((size_t)c * a.nblk_solve + b) * a.solve_stride + 0);
        q += __ldcg(a.solve_partial + ((size_t)c * a.nblk_solve + b) * a.solve_stride + 1);
    }
    ld = block_sum<NT>(ld, red);
    q = block_sum<NT>(q, red);
    if (threadIdx.x == 0) {
        out[OUT_LOGDET] = ld;
        out[OUT_QUAD] = q;
        out[OUT_NLL] = q + ld;  // rT c + logdet (gp_core.cpp:207-211)
    }
    if (!a.grad_partial) return;
    // one warp per (pair, component): fixed-order strided sums + warp tree (deterministic)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = warp; t < P * (MAXD + 1); t += NT / 32) {
        const int p = t / (MAXD + 1), i = t % (MAXD + 1);
        double acc = 0.0;
        if (i < d || i == MAXD)
            for (int b = lane; b < a.nblk_grad; b += 32)
                acc += __ldcg(a.grad_partial + (((size_t)c * P + p) * a.nblk_grad + b) * (MAXD + 1) + i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) S[p][i] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double dgam = 0.0;
        double deta[MAXD];
        for (int j = 0; j < MAXD; ++j) deta[j] = 0.0;
        for (int x = 0; x < MAXT * MAXT; ++x) out[OUT_DR + x] = 0.0;
        for (int p = 0; p < P; ++p) {
            const int pa = a.pair_a[p], pb = a.pair_b[p];
            const double w = pa == pb ? 1.0 : 2.0;
            const double Rp = a.Rpair[(size_t)c * P + p];
            const double dRp = w * S[p][MAXD];  // dNLL / dR_ab, symmetric pair counted once
            for (int j = 0; j < d; ++j) deta[j] += w * Rp * S[p][j];
            dgam += w * Rp * S[p][MAXD];
            if (pa == pb) out[OUT_DR + pa * MAXT + pb] = dRp;
            else {
                out[OUT_DR + pa * MAXT + pb] = 0.5 * dRp;
                out[OUT_DR + pb * MAXT + pa] = 0.5 * dRp;
            }
        }
        (void)dgam;
        out[OUT_DGAMMA] = 0.0;  // formed on the host from the dR record (finish_results)
        for (int j = 0; j < MAXD; ++j) out[OUT_DETA + j] = deta[j];
    }
}


// Gradient bookkeeping when the transforms run per OFFSET CLASS instead of per pair (pairs whose
// generators share the shift difference Delta_a - Delta_b share q, e.g. every diagonal pair):
//   dNLL/dR_p = w_p <W_p, q_o> = w_p sum_k M_p(k) qhat_o(k)        (Parseval, per-frequency partials)
//   dNLL/deta = sum_o <Z_o, dq_o/deta>,  Z_o = H^-1 (sum_{p in o} w_p R_p M_p)   (one inverse per class)
//   dNLL/dgamma = sum_p R_p dNLL/dR_p / gamma                          (q is linear in gamma)
// Class-layout result assembly (per candidate, one CTA).  Inputs: per-block solve partials
// `mid` [nrows][2 + P] (logdet, quad, Parseval dR sums) and per-block class gradient partials
// `dot` [V][nblk][dstride] (component j < d = <Z_o, dq_o/deta_j>).  Every sum is one warp's
// fixed-order strided loop (four independent accumulators) + shuffle tree: deterministic.
// Kept out of line and small: in the digital path it is the last CTA's tail, whose
// instructions come from DRAM after an L2 flush.
struct ClassSums {
    int T, P, V, d, nrows, nblk, dstride;
    const double* mid;
    const double* dot;
    const int* pair_a;
    const int* pair_b;
    const double* Rpair;  // [P] of this candidate
    double gamma;
    double* out;          // [NOUT] of this candidate
};

template <int NT>
__device__ __noinline__ void class_sums_out(const ClassSums& t) {
    // Short code on purpose: in the fused kernels this runs in ONE CTA after every other CTA
    // finished, with cold instruction lines (FMTGP_TRACE: 6.0 us with the previous per-output
    // branch ladder and a device fp64 division).
    __shared__ double res[2 + MAXP + MAXP * MAXD];
    const int S = 2 + t.P, Q = S + t.V * t.d;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // compact loops: the tail's time is instruction fetch (a 4-quantity ILP variant of this loop
    // measured 5.1 us against 4.1 us for this one — more code, more cold lines)
#pragma unroll 1
    for (int q = warp; q < Q; q += NT / 32) {
        const double* base;
        int stride, count;
        if (q < S) {
            base = t.mid + q, stride = S, count = t.nrows;
        } else {
            const int o = (q - S) / t.d, j = (q - S) - o * t.d;
            base = t.dot + size_t(o) * t.nblk * t.dstride + j, stride = t.dstride, count = t.nblk;
        }
        double sum = 0.0;
#pragma unroll 1
        for (int b = lane; b < count; b += 32) sum += base[size_t(b) * stride];
#pragma unroll 1
        for (int o2 = 16; o2 > 0; o2 >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o2);
        if (lane == 0) res[q] = sum;
    }
    __syncthreads();
#pragma unroll 1
    for (int x = threadIdx.x; x < NOUT; x += NT) {  // NT may be below NOUT (small column tiles)
    double v = 0.0;
    if (x < OUT_NLL) {
        v = res[x];
    } else if (x == OUT_NLL) {
        v = res[0] + res[1];  // rT c + logdet (gp_core.cpp:207-211)
    } else if (x == OUT_DGAMMA) {
        // dNLL/dgamma = sum_ab R_ab G_ab / gamma (q is linear in gamma): formed on the host from
        // the dR record (finish_results), like dB = 2 G B and dt = diag G
    } else if (x < OUT_DR) {
        const int j = x - OUT_DETA;
#pragma unroll 1
        for (int o = 0; o < t.V && j < t.d; ++o) v += res[S + o * t.d + j];
    } else {
        // G_ab = G_ba = dNLL/dR_pair (diagonal) or its half-sum convention (2 res) / 2
        int a = (x - OUT_DR) / MAXT, b = (x - OUT_DR) - a * MAXT;
        if (a > b) {
            const int tmp = a;
            a = b;
            b = tmp;
        }
        if (b < t.T) v = res[2 + a * t.T - a * (a - 1) / 2 + (b - a)];
    }
    t.out[x] = v;
    }
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Class-layout finalize as its own kernel (generic equal-n path): one CTA per candidate.
struct ClassFinalArgs {
    int T, P, V, d, nblk_solve, nblk_grad;
    const double* solve_partial;  // [ncand][nblk_solve][2 + P]
    const double* grad_partial;   // [ncand][V][nblk_grad][MAXD + 1] (nullptr: no gradient)
    const double* Rpair;          // [ncand][P]
    const double* gamma;          // [ncand]
    const int* pair_a;
    const int* pair_b;
    double* out;                  // [ncand][NOUT]
};
void finalize_classes(const ClassFinalArgs& a, int ncand, cudaStream_t s);

// ---------------------------------------------------------------- per-slot matvec (solve / gram apply)
// out_a = sum_b Op_ab(k) in_b(k) with Op Hermitian given by upper pairs (equal n)
void apply_hermitian(int lattice, int T, long long nslots, const void* op_upper, const void* in, void* out,
                     cudaStream_t s);

}  // namespace fmtgp
