// Host orchestration + C ABI (include/fastmtgp_b200.h).
//
// The C++ here replaces the reference's fast_gram.cpp / gp_core.cpp control flow for the
// hot path: it owns device memory, plans transforms, launches the kernels of kernels.cu on
// one stream, and maps failures onto the reference's exception semantics
// (SchurBreakdown -> FMTGP_ERR_SCHUR, FastMtgpError -> FMTGP_ERR_INVALID / NONREAL).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fastmtgp_b200.h"
#include "kernels.cuh"
#include "digital.cuh"
#include "lattice.cuh"
#include "fold.cuh"
#include "problems.cuh"
#include "posterior.cuh"
#include "unequal.cuh"

using namespace fmtgp;

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

#define CK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess)                                                                         \
            throw Fail{e_ == cudaErrorMemoryAllocation ? FMTGP_ERR_OOM : FMTGP_ERR_CUDA,              \
                       std::string(#x) + ": " + cudaGetErrorString(e_)};                               \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FMTGP_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FMTGP_ERR_INVALID;
    }
}

constexpr int BAD_NONE = 0x7f7f7f7f;  // cudaMemset(0x7f) sentinel: no failing slot

[[noreturn]] void invalid(const std::string& m) { throw Fail{FMTGP_ERR_INVALID, m}; }

template <class T>
T* dalloc(size_t count) {
    if (count == 0) count = 1;
    void* p = nullptr;
    CK(cudaMalloc(&p, count * sizeof(T)));
    return static_cast<T*>(p);
}

// twiddle table per device (27 levels x 8192 entries)
double2* twiddles_for(int dev) {
    static std::mutex mu;
    static std::vector<double2*> tabs;
    std::lock_guard<std::mutex> lock(mu);
    if (int(tabs.size()) <= dev) tabs.resize(dev + 1, nullptr);
    if (!tabs[dev]) {
        double2* t = dalloc<double2>(size_t(27) << TW_BASE_LOG);
        init_twiddles(t, 0);
        CK(cudaStreamSynchronize(0));
        tabs[dev] = t;
    }
    return tabs[dev];
}

struct Group {            // pairs whose generating (row) task has the same length
    int m;
    Geo geo;
    std::vector<int> pairs;  // global pair ids
    int* d_vec_pair = nullptr;
    long long* d_voff = nullptr;   // slot offset of each pair's vector
    double* d_coef = nullptr;      // [max_cand][npairs]
    double* d_xi = nullptr;
    int coef_off = 0;              // offset into the host staging coef array
};

struct TaskGroup {  // tasks of the same length (yhat / solve / coefficient transforms)
    int m;
    Geo geo;
    std::vector<int> tasks;
    long long* d_yoff = nullptr;   // element offset into y of each task
    long long* d_soff = nullptr;   // slot offset into yhat-like arrays of each task
};

// Per-launch event pairs, aggregated per kernel name (see kernels.cuh Profiler).
struct EventProfiler : Profiler {
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> open, done;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t get() {
        if (pool.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    std::vector<Rec>* capture_list = nullptr;  // set while a graph is being captured
    static bool capturing(cudaStream_t s) {
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &st);
        return st == cudaStreamCaptureStatusActive;
    }
    void begin(const char* name, cudaStream_t s) override {
        Rec r{name, get(), get()};
        if (capturing(s)) cudaEventRecordWithFlags(r.a, s, cudaEventRecordExternal);
        else cudaEventRecord(r.a, s);
        open.push_back(r);
    }
    void end(cudaStream_t s) override {
        Rec r = open.back();
        open.pop_back();
        if (capturing(s)) {
            cudaEventRecordWithFlags(r.b, s, cudaEventRecordExternal);
            if (capture_list) capture_list->push_back(r);  // owned by the graph, re-recorded per replay
        } else {
            cudaEventRecord(r.b, s);
            done.push_back(r);
        }
    }
    void add(const char* name, float ms) {
        auto it = std::find_if(agg.begin(), agg.end(), [&](auto& x) { return x.first == name; });
        if (it == agg.end()) {
            agg.push_back({name, {0.0, 0}});
            it = agg.end() - 1;
        }
        it->second.first += ms;
        it->second.second += 1;
    }
    void add_graph(const std::vector<Rec>& recs) {
        for (const auto& r : recs) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            add(r.name, ms);
        }
    }
    // name -> (total ms, launches)
    std::vector<std::pair<std::string, std::pair<double, int>>> agg;
    void collect() {
        for (auto& r : done) {
            cudaEventSynchronize(r.b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            add(r.name, ms);
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        done.clear();
    }
    void reset() {
        collect();
        agg.clear();
    }
    ~EventProfiler() override {
        for (auto& r : done) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

}  // namespace

struct fmtgp_model {
    EventProfiler prof;
    bool profiling = false;
    int dev = 0;
    cudaStream_t st = nullptr;
    int kind = 0, lattice = 1, d = 0, T = 0, P = 0, max_cand = 1;
    int m[MAXT]{};
    long long n[MAXT]{}, off[MAXT + 1]{}, N = 0;
    bool equal = true;
    std::vector<int> pa, pb;  // pair -> (a, b)
    std::vector<long long> poff, pslots;  // pair slot offset / count
    long long total_slots = 0;            // per candidate
    std::vector<long long> toff_slots;    // task slot offsets (yhat layout)
    long long task_slots = 0;
    std::vector<Group> groups;
    std::vector<TaskGroup> tgroups;
    double2* tw = nullptr;
    // design tables
    uint64_t* d_g = nullptr;
    uint64_t* d_cols = nullptr;
    int m_cols = 0;
    uint64_t* d_offs = nullptr;  // [P][MAXD]
    uint64_t* d_shifts = nullptr;  // [T][d]
    uint64_t n_max = 0;
    int mgen = 0;
    double* d_fit = nullptr;       // last fit: eta [d] | R [T*T]
    bool fit_dirty = true;
    double* d_c = nullptr;         // coefficients of the last fit [N]
    bool have_c = false;
    int *d_pa = nullptr, *d_pb = nullptr;
    std::vector<uint64_t> shifts;  // host [T][d]
    // data
    double* d_y = nullptr;
    void* d_yhat = nullptr;
    void* d_yperm = nullptr;    // fused lattice path: yhat rows in DIF position order
    bool have_y = false;
    double tau[MAXT]{};
    // per-candidate buffers
    double *d_eta = nullptr, *d_gamma = nullptr, *d_Rpair = nullptr;
    void *d_lam = nullptr, *d_M = nullptr, *d_work = nullptr, *d_laminv = nullptr, *d_chat = nullptr;
    size_t work_elems = 0;
    double* d_psolve = nullptr;
    double* d_pgrad = nullptr;
    int* d_bad = nullptr;
    unsigned long long* d_imre = nullptr;  // [max_cand][MAXT][2]
    double* h_imre = nullptr;
    double* d_res = nullptr;   // [out | bad | imre] block
    double* h_res = nullptr;
    size_t res_len = 0;
    double* d_out = nullptr;
    int nblk_solve = 0, nblk_grad = 0;
    // scratch vectors for the seam calls
    double *d_vecA = nullptr, *d_vecB = nullptr;
    void *d_sA = nullptr, *d_sB = nullptr;
    // pinned staging
    double* h_out = nullptr;
    int* h_bad = nullptr;
    // equal n: tau_l = yhat_l(0)/sqrt(n) travels with the next fit's result block (no sync in set_y)
    double* d_tau_raw = nullptr;
    double* h_tau_raw = nullptr;
    bool tau_pending = false;
    cudaEvent_t ev_h2d = nullptr;
    cudaStream_t st_copy = nullptr;     // set_y: per-task H2D copies overlapped with the transforms
    cudaEvent_t ev_set = nullptr, ev_task[MAXT] = {};

    // state of the last spectrum / fit (candidate 0)
    bool have_spec = false, have_inv = false, have_fit = false;
    // fmtgp_nll does not write the fit's spectrum / chat (hot loop); they are re-derived from the
    // remembered hyperparameters (incl. the escalated noise scale) when an API call needs them
    bool fit_lazy = false;
    double* d_scratch = nullptr;  // per-call workspace (posterior queries), grown on demand
    size_t scratch_len = 0;
    bool class_mode = true;  // nll transforms per pair-offset class (FMTGP_CLASSES=0: per pair)
    double fit_xi_scale = 1.0;
    struct StoredHyper {
        fmtgp_hyper h{};
        std::vector<double> eta, B, t, xi;
        void store(const fmtgp_hyper* src, int d, int L) {
            h = *src;
            eta.assign(src->eta, src->eta + d);
            B.assign(src->B, src->B + size_t(L) * src->s);
            t.assign(src->t, src->t + L);
            xi.assign(src->xi, src->xi + L);
            h.eta = eta.data();
            h.B = B.data();
            h.t = t.data();
            h.xi = xi.data();
        }
    } fit_h;
    double last_gamma = 1.0;
    std::vector<double> last_eta, last_R;  // R internal [T*T]
    int last_alpha = 1;
    double last_b[4]{};
    double last_logdet = 0.0;
    unequal::Plan* uneq = nullptr;
    Geo geo_m[28]{};           // transform geometry per log2 length (shared by pairs and tasks)
    bool split = false;        // small problem: separate full-parallelism generator / dot kernels
    void* d_gen = nullptr;     // split-mode generator / W buffer
    // packed per-candidate hyperparameter block (fixed layout, one H2D copy per evaluation)
    double* d_hyp = nullptr;
    double* h_hyp = nullptr;
    size_t hyp_len = 0;
    // CUDA graphs of the equal-n evaluation, keyed on everything baked into kernel params
    struct GraphEntry {
        int nc, grad, keep_chat, si_alpha, prof;
        double b[4];
        int runs = 0;
        cudaGraphExec_t exec = nullptr;
        std::vector<EventProfiler::Rec> recs;
        // fused digital fit with hyperparameters in the kernel parameters: the captured launches
        // and their nodes, re-parameterised before every replay (no H2D copy node)
        cudaGraph_t graph = nullptr;
        std::vector<DigLaunchRec> dig_recs;
        std::vector<cudaGraphNode_t> dig_nodes;
    };
    std::vector<GraphEntry> graphs;
    bool use_graphs = true;
    long long spec_version = 0;  // bumped whenever d_lam is rewritten
    // fused three-kernel digital path (digital.cuh)
    bool dig = false;
    DigGeo dgeo{};
    double* d_part_mid = nullptr;
    double* d_part_dot = nullptr;
    unsigned int* d_counter = nullptr;
    double* d_vec_sum = nullptr;
    int* d_pair_ofs = nullptr;
    std::vector<int> h_pair_ofs;
    int* d_iota = nullptr;           // [P] 0..P-1 (class vector -> class offset row)
    long long* d_cvoff = nullptr;    // [P] slot offset of class vector o (o * pslots)
    double* d_ones = nullptr;        // [max_cand * P]
    double* d_zeros = nullptr;       // [max_cand * P]
    uint64_t* d_ofs = nullptr;  // distinct pair offsets [nofs][MAXD]
    int nofs = 0;
    double* d_kap = nullptr;    // design-time kappa table [nofs][d][n]
    // fused three-kernel lattice path (lattice.cuh); shares part_mid / part_dot / counter
    bool lat = false;
    LatGeo lgeo{};
    int dig_tail = 1;
    bool zero_copy = true;  // FMTGP_ZERO_COPY=0: D2H copy node instead of the mapped record
    bool zero_copy_hyper = false;  // FMTGP_ZERO_COPY_HYPER=1: kernels read the pinned hyper block
    bool hv_params = true;         // FMTGP_HV_PARAMS=0: H2D copy node instead of kernel-parameter values
    volatile unsigned long long* h_done = nullptr;  // completion word (pinned, mapped), see DigArgs
    unsigned long long done_seq = 0;
    // frequency sharding of the fused lattice fit (fmtgp_shard_*): world size / rank
    int sh_G = 1, sh_g = 0;
    int sh_lkc = 0;  // log2 exchange chunks (fmtgp_shard_chunks)
    LatArgs sh_args{};
    fmtgp_hyper sh_h{};
    bool sh_grad = false;
    unsigned long long* d_trace = nullptr;  // FMTGP_TRACE=1: digital-fit phase timestamps to stderr  // digital K3 finalize mode (DigArgs::tail), FMTGP_DIG_TAIL
    double kap_b[4]{};
    bool kap_valid = false;
    bool kap_enabled = true;
};

namespace {

int pair_index(int T, int a, int b) { return a * T - a * (a - 1) / 2 + (b - a); }

Spatial spatial_of(const fmtgp_model* M, int si_alpha, const double* b) {
    Spatial sp{};
    sp.family = M->lattice ? 0 : 1;
    sp.d = M->d;
    sp.si_alpha = si_alpha;
    for (int i = 0; i < 4; ++i) sp.b[i] = b[i];
    return sp;
}

PointGen pointgen_of(const fmtgp_model* M, int m) {
    PointGen pg{};
    pg.family = M->lattice ? 0 : 1;
    pg.m = m;
    pg.g = M->d_g;
    pg.cols = M->d_cols;
    pg.m_cols = M->m_cols;
    return pg;
}

void validate_hyper(const fmtgp_model* M, const fmtgp_hyper* h) {
    if (!h) invalid("null hyperparameters");
    if (!h->eta || !h->t || !h->xi) invalid("hyperparameters: null eta / t / xi");
    if (h->s < 0 || (h->s > 0 && !h->B)) invalid("hyperparameters: bad task factor B");
    for (int l = 0; l < M->T; ++l)
        if (!(h->t[l] > 0.0)) invalid("task_gram: non-positive diagonal entry");
    if (M->lattice && h->si_alpha != 1 && h->si_alpha != 2) invalid("si_bernoulli_1d: alpha must be 1 or 2");
}

// R = B B^T + diag(t) (kernels.cpp:124-135), internal order
std::vector<double> task_gram(const fmtgp_model* M, const fmtgp_hyper* h) {
    std::vector<double> R(size_t(M->T) * M->T, 0.0);
    for (int a = 0; a < M->T; ++a)
        for (int b = 0; b < M->T; ++b) {
            double s = 0.0;
            for (int k = 0; k < h->s; ++k) s += h->B[a * h->s + k] * h->B[b * h->s + k];
            R[a * M->T + b] = s + (a == b ? h->t[a] : 0.0);
        }
    return R;
}


// Fill the pinned hyperparameter block (eta, gamma, Rpair, per-group coef and xi) for nc
// candidates; xi_scale[c] is the escalation factor of candidate c.  Host-only: the H2D copy
// is issued by copy_hyper (inside the captured graph).
void fill_hyper(fmtgp_model* M, int nc, const fmtgp_hyper* const* hs, const double* xi_scale) {
    const int d = M->d, P = M->P, mc = M->max_cand;
    double* eta = M->h_hyp;
    double* gam = eta + size_t(mc) * d;
    double* Rp = gam + mc;
    for (int c = 0; c < nc; ++c) {
        const fmtgp_hyper* h = hs[c];
        for (int j = 0; j < d; ++j) eta[c * d + j] = h->eta[j];
        gam[c] = h->gamma;
        const std::vector<double> R = task_gram(M, h);
        for (int p = 0; p < P; ++p) Rp[c * P + p] = R[M->pa[p] * M->T + M->pb[p]];
    }
    double* cur = Rp + size_t(mc) * P;
    for (auto& g : M->groups) {
        const int np = int(g.pairs.size());
        double* co = cur;
        double* xi = cur + size_t(mc) * np;
        for (int c = 0; c < nc; ++c) {
            const fmtgp_hyper* h = hs[c];
            for (int q = 0; q < np; ++q) {
                const int p = g.pairs[q], a = M->pa[p], b = M->pb[p];
                // sqrt(n_b) * V̄_{m_a} = sqrt(n_b / n_a) * unnormalised transform (fast_gram.cpp:82-83)
                const double scale = std::sqrt(double(M->n[b]) / double(M->n[a]));
                co[c * np + q] = Rp[c * P + p] * scale;
                double x = 0.0;
                if (a == b) {
                    x = h->xi[a] * xi_scale[c];
                    if (xi_scale[c] > 1.0 && h->xi[a] == 0.0) x = 1e-12 * xi_scale[c];  // gp_core.cpp:103-105
                }
                xi[c * np + q] = x;
            }
        }
        cur += 2 * size_t(mc) * np;
    }
}

void copy_hyper(fmtgp_model* M) {
    CK(cudaMemcpyAsync(M->d_hyp, M->h_hyp, M->hyp_len * sizeof(double), cudaMemcpyHostToDevice, M->st));
}

void upload_hyper(fmtgp_model* M, int nc, const fmtgp_hyper* const* hs, const double* xi_scale) {
    fill_hyper(M, nc, hs, xi_scale);
    copy_hyper(M);
}

GenSrc gensrc_of(fmtgp_model* M, const Group& g, int si_alpha, const double* b) {
    GenSrc s{};
    s.sp = spatial_of(M, si_alpha, b);
    s.pg = pointgen_of(M, g.m);
    s.offs = M->d_offs;
    s.eta = M->d_eta;
    s.gamma = M->d_gamma;
    s.vec_pair = g.d_vec_pair;
    s.nvpc = int(g.pairs.size());
    return s;
}

// build_spectrum for nc candidates (fast_gram.cpp:42-89)
void build_spectra(fmtgp_model* M, int nc, int si_alpha, const double* b) {
    ++M->spec_version;
    for (auto& g : M->groups) {
        const int np = int(g.pairs.size());
        GenSrc src = gensrc_of(M, g, si_alpha, b);
        SpecSink snk{};
        snk.out = M->d_lam;
        snk.voff = g.d_voff;
        snk.cstride = M->total_slots;
        snk.coef = g.d_coef;
        snk.xi = g.d_xi;
        snk.nvpc = np;
        fwd_gen(M->lattice, g.geo, np * nc, src, snk, M->d_work, M->split ? M->d_gen : nullptr, M->tw, M->st);
    }
    CK(cudaGetLastError());
}

// raw spectra of the V pair-offset classes (equal n, nll path): lambda_p is formed in the solve
void build_class_spectra(fmtgp_model* M, int nc, int si_alpha, const double* b) {
    ++M->spec_version;
    const Group& g = M->groups[0];
    GenSrc src = gensrc_of(M, g, si_alpha, b);
    src.offs = M->d_ofs;
    src.vec_pair = M->d_iota;
    src.nvpc = M->nofs;
    SpecSink snk{};
    snk.out = M->d_lam;
    snk.voff = M->d_cvoff;
    snk.cstride = M->total_slots;
    snk.coef = M->d_ones;
    snk.xi = M->d_zeros;
    snk.nvpc = M->nofs;
    fwd_gen(M->lattice, g.geo, M->nofs * nc, src, snk, M->d_work, M->split ? M->d_gen : nullptr, M->tw, M->st);
    CK(cudaGetLastError());
}

size_t elem_size(const fmtgp_model* M) { return M->lattice ? sizeof(double2) : sizeof(double); }

// forward transform of a length-N vector (device) into task-slot layout
void forward_vector(fmtgp_model* M, const double* dvec, void* dslots) {
    for (auto& tg : M->tgroups) {
        ArraySrc src{dvec, tg.d_yoff, tg.m, M->lattice};
        ScaleSink snk{dslots, tg.d_soff, 1.0 / std::sqrt(double(1ll << tg.m))};
        fwd_array(M->lattice, tg.geo, int(tg.tasks.size()), src, snk, M->d_work, M->tw, M->st);
    }
    CK(cudaGetLastError());
}

// inverse transform from task-slot layout into a length-N vector (device)
void inverse_vector(fmtgp_model* M, const void* dslots, double* dvec) {
    for (auto& tg : M->tgroups) {
        CoefSink cs{dvec, tg.d_yoff, tg.m, 1.0 / std::sqrt(double(1ll << tg.m))};
        inv_coef(M->lattice, tg.geo, int(tg.tasks.size()), dslots, tg.d_soff, cs, M->d_work, M->tw, M->st);
    }
    CK(cudaGetLastError());
}

void compute_tau(fmtgp_model* M);

void compute_yhat_tau(fmtgp_model* M) {
    forward_vector(M, M->d_y, M->d_yhat);
    if (M->lat) lat_perm_yhat(M->lgeo, M->T, M->pslots[0], M->d_yhat, M->d_yperm, M->st);
    compute_tau(M);
}

// set_y from host memory with the upload pipelined against the transform: task t's copy runs on
// the copy stream, its transform (and the fused path's yhat permutation) on the model stream as
// soon as that copy has landed, so the next task's H2D overlaps the previous task's transform
void upload_yhat_tau(fmtgp_model* M, const double* y) {
    CK(cudaEventRecord(M->ev_set, M->st));
    CK(cudaStreamWaitEvent(M->st_copy, M->ev_set, 0));
    for (int t = 0; t < M->T; ++t) {
        CK(cudaMemcpyAsync(M->d_y + M->off[t], y + M->off[t], sizeof(double) * M->n[t], cudaMemcpyHostToDevice,
                           M->st_copy));
        CK(cudaEventRecord(M->ev_task[t], M->st_copy));
    }
    CK(cudaEventRecord(M->ev_h2d, M->st_copy));
    const size_t es = elem_size(M);
    for (auto& tg : M->tgroups)
        for (size_t i = 0; i < tg.tasks.size(); ++i) {
            const int t = tg.tasks[i];
            CK(cudaStreamWaitEvent(M->st, M->ev_task[t], 0));
            ArraySrc src{M->d_y, tg.d_yoff + i, tg.m, M->lattice};
            ScaleSink snk{M->d_yhat, tg.d_soff + i, 1.0 / std::sqrt(double(1ll << tg.m))};
            fwd_array(M->lattice, tg.geo, 1, src, snk, M->d_work, M->tw, M->st);
            if (M->lat)
                lat_perm_yhat(M->lgeo, 1, M->pslots[0], static_cast<char*>(M->d_yhat) + M->toff_slots[t] * es,
                              static_cast<char*>(M->d_yperm) + M->toff_slots[t] * es, M->st);
        }
    CK(cudaGetLastError());
    compute_tau(M);
}

void compute_tau(fmtgp_model* M) {
    // tau: equal n -> tau_l = yhat_l(0) / sqrt(n) (the sample mean, gp_core.cpp:67-88 with
    // V̄ 1 = sqrt(n) e_0); unequal n -> class-0 normal equations at fit time.
    if (M->equal) {
        // yhat_l(0) (first double of each task block, uniform stride) -> tail of the result block,
        // read back with the next fit's single D2H copy: no host round trip here
        const size_t es = elem_size(M), pitch = size_t(M->T > 1 ? M->toff_slots[1] : 0) * es;
        CK(cudaMemcpy2DAsync(M->d_tau_raw, sizeof(double), M->d_yhat, pitch ? pitch : sizeof(double), sizeof(double),
                             M->T, cudaMemcpyDeviceToDevice, M->st));
        M->tau_pending = true;
    } else {
        std::vector<double> y0(M->T);
        for (int t = 0; t < M->T; ++t) {
            CK(cudaMemcpyAsync(&y0[t], static_cast<char*>(M->d_yhat) + M->toff_slots[t] * elem_size(M),
                               sizeof(double), cudaMemcpyDeviceToHost, M->st));
        }
        CK(cudaStreamSynchronize(M->st));
        for (int t = 0; t < M->T; ++t) M->tau[t] = y0[t] / std::sqrt(double(M->n[t]));
    }
    M->have_y = true;
}

// model-owned device workspace (no cudaMalloc / cudaFree — which synchronises — per call)
double* scratch(fmtgp_model* M, size_t words) {
    if (words > M->scratch_len) {
        CK(cudaStreamSynchronize(M->st));
        if (M->d_scratch) cudaFree(M->d_scratch);
        M->d_scratch = nullptr;
        M->scratch_len = 0;
        const size_t len = std::max(words, M->scratch_len * 2);
        M->d_scratch = dalloc<double>(len);
        M->scratch_len = len;
    }
    return M->d_scratch;
}

void take_tau(fmtgp_model* M) {  // after a D2H of the result block
    if (!M->tau_pending) return;
    for (int t = 0; t < M->T; ++t) M->tau[t] = M->h_tau_raw[t] / std::sqrt(double(M->n[t]));
    M->tau_pending = false;
}

void finish_results(fmtgp_model* M, int nc, const fmtgp_hyper* const* hs, bool grad, fmtgp_result* out,
                    const double* xi_scale, const int* esc) {
    const int T = M->T;
    take_tau(M);
    for (int c = 0; c < nc; ++c) {
        const double* o = M->h_out + size_t(c) * NOUT;
        fmtgp_result& r = out[c];
        std::memset(&r, 0, sizeof(r));
        r.logdet = o[OUT_LOGDET];
        r.quad = o[OUT_QUAD];
        r.nll = o[OUT_NLL];
        r.xi_scale = xi_scale[c];
        r.escalations = esc[c];
        for (int t = 0; t < T; ++t) r.tau[t] = M->tau[t];
        if (grad) {
            r.dgamma = 0.0;  // q is linear in gamma: dNLL/dgamma = sum_ab R_ab G_ab / gamma
            for (int j = 0; j < M->d; ++j) r.deta[j] = o[OUT_DETA + j];
            const fmtgp_hyper* h = hs[c];
            for (int a = 0; a < T; ++a)
                for (int b = 0; b < T; ++b) r.dR[a * T + b] = o[OUT_DR + a * MAXT + b];
            const std::vector<double> R = task_gram(M, h);
            for (int x = 0; x < T * T; ++x) r.dgamma += R[x] * r.dR[x];
            r.dgamma /= h->gamma;
            for (int a = 0; a < T; ++a) {
                r.dt[a] = r.dR[a * T + a];
                for (int k = 0; k < h->s; ++k) {
                    double acc = 0.0;
                    for (int b = 0; b < T; ++b) acc += r.dR[a * T + b] * h->B[b * h->s + k];
                    r.dB[a * h->s + k] = 2.0 * acc;  // dNLL/dB = 2 G B
                }
            }
        }
    }
}

// Fused digital fit (digital.cuh): three kernels, spectra never leave L2 between them.
// host alias of a pointer into the device hyperparameter block (pinned = mapped under UVA)
const double* hyper_host(const fmtgp_model* M, const double* dptr) { return M->h_hyp + (dptr - M->d_hyp); }

// one-candidate fused digital fits carry the hyperparameters in the kernel parameters
bool dig_use_hv(const fmtgp_model* M, int nc, bool keep_chat) {
    return M->dig && M->hv_params && nc == 1 && !keep_chat && !M->zero_copy_hyper;
}

// candidate 0's values from the filled host block (fill_hyper)
void fill_hv(const fmtgp_model* M, DigHyperVals& hv) {
    const Group& g = M->groups[0];
    for (int j = 0; j < M->d; ++j) hv.eta[j] = hyper_host(M, M->d_eta)[j];
    hv.gamma = hyper_host(M, M->d_gamma)[0];
    for (int p = 0; p < M->P; ++p) {
        hv.coef[p] = hyper_host(M, g.d_coef)[p];
        hv.xi[p] = hyper_host(M, g.d_xi)[p];
        hv.Rpair[p] = hyper_host(M, M->d_Rpair)[p];
    }
}

void eval_digital_body(fmtgp_model* M, int nc, int si_alpha, const double* bw, bool grad, bool keep_chat) {
    // zero-copy hyperparameters: with one candidate the kernels read the pinned host block
    // directly (a few dozen doubles, loaded in prologues that overlap the previous kernel) and the
    // graph has no H2D copy node; failure flags are zeroed by the first kernel
    const bool zch = M->zero_copy_hyper && nc == 1 && !keep_chat;
    const bool hv = dig_use_hv(M, nc, keep_chat);
    if (!zch && !hv) copy_hyper(M);
    const Group& g = M->groups[0];
    DigArgs a{};
    a.T = M->T;
    a.P = M->P;
    a.d = M->d;
    a.nc = nc;
    a.n = M->n[0];
    a.sp = spatial_of(M, si_alpha, bw);
    a.pg = pointgen_of(M, M->m[0]);
    a.V = M->nofs;
    a.cofs = M->d_ofs;
    a.kap = M->kap_valid ? M->d_kap : nullptr;
    a.pair_ofs = M->d_pair_ofs;
    a.eta = M->d_eta;
    a.gamma = M->d_gamma;
    a.coef = g.d_coef;
    a.xi = g.d_xi;
    a.Rpair = M->d_Rpair;
    a.pair_a = M->d_pa;
    a.pair_b = M->d_pb;
    a.yhat = static_cast<const double*>(M->d_yhat);
    a.Y = static_cast<double*>(M->d_work);
    a.lam_out = keep_chat ? static_cast<double*>(M->d_lam) : nullptr;
    a.chat_out = keep_chat ? static_cast<double*>(M->d_chat) : nullptr;
    a.part_mid = M->d_part_mid;
    a.part_dot = M->d_part_dot;
    a.bad = M->d_bad;
    a.imre = M->d_imre;
    a.counter = M->d_counter;
    a.vec_sum = M->d_vec_sum;
    a.out = M->d_out;
    a.want_grad = grad;
    if (hv) {
        a.use_hv = 1;
        fill_hv(M, a.hv);
    }
    if (zch) {
        a.eta = hyper_host(M, M->d_eta);
        a.gamma = hyper_host(M, M->d_gamma);
        a.coef = hyper_host(M, g.d_coef);
        a.xi = hyper_host(M, g.d_xi);
        a.Rpair = hyper_host(M, M->d_Rpair);
    }
    a.tail = M->dig_tail;
    // candidate batches: one kappa tile per CTA serves a group of candidates (config 5 reads the
    // design-time table once per group instead of once per candidate); groups keep >= 2 CTAs per SM
    if (nc > 1 && a.kap) {
        const long long ctas = (long long)M->dgeo.nblk_col * a.V;
        int groups = int(std::max<long long>(1, (2 * 148 + ctas - 1) / ctas));
        groups = std::min(groups, nc);
        a.cpb = (nc + groups - 1) / groups;
        if (const char* e = std::getenv("FMTGP_DIG_CPB")) a.cpb = std::max(1, std::min(nc, std::atoi(e)));
    }
    if (a.cpb > 1) a.tail = 2;  // per-candidate finalize kernel (the last-CTA tail is per CTA)
    const bool zc = grad && a.tail == 1 && nc == 1 && M->zero_copy && !keep_chat;
    if (zc) {
        if (hv) a.done_flag = M->h_done;  // the host spins on it (eval_equal)
        a.zc_res = M->h_res;  // pinned = mapped (UVA): the same pointer on the device
        a.res_dev = M->d_res;
        a.res_flags_off = int(size_t(M->max_cand) * NOUT);
        a.res_len = int(M->res_len);
    }
    if (M->d_trace) {
        std::vector<unsigned long long> init(16, 0);
        for (int i : {0, 2, 3, 5, 6, 11, 12, 13}) init[i] = ~0ull;
        CK(cudaMemcpyAsync(M->d_trace, init.data(), 16 * sizeof(unsigned long long), cudaMemcpyHostToDevice, M->st));
        CK(cudaStreamSynchronize(M->st));
        a.trace = M->d_trace;
    }
    dig_fit(M->dgeo, a, M->st);
    CK(cudaGetLastError());
    if (zc) return;  // the record is already in the host block
    if (!grad) {
        FinalArgs fa{};
        fa.T = M->T;
        fa.P = M->P;
        fa.d = M->d;
        fa.ncand = nc;
        fa.nblk_solve = 1 << M->dgeo.l1;
        fa.solve_partial = M->d_part_mid;
        fa.solve_stride = 2 + M->P;
        fa.Rpair = M->d_Rpair;
        fa.gamma = M->d_gamma;
        fa.pair_a = M->d_pa;
        fa.pair_b = M->d_pb;
        fa.out = M->d_out;
        finalize(fa, M->st);
    }
    CK(cudaMemcpyAsync(M->h_res, M->d_res, sizeof(double) * M->res_len, cudaMemcpyDeviceToHost, M->st));
}

// Fused lattice fit (lattice.cuh): three kernels, spectra and adjoints never leave the SMs /
// L2 between the row FFT, the solve and the inverse row FFT.
LatArgs lat_args(fmtgp_model* M, int nc, int si_alpha, bool grad) {
    const Group& g = M->groups[0];
    LatArgs a{};
    a.T = M->T;
    a.P = M->P;
    a.V = M->nofs;
    a.d = M->d;
    a.nc = nc;
    a.m = M->m[0];
    a.half = M->pslots[0];
    a.si_alpha = si_alpha;
    a.g = M->d_g;
    a.cofs = M->d_ofs;
    a.pair_ofs = M->d_pair_ofs;
    a.eta = M->d_eta;
    a.gamma = M->d_gamma;
    a.coef = g.d_coef;
    a.xi = g.d_xi;
    a.Rpair = M->d_Rpair;
    a.pair_a = M->d_pa;
    a.pair_b = M->d_pb;
    a.yhat = static_cast<const double2*>(M->d_yhat);
    a.yperm = static_cast<const double2*>(M->d_yperm);
    a.Y = static_cast<double2*>(M->d_work);
    a.part_mid = M->d_part_mid;
    a.part_dot = M->d_part_dot;
    a.bad = M->d_bad;
    a.imre = M->d_imre;
    a.counter = M->d_counter;
    a.out = M->d_out;
    a.tw = M->tw;
    a.want_grad = grad;
    a.distinct = M->nofs == M->P - M->T + 1;
    for (int p = 0, off = 0; p < M->P && a.distinct; ++p) {
        const int want = M->pa[p] == M->pb[p] ? 0 : 1 + off++;
        if (M->h_pair_ofs[p] != want) a.distinct = 0;
    }
    const LatGeo& lg = M->lgeo;
    a.nrank = M->sh_G;
    a.rank = M->sh_g;
    a.QP = (1 << lg.l1) / 2 / a.nrank;
    a.R = 2 * a.QP;
    a.WC = (1 << lg.l2) / a.nrank;
    while ((1 << a.lwc) < a.WC) ++a.lwc;
    while ((1 << a.lqp) < a.QP) ++a.lqp;
    a.ncb = lg.nblk_col / a.nrank;
    while ((1 << a.lg) < a.nrank) ++a.lg;
    a.lkc = M->sh_lkc;
    a.Cbuf = a.Y;
    if (const char* e = std::getenv("FMTGP_LAT_PF")) a.next_pf = std::atoi(e) & 3;
    return a;
}

void lat_finalize_nograd(fmtgp_model* M, int nc) {
    FinalArgs fa{};
    fa.T = M->T;
    fa.P = M->P;
    fa.d = M->d;
    fa.ncand = nc;
    fa.nblk_solve = (1 << M->lgeo.l1) / M->sh_G;
    fa.solve_partial = M->d_part_mid;
    fa.solve_stride = 2 + M->P;
    fa.Rpair = M->d_Rpair;
    fa.gamma = M->d_gamma;
    fa.pair_a = M->d_pa;
    fa.pair_b = M->d_pb;
    fa.out = M->d_out;
    finalize(fa, M->st);
}

void eval_lattice_body(fmtgp_model* M, int nc, int si_alpha, bool grad) {
    copy_hyper(M);  // failure flags are zeroed by the first kernel
    const LatArgs a = lat_args(M, nc, si_alpha, grad);
    lat_fit(M->lgeo, a, M->st);
    CK(cudaGetLastError());
    if (!grad) lat_finalize_nograd(M, nc);
    CK(cudaMemcpyAsync(M->h_res, M->d_res, sizeof(double) * M->res_len, cudaMemcpyDeviceToHost, M->st));
}

// The design-time kappa table depends on the design and the Walsh order weights only
// (not on gamma, eta, R, xi): rebuilt when b changes, outside any captured graph.
void ensure_kappa_table(fmtgp_model* M, int si_alpha, const double* bw) {
    if (!M->dig || !M->d_kap || !M->kap_enabled) {
        M->kap_valid = false;
        return;
    }
    if (M->kap_valid && std::memcmp(M->kap_b, bw, sizeof(M->kap_b)) == 0) return;
    dig_kappa_table(spatial_of(M, si_alpha, bw), pointgen_of(M, M->m[0]), M->d_ofs, M->nofs, M->n[0], M->d_kap,
                    M->st);
    CK(cudaGetLastError());
    std::memcpy(M->kap_b, bw, sizeof(M->kap_b));
    M->kap_valid = true;
}

// Stream-ordered body of one equal-n evaluation (captured into a CUDA graph).
void eval_equal_body(fmtgp_model* M, int nc, int si_alpha, const double* bw, bool grad, bool keep_chat) {
    if (M->dig) {
        eval_digital_body(M, nc, si_alpha, bw, grad, keep_chat);
        return;
    }
    if (M->lat && M->sh_G == 1 && !keep_chat) {  // a sharded model's plain nll takes the generic path
        eval_lattice_body(M, nc, si_alpha, grad);
        return;
    }
    copy_hyper(M);
    const bool classes = !keep_chat && M->class_mode;
    if (classes) build_class_spectra(M, nc, si_alpha, bw);
    else build_spectra(M, nc, si_alpha, bw);
    CK(cudaMemsetAsync(M->d_bad, 0x7f, sizeof(int) * nc, M->st));
    CK(cudaMemsetAsync(M->d_bad + nc, 0, sizeof(int) * nc, M->st));
    CK(cudaMemsetAsync(M->d_imre, 0, sizeof(unsigned long long) * 2 * MAXT * nc, M->st));
    SolveArgs sa{};
    sa.T = M->T;
    sa.P = M->P;
    sa.lattice = M->lattice;
    sa.nslots = M->pslots[0];
    sa.has_nyq = M->n[0] >= 2;
    sa.cstride = M->total_slots;
    sa.lam = M->d_lam;
    sa.yhat = M->d_yhat;
    sa.M = grad ? M->d_M : nullptr;
    sa.lam_inv = nullptr;
    sa.chat = keep_chat ? M->d_chat : nullptr;
    sa.partial = M->d_psolve;
    sa.bad = M->d_bad;
    sa.imre = M->d_imre;
    sa.nblk = M->nblk_solve;
    const Group& g = M->groups[0];
    if (classes) {
        sa.classes = 1;
        sa.V = M->nofs;
        sa.pair_cls = M->d_pair_ofs;
        sa.coef = g.d_coef;
        sa.xi = g.d_xi;
        sa.Rpair = M->d_Rpair;
        sa.pair_a = M->d_pa;
        sa.pair_b = M->d_pb;
        solve_equal(sa, nc, M->st);
        CK(cudaGetLastError());
        if (grad) {
            GradSink gs{};
            gs.gen = gensrc_of(M, g, si_alpha, bw);
            gs.gen.offs = M->d_ofs;
            gs.gen.vec_pair = M->d_iota;
            gs.gen.nvpc = M->nofs;
            gs.partial = M->d_pgrad;
            gs.nblk = M->nblk_grad;
            gs.acc_n = M->d + 1;
            inv_grad(M->lattice, g.geo, M->nofs * nc, M->d_M, M->d_cvoff, M->total_slots, M->nofs, gs, M->d_work,
                     M->split ? M->d_gen : nullptr, M->tw, M->st);
            CK(cudaGetLastError());
        }
        ClassFinalArgs fa{};
        fa.T = M->T;
        fa.P = M->P;
        fa.V = M->nofs;
        fa.d = M->d;
        fa.nblk_solve = M->nblk_solve;
        fa.nblk_grad = M->nblk_grad;
        fa.solve_partial = M->d_psolve;
        fa.grad_partial = grad ? M->d_pgrad : nullptr;
        fa.Rpair = M->d_Rpair;
        fa.gamma = M->d_gamma;
        fa.pair_a = M->d_pa;
        fa.pair_b = M->d_pb;
        fa.out = M->d_out;
        finalize_classes(fa, nc, M->st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(M->h_res, M->d_res, sizeof(double) * M->res_len, cudaMemcpyDeviceToHost, M->st));
        return;
    }
    solve_equal(sa, nc, M->st);
    CK(cudaGetLastError());
    if (grad) {
        GradSink gs{};
        gs.gen = gensrc_of(M, g, si_alpha, bw);
        gs.partial = M->d_pgrad;
        gs.nblk = M->nblk_grad;
        gs.acc_n = M->d + 1;
        inv_grad(M->lattice, g.geo, M->P * nc, M->d_M, g.d_voff, M->total_slots, M->P, gs, M->d_work,
                 M->split ? M->d_gen : nullptr, M->tw, M->st);
        CK(cudaGetLastError());
    }
    FinalArgs fa{};
    fa.T = M->T;
    fa.P = M->P;
    fa.d = M->d;
    fa.ncand = nc;
    fa.nblk_solve = M->nblk_solve;
    fa.nblk_grad = M->nblk_grad;
    fa.solve_partial = M->d_psolve;
    fa.grad_partial = grad ? M->d_pgrad : nullptr;
    fa.Rpair = M->d_Rpair;
    fa.gamma = M->d_gamma;
    fa.pair_a = M->d_pa;
    fa.pair_b = M->d_pb;
    fa.out = M->d_out;
    finalize(fa, M->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(M->h_res, M->d_res, sizeof(double) * M->res_len, cudaMemcpyDeviceToHost, M->st));
}

// non-real Schur complement test of candidate c (fast_gram.cpp:167-172), stage-global like the reference
bool nonreal_of(const fmtgp_model* M, int c) {
    for (int t = 0; t < M->T; ++t) {
        const double im = M->h_imre[(size_t(c) * MAXT + t) * 2], re = M->h_imre[(size_t(c) * MAXT + t) * 2 + 1];
        if (im > 1e-8 * std::max(1.0, re)) return true;
    }
    return false;
}

// One batched evaluation attempt (equal n).  Results land in M->h_out / M->h_bad.  The first
// run of a configuration executes eagerly; later runs replay a captured CUDA graph (one
// launch per fit instead of ~10 kernel launches + copies).
void eval_equal(fmtgp_model* M, int nc, const fmtgp_hyper* const* hs, const double* xi_scale, bool grad,
                bool keep_chat) {
    const fmtgp_hyper* h0 = hs[0];
    fill_hyper(M, nc, hs, xi_scale);
    ensure_kappa_table(M, h0->si_alpha, h0->b);
    const int prof = M->profiling ? 1 : 0;
    fmtgp_model::GraphEntry* ge = nullptr;
    for (auto& e : M->graphs)
        if (e.nc == nc && e.grad == int(grad) && e.keep_chat == int(keep_chat) && e.si_alpha == h0->si_alpha &&
            e.prof == prof && std::memcmp(e.b, h0->b, sizeof(e.b)) == 0)
            ge = &e;
    if (M->d_trace) {  // diagnostics: always eager, print the phase marks
        eval_equal_body(M, nc, h0->si_alpha, h0->b, grad, keep_chat);
        CK(cudaStreamSynchronize(M->st));
        unsigned long long t[16];
        CK(cudaMemcpy(t, M->d_trace, sizeof(t), cudaMemcpyDeviceToHost));
        const char* nm[14] = {"K1 first entry", "K1 last exit", "K2 first entry", "K2 first past wait", "K2 last exit",
                              "K3 first entry", "K3 first past wait", "K3 last exit (pre-ticket)", "tail: ticket",
                              "tail: staged", "tail: done", "K1 first exit", "K2 first exit", "K3 first exit"};
        for (int i = 0; i < 14; ++i)
            if (t[i] && t[i] != ~0ull) std::fprintf(stderr, "trace %-26s %8.2f us\n", nm[i], 1e-3 * double(t[i] - t[0]));
        return;
    }
    if (!M->use_graphs || !ge || ge->runs == 0) {
        eval_equal_body(M, nc, h0->si_alpha, h0->b, grad, keep_chat);
        CK(cudaStreamSynchronize(M->st));
        if (M->use_graphs) {
            if (!ge) {
                M->graphs.push_back(fmtgp_model::GraphEntry{});
                ge = &M->graphs.back();
                ge->nc = nc;
                ge->grad = grad;
                ge->keep_chat = keep_chat;
                ge->si_alpha = h0->si_alpha;
                ge->prof = prof;
                std::memcpy(ge->b, h0->b, sizeof(ge->b));
            }
            ge->runs = 1;
        }
        return;
    }
    if (!ge->exec) {
        cudaGraph_t graph = nullptr;
        M->prof.capture_list = &ge->recs;
        const bool hv = dig_use_hv(M, nc, keep_chat);
        ge->dig_recs.clear();
        if (hv) dig_rec = &ge->dig_recs;
        CK(cudaStreamBeginCapture(M->st, cudaStreamCaptureModeThreadLocal));
        try {
            eval_equal_body(M, nc, h0->si_alpha, h0->b, grad, keep_chat);
        } catch (...) {
            dig_rec = nullptr;
            cudaStreamEndCapture(M->st, &graph);
            if (graph) cudaGraphDestroy(graph);
            M->prof.capture_list = nullptr;
            throw;
        }
        dig_rec = nullptr;
        CK(cudaStreamEndCapture(M->st, &graph));
        M->prof.capture_list = nullptr;
        CK(cudaGraphInstantiate(&ge->exec, graph, 0));
        if (hv) {
            // the kernel node of every recorded launch (each kernel appears once in this graph)
            size_t cnt = 0;
            CK(cudaGraphGetNodes(graph, nullptr, &cnt));
            std::vector<cudaGraphNode_t> nodes(cnt);
            CK(cudaGraphGetNodes(graph, nodes.data(), &cnt));
            ge->dig_nodes.assign(ge->dig_recs.size(), nullptr);
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType ty;
                CK(cudaGraphNodeGetType(nd, &ty));
                if (ty != cudaGraphNodeTypeKernel) continue;
                cudaKernelNodeParams kp{};
                CK(cudaGraphKernelNodeGetParams(nd, &kp));
                for (size_t i = 0; i < ge->dig_recs.size(); ++i)
                    if (ge->dig_recs[i].func == kp.func) ge->dig_nodes[i] = nd;
            }
            for (cudaGraphNode_t nd : ge->dig_nodes)
                if (!nd) throw Fail{FMTGP_ERR_CUDA, "graph: captured digital kernel node not found"};
            ge->graph = graph;  // node handles stay valid with the template graph
        } else {
            cudaGraphDestroy(graph);
        }
    }
    bool spin = false;
    const unsigned long long seq = ++M->done_seq;
    if (!ge->dig_recs.empty()) {  // this fit's hyperparameter values into the captured kernels
        DigHyperVals hvv{};
        fill_hv(M, hvv);
        for (size_t i = 0; i < ge->dig_recs.size(); ++i) {
            DigLaunchRec& r = ge->dig_recs[i];
            r.a.hv = hvv;
            r.a.seq = seq;
            if (r.a.done_flag) spin = true;
            void* args[5] = {&r.a, &r.ints[0], &r.ints[1], &r.ints[2], &r.ints[3]};
            cudaKernelNodeParams kp{};
            kp.func = const_cast<void*>(r.func);
            kp.gridDim = r.grid;
            kp.blockDim = r.block;
            kp.sharedMemBytes = static_cast<unsigned>(r.smem);
            kp.kernelParams = args;
            CK(cudaGraphExecKernelNodeSetParams(ge->exec, ge->dig_nodes[i], &kp));
        }
    }
    ++M->spec_version;
    CK(cudaGraphLaunch(ge->exec, M->st));
    if (spin && !prof) {
        // the record is complete once the completion word carries this fit's sequence number;
        // the graph retires asynchronously (stream order protects every later call).  A fault or a
        // stall past ~2 s falls back to the stream synchronisation, which reports it.
        const auto t0 = std::chrono::steady_clock::now();
        while (*M->h_done != seq) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
                CK(cudaStreamSynchronize(M->st));
                break;
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    } else {
        CK(cudaStreamSynchronize(M->st));
    }
    if (prof) M->prof.add_graph(ge->recs);
    ge->runs++;
}

void remember_hyper(fmtgp_model* M, const fmtgp_hyper* h) {
    M->last_gamma = h->gamma;
    M->last_eta.assign(h->eta, h->eta + M->d);
    M->last_R = task_gram(M, h);
    M->last_alpha = h->si_alpha;
    for (int i = 0; i < 4; ++i) M->last_b[i] = h->b[i];
    M->fit_dirty = true;  // device copy (posterior kernels only) refreshed lazily
}

void upload_fit(fmtgp_model* M) {
    if (!M->fit_dirty) return;
    std::vector<double> buf(MAXD + MAXT * MAXT, 0.0);
    for (int j = 0; j < M->d; ++j) buf[j] = M->last_eta[j];
    for (size_t k = 0; k < M->last_R.size(); ++k) buf[MAXD + k] = M->last_R[k];
    CK(cudaMemcpyAsync(M->d_fit, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice, M->st));
    CK(cudaStreamSynchronize(M->st));
    M->fit_dirty = false;
}

// nll over a batch with the reference's escalation schedule per candidate
void nll_batch_impl(fmtgp_model* M, int nc, const fmtgp_hyper* hin, bool grad, fmtgp_result* out, bool keep_chat) {
    if (!M->have_y) invalid("nll: observations not set (fmtgp_model_set_y)");
    for (int c = 0; c < nc; ++c) validate_hyper(M, hin + c);
    if (!M->equal) {
        if (nc != 1) throw Fail{FMTGP_ERR_UNSUPPORTED, "nll_batch: unequal sample sizes support one candidate"};
        unequal::nll(M->uneq, M, hin, grad, out);
        return;
    }
    std::vector<int> todo(nc);
    for (int c = 0; c < nc; ++c) todo[c] = c;
    std::vector<double> scale(nc, 1.0);
    std::vector<int> esc(nc, 0);
    std::vector<int> status(nc, FMTGP_OK);
    // one launch serves candidates of one base kernel only: the Walsh order weights b (digital) or
    // the Bernoulli order (lattice) select the kernel code and the design-time kappa table, so
    // candidates are grouped by them (stable) and every group is evaluated on its own
    auto same_kernel = [&](int x, int y) {
        return M->lattice ? hin[x].si_alpha == hin[y].si_alpha : std::memcmp(hin[x].b, hin[y].b, sizeof(hin[x].b)) == 0;
    };
    {
        std::vector<int> grouped;
        std::vector<char> used(nc, 0);
        for (int c = 0; c < nc; ++c) {
            if (used[c]) continue;
            for (int e = c; e < nc; ++e)
                if (!used[e] && same_kernel(c, e)) used[e] = 1, grouped.push_back(e);
        }
        todo.swap(grouped);
    }
    for (int attempt = 0; !todo.empty(); ++attempt) {
        for (size_t base = 0, cnt = 0; base < todo.size(); base += cnt) {
            cnt = 1;
            while (base + cnt < todo.size() && int(cnt) < M->max_cand && same_kernel(todo[base], todo[base + cnt])) ++cnt;
            const int nb = int(cnt);
            std::vector<const fmtgp_hyper*> hs(nb);
            std::vector<double> sc(nb);
            std::vector<int> es(nb);
            for (int i = 0; i < nb; ++i) {
                hs[i] = hin + todo[base + i];
                sc[i] = scale[todo[base + i]];
                es[i] = attempt;
            }
            eval_equal(M, nb, hs.data(), sc.data(), grad, keep_chat && todo[base] == 0 && nb == 1);
            std::vector<fmtgp_result> tmp(nb);
            finish_results(M, nb, hs.data(), grad, tmp.data(), sc.data(), es.data());
            for (int i = 0; i < nb; ++i) {
                const int c = todo[base + i];
                out[c] = tmp[i];
                if (nonreal_of(M, i)) status[c] = FMTGP_ERR_NONREAL;
                else if (M->h_bad[i] != BAD_NONE) status[c] = FMTGP_ERR_SCHUR;
                else status[c] = FMTGP_OK;
            }
        }
        std::vector<int> next;
        for (int c : todo)
            if (status[c] == FMTGP_ERR_SCHUR) {
                if (attempt + 1 > 6) continue;  // schedule exhausted (gp_core.cpp:100)
                scale[c] *= 10.0;
                next.push_back(c);
            }
        todo.swap(next);
    }
    for (int c = 0; c < nc; ++c) out[c].status = status[c];
}

long long slots_of(const fmtgp_model* M, int m) { return M->lattice ? (m > 0 ? (1ll << (m - 1)) : 1) : (1ll << m); }

void model_create_impl(const fmtgp_design* dz, int device, int max_cand, fmtgp_model** out) {
    if (!dz || !out) invalid("model_create: null argument");
    if (dz->kind != 0 && dz->kind != 1) invalid("design: kind must be 0 (lattice) or 1 (digital)");
    if (dz->d < 1 || dz->d > MAXD) throw Fail{FMTGP_ERR_UNSUPPORTED, "design: d must be in [1, 16]"};
    if (dz->L < 1 || dz->L > MAXT) invalid("make_design: at most 8 tasks supported");
    if (!dz->m || !dz->shift_bits) invalid("design: null m / shift_bits");
    for (int l = 0; l < dz->L; ++l) {
        if (dz->m[l] < 0 || dz->m[l] > 27) invalid("design: log2 size out of range");
        if (l + 1 < dz->L && dz->m[l] < dz->m[l + 1]) invalid("build_spectrum: task sizes must be descending");
    }
    if (dz->kind == 0) {
        if (!dz->g || dz->n_max == 0 || (dz->n_max & (dz->n_max - 1)) || dz->n_max < (1ull << dz->m[0]))
            invalid("lattice design: bad generating vector / n_max");
    } else {
        if (!dz->columns || dz->m_cols < dz->m[0] || dz->m_cols > 64) invalid("digital design: bad columns");
    }
    if (max_cand < 1) max_cand = 1;
    CK(cudaSetDevice(device));
    auto* M = new fmtgp_model;
    try {
        M->dev = device;
        CK(cudaStreamCreateWithFlags(&M->st, cudaStreamNonBlocking));
        M->kind = dz->kind;
        M->lattice = dz->kind == 0;
        M->d = dz->d;
        M->T = dz->L;
        M->max_cand = max_cand;
        if (const char* e = std::getenv("FMTGP_KAPPA_TABLE")) M->kap_enabled = e[0] != '0';
        if (const char* e = std::getenv("FMTGP_CLASSES")) M->class_mode = e[0] != '0';
        if (const char* e = std::getenv("FMTGP_DIG_TAIL")) M->dig_tail = std::atoi(e);
        if (const char* e = std::getenv("FMTGP_ZERO_COPY")) M->zero_copy = e[0] != '0';
        if (const char* e = std::getenv("FMTGP_ZERO_COPY_HYPER")) M->zero_copy_hyper = e[0] != '0';
        if (const char* e = std::getenv("FMTGP_HV_PARAMS")) M->hv_params = e[0] != '0';
        if (const char* e = std::getenv("FMTGP_TRACE"))
            if (e[0] == '1') M->d_trace = dalloc<unsigned long long>(16);
        M->off[0] = 0;
        for (int l = 0; l < M->T; ++l) {
            M->m[l] = dz->m[l];
            M->n[l] = 1ll << dz->m[l];
            M->off[l + 1] = M->off[l] + M->n[l];
            if (M->m[l] != M->m[0]) M->equal = false;
        }
        M->N = M->off[M->T];
        M->tw = twiddles_for(device);
        // pairs, row by row
        for (int a = 0; a < M->T; ++a)
            for (int b = a; b < M->T; ++b) {
                M->pa.push_back(a);
                M->pb.push_back(b);
            }
        M->P = int(M->pa.size());
        M->poff.resize(M->P);
        M->pslots.resize(M->P);
        long long acc = 0;
        for (int p = 0; p < M->P; ++p) {
            M->poff[p] = acc;
            M->pslots[p] = slots_of(M, M->m[M->pa[p]]);
            acc += M->pslots[p];
        }
        M->total_slots = acc;
        M->toff_slots.resize(M->T);
        acc = 0;
        for (int t = 0; t < M->T; ++t) {
            M->toff_slots[t] = acc;
            acc += slots_of(M, M->m[t]);
        }
        M->task_slots = acc;
        // design tables
        M->shifts.assign(dz->shift_bits, dz->shift_bits + size_t(M->T) * M->d);
        std::vector<uint64_t> offs(size_t(M->P) * MAXD, 0);
        for (int p = 0; p < M->P; ++p)
            for (int j = 0; j < M->d; ++j) {
                const uint64_t sa = dz->shift_bits[M->pa[p] * M->d + j] & MASK53;
                const uint64_t sb = dz->shift_bits[M->pb[p] * M->d + j] & MASK53;
                offs[size_t(p) * MAXD + j] = M->lattice ? ((sa - sb) & MASK53) : (sa ^ sb);
            }
        M->d_shifts = dalloc<uint64_t>(M->shifts.size());
        CK(cudaMemcpy(M->d_shifts, M->shifts.data(), M->shifts.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        M->d_fit = dalloc<double>(MAXD + MAXT * MAXT);
        M->d_c = dalloc<double>(M->N);
        if (dz->kind == 0) {
            M->n_max = dz->n_max;
            while ((1ull << M->mgen) < M->n_max) ++M->mgen;
        }
        M->d_offs = dalloc<uint64_t>(offs.size());
        CK(cudaMemcpy(M->d_offs, offs.data(), offs.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        if (M->lattice) {
            M->d_g = dalloc<uint64_t>(M->d);
            CK(cudaMemcpy(M->d_g, dz->g, M->d * sizeof(uint64_t), cudaMemcpyHostToDevice));
        } else {
            M->m_cols = dz->m_cols;
            M->d_cols = dalloc<uint64_t>(size_t(M->d) * M->m_cols);
            CK(cudaMemcpy(M->d_cols, dz->columns, size_t(M->d) * M->m_cols * sizeof(uint64_t),
                          cudaMemcpyHostToDevice));
        }
        M->d_pa = dalloc<int>(M->P);
        M->d_pb = dalloc<int>(M->P);
        CK(cudaMemcpy(M->d_pa, M->pa.data(), M->P * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(M->d_pb, M->pb.data(), M->P * sizeof(int), cudaMemcpyHostToDevice));
        // distinct pair offsets (diagonal pairs share offset 0): the transforms run per class
        std::vector<int> pofs(M->P);
        std::vector<uint64_t> uniq;
        for (int p = 0; p < M->P; ++p) {
            int found = -1;
            for (int o = 0; o < M->nofs; ++o)
                if (std::equal(offs.begin() + size_t(p) * MAXD, offs.begin() + size_t(p + 1) * MAXD,
                               uniq.begin() + size_t(o) * MAXD))
                    found = o;
            if (found < 0) {
                uniq.insert(uniq.end(), offs.begin() + size_t(p) * MAXD, offs.begin() + size_t(p + 1) * MAXD);
                found = M->nofs++;
            }
            pofs[p] = found;
        }
        M->h_pair_ofs = pofs;
        M->d_pair_ofs = dalloc<int>(M->P);
        M->d_ofs = dalloc<uint64_t>(uniq.size());
        CK(cudaMemcpy(M->d_pair_ofs, pofs.data(), M->P * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(M->d_ofs, uniq.data(), uniq.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        // transform geometry per length: tiles sized from all vectors of that length
        {
            long long tot[28] = {0};
            long long all = 0;
            for (int p = 0; p < M->P; ++p) {
                tot[M->m[M->pa[p]]] += (1ll << M->m[M->pa[p]]) * max_cand;
                all += (1ll << M->m[M->pa[p]]) * max_cand;
            }
            for (int mm = 0; mm < 28; ++mm) M->geo_m[mm] = Geo::make(mm, M->lattice, tot[mm]);
            M->split = all <= (1ll << 22);
            // fused lattice path: its row split becomes the slot layout of every vector of that length
            const char* lf = std::getenv("FMTGP_LAT_FUSED");
            if (M->equal && M->lattice && M->class_mode && !(lf && lf[0] == '0') &&
                LatGeo::make(M->m[0], M->nofs, M->T, M->d, M->lgeo)) {
                M->lat = true;
                M->geo_m[M->m[0]] = M->lgeo.slot_geo();
            }
        }
        // groups of pairs by generating-task length
        size_t work = 0;
        for (int p = 0; p < M->P; ++p) {
            const int mm = M->m[M->pa[p]];
            auto it = std::find_if(M->groups.begin(), M->groups.end(), [&](const Group& g) { return g.m == mm; });
            if (it == M->groups.end()) {
                M->groups.push_back(Group{});
                M->groups.back().m = mm;
                M->groups.back().geo = M->geo_m[mm];
                it = M->groups.end() - 1;
            }
            it->pairs.push_back(p);
        }
        for (auto& g : M->groups) {
            const int np = int(g.pairs.size());
            std::vector<long long> vo(np);
            for (int q = 0; q < np; ++q) vo[q] = M->poff[g.pairs[q]];
            g.d_vec_pair = dalloc<int>(np);
            g.d_voff = dalloc<long long>(np);
            CK(cudaMemcpy(g.d_vec_pair, g.pairs.data(), np * sizeof(int), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(g.d_voff, vo.data(), np * sizeof(long long), cudaMemcpyHostToDevice));
            if (g.geo.two) work = std::max(work, size_t(np) * max_cand * (size_t(1) << g.geo.lt));
        }
        for (int t = 0; t < M->T; ++t) {
            const int mm = M->m[t];
            auto it = std::find_if(M->tgroups.begin(), M->tgroups.end(), [&](const TaskGroup& g) { return g.m == mm; });
            if (it == M->tgroups.end()) {
                M->tgroups.push_back(TaskGroup{});
                M->tgroups.back().m = mm;
                M->tgroups.back().geo = M->geo_m[mm];
                it = M->tgroups.end() - 1;
            }
            it->tasks.push_back(t);
        }
        for (auto& tg : M->tgroups) {
            const int nt = int(tg.tasks.size());
            std::vector<long long> yo(nt), so(nt);
            for (int q = 0; q < nt; ++q) {
                yo[q] = M->off[tg.tasks[q]];
                so[q] = M->toff_slots[tg.tasks[q]];
            }
            tg.d_yoff = dalloc<long long>(nt);
            tg.d_soff = dalloc<long long>(nt);
            CK(cudaMemcpy(tg.d_yoff, yo.data(), nt * sizeof(long long), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(tg.d_soff, so.data(), nt * sizeof(long long), cudaMemcpyHostToDevice));
            if (tg.geo.two) work = std::max(work, size_t(nt) * (size_t(1) << tg.geo.lt));
        }
        const size_t es = elem_size(M);
        M->work_elems = work;
        M->d_work = dalloc<char>(std::max<size_t>(work, 1) * es);
        if (M->split) {
            size_t gen = 0;
            for (auto& g : M->groups) gen = std::max(gen, g.pairs.size() * size_t(max_cand) * (size_t(1) << g.m));
            M->d_gen = dalloc<double>(gen);
        }
        M->d_y = dalloc<double>(M->N);
        M->d_yhat = dalloc<char>(M->task_slots * es);
        if (M->lat) M->d_yperm = dalloc<char>(M->task_slots * es);
        // hyper block: eta [mc*d] | gamma [mc] | Rpair [mc*P] | per group: coef [mc*np] | xi [mc*np]
        {
            size_t len = size_t(max_cand) * (M->d + 1 + M->P);
            for (auto& g : M->groups) len += 2 * size_t(max_cand) * g.pairs.size();
            M->hyp_len = len;
            M->d_hyp = dalloc<double>(len);
            CK(cudaMallocHost(reinterpret_cast<void**>(&M->h_hyp), len * sizeof(double)));
            std::memset(M->h_hyp, 0, len * sizeof(double));
            M->d_eta = M->d_hyp;
            M->d_gamma = M->d_eta + size_t(max_cand) * M->d;
            M->d_Rpair = M->d_gamma + max_cand;
            double* cur = M->d_Rpair + size_t(max_cand) * M->P;
            for (auto& g : M->groups) {
                g.d_coef = cur;
                g.d_xi = cur + size_t(max_cand) * g.pairs.size();
                cur += 2 * size_t(max_cand) * g.pairs.size();
            }
        }
        M->d_lam = dalloc<char>(size_t(max_cand) * M->total_slots * es);
        M->d_laminv = dalloc<char>(size_t(M->total_slots) * es);
        M->d_chat = dalloc<char>(size_t(M->task_slots) * es);
        {
            std::vector<int> iota(M->P);
            std::vector<long long> cvo(M->P);
            for (int i = 0; i < M->P; ++i) iota[i] = i, cvo[i] = (long long)i * M->pslots[0];
            M->d_iota = dalloc<int>(M->P);
            M->d_cvoff = dalloc<long long>(M->P);
            CK(cudaMemcpy(M->d_iota, iota.data(), M->P * sizeof(int), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(M->d_cvoff, cvo.data(), M->P * sizeof(long long), cudaMemcpyHostToDevice));
            std::vector<double> ones(size_t(max_cand) * M->P, 1.0), zeros(size_t(max_cand) * M->P, 0.0);
            M->d_ones = dalloc<double>(ones.size());
            M->d_zeros = dalloc<double>(zeros.size());
            CK(cudaMemcpy(M->d_ones, ones.data(), ones.size() * sizeof(double), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(M->d_zeros, zeros.data(), zeros.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
        if (M->equal && !M->lattice && DigGeo::make(M->m[0], M->nofs, M->dgeo, (long long)M->nofs * max_cand, M->d)) {
            M->dig = true;
            const DigGeo& g = M->dgeo;
            // the fused kernels always stage the class vectors in d_work (column pass -> row
            // pass), also where the generic geometry of this length is single-pass and sized none
            const size_t need = size_t(max_cand) * M->nofs * (size_t(1) << M->m[0]);
            if (M->work_elems < need) {
                if (M->d_work) cudaFree(M->d_work);
                M->d_work = dalloc<char>(need * sizeof(double));
                M->work_elems = need;
            }
            M->d_part_mid = dalloc<double>(size_t(max_cand) * (size_t(1) << g.l1) * (2 + M->P));
            M->d_part_dot = dalloc<double>(size_t(max_cand) * M->nofs * g.nblk_col * (MAXD + 1));
            M->d_counter = dalloc<unsigned int>(size_t(max_cand) * (1 + M->nofs));
            CK(cudaMemset(M->d_counter, 0, sizeof(unsigned int) * max_cand * (1 + M->nofs)));
            M->d_vec_sum = dalloc<double>(size_t(max_cand) * M->nofs * (MAXD + 1));
            const size_t kbytes = size_t(M->nofs) * M->d * (size_t(1) << M->m[0]) * sizeof(double);
            if (kbytes <= (size_t(1) << 30)) M->d_kap = dalloc<double>(kbytes / sizeof(double));
        }
        if (M->lat) {
            const LatGeo& g = M->lgeo;
            M->d_part_mid = dalloc<double>(size_t(max_cand) * (size_t(1) << g.l1) * (2 + M->P));
            // L3 writes one gradient-dot slot per (candidate x class, CTA): grid <= LAT_MAX_INV_GRID
            M->d_part_dot = dalloc<double>(size_t(max_cand) * M->nofs * std::max(g.nblk_col, LAT_MAX_INV_GRID) * (MAXD + 1));
            M->d_counter = dalloc<unsigned int>(size_t(max_cand) * (1 + M->nofs));
            CK(cudaMemset(M->d_counter, 0, sizeof(unsigned int) * max_cand * (1 + M->nofs)));
        }
        if (M->equal) {
            M->d_M = dalloc<char>(size_t(max_cand) * M->total_slots * es);
            const long long ns = M->pslots[0];
            M->nblk_solve = int(std::min<long long>((ns + 255) / 256, 148 * 8));
            M->nblk_grad = grad_blocks(M->lattice, M->groups[0].geo, M->split);
            M->d_pgrad = dalloc<double>(size_t(max_cand) * M->P * M->nblk_grad * (MAXD + 1));
        } else {
            M->nblk_solve = 1;
        }
        M->d_psolve = dalloc<double>(size_t(max_cand) * std::max(M->nblk_solve, 1) * (3 + M->P));
        // one result block [out | bad | imre] -> a single D2H copy per evaluation
        M->res_len = size_t(max_cand) * (NOUT + 1 + 2 * MAXT) + MAXT;
        M->d_res = dalloc<double>(M->res_len);
        CK(cudaMallocHost(reinterpret_cast<void**>(&M->h_res), sizeof(double) * M->res_len));
        {
            void* p = nullptr;
            CK(cudaMallocHost(&p, 64));
            std::memset(p, 0, 64);
            M->h_done = static_cast<volatile unsigned long long*>(p);
        }
        M->d_tau_raw = M->d_res + size_t(max_cand) * (NOUT + 1 + 2 * MAXT);
        M->h_tau_raw = M->h_res + size_t(max_cand) * (NOUT + 1 + 2 * MAXT);
        CK(cudaEventCreateWithFlags(&M->ev_h2d, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&M->ev_set, cudaEventDisableTiming));
        for (int t = 0; t < M->T; ++t) CK(cudaEventCreateWithFlags(&M->ev_task[t], cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&M->st_copy, cudaStreamNonBlocking));
        M->d_out = M->d_res;
        M->d_bad = reinterpret_cast<int*>(M->d_res + size_t(max_cand) * NOUT);
        M->d_imre = reinterpret_cast<unsigned long long*>(M->d_res + size_t(max_cand) * (NOUT + 1));
        M->h_out = M->h_res;
        M->h_bad = reinterpret_cast<int*>(M->h_res + size_t(max_cand) * NOUT);
        M->h_imre = M->h_res + size_t(max_cand) * (NOUT + 1);

        M->d_vecA = dalloc<double>(M->N);
        M->d_vecB = dalloc<double>(M->N);
        M->d_sA = dalloc<char>(M->task_slots * es);
        M->d_sB = dalloc<char>(M->task_slots * es);

        CK(cudaMemsetAsync(M->d_yhat, 0, M->task_slots * es, M->st));
        M->uneq = unequal::create(M);
        CK(cudaStreamSynchronize(M->st));
    } catch (...) {
        fmtgp_model_destroy(M);
        throw;
    }
    *out = M;
}

}  // namespace

void ensure_fit_state(fmtgp_model* M) {
    if (!M->fit_lazy) return;
    const fmtgp_hyper* hs[1] = {&M->fit_h.h};
    eval_equal(M, 1, hs, &M->fit_xi_scale, /*grad=*/false, /*keep_chat=*/true);
    M->fit_lazy = false;
}

void ensure_coefficients(fmtgp_model* M) {
    ensure_fit_state(M);
    if (M->have_c) return;
    if (M->equal) inverse_vector(M, M->d_chat, M->d_c);
    else unequal::coefficients(M->uneq, M, M->d_c);
    M->have_c = true;
}

// ===================================================================== accessors for unequal.cu
namespace fmtgp::hostapi {
cudaStream_t stream(fmtgp_model* M) { return M->st; }
}  // namespace fmtgp::hostapi

#include "unequal_impl.inc"

// Routes the kernels.cu launch brackets to the model's profiler for one API call.
struct ProfGuard {
    Profiler* prev;
    explicit ProfGuard(fmtgp_model* M) : prev(g_prof) { g_prof = (M && M->profiling) ? &M->prof : nullptr; }
    ~ProfGuard() { g_prof = prev; }
};

// fmtgp_nll without the C-ABI guard: one refresh + loss (+ gradient) with escalation; the fit's
// spectrum / chat are re-derived lazily when a later call needs them.
void nll_public(fmtgp_model* M, const fmtgp_hyper* h, bool grad, fmtgp_result* out) {
    M->fit_lazy = false;
    nll_batch_impl(M, 1, h, grad, out, /*keep_chat=*/!M->equal);
    if (out->status != FMTGP_OK) {
        if (out->status == FMTGP_ERR_SCHUR) throw Fail{FMTGP_ERR_SCHUR, "noise escalation schedule exhausted"};
        throw Fail{out->status, "invert_and_logdet: non-real Schur complement"};
    }
    remember_hyper(M, h);
    if (M->equal) {
        M->fit_h.store(h, M->d, M->T);
        M->fit_xi_scale = out->xi_scale;
        M->fit_lazy = true;
    }
    M->have_fit = true;
    M->have_c = false;
    M->have_spec = true;
    M->have_inv = false;
}

// Hyperparameters as the reference's ParamPack (gp_core.cpp:243-304): log gamma, log eta, B, log t,
// log b (digital).  Owns its arrays; view() is a fmtgp_hyper over them.
struct PackedHyper {
    int d, L, s, dig;
    std::vector<double> eta, B, t, xi;
    fmtgp_hyper h{};
    PackedHyper(const fmtgp_model* M, const fmtgp_hyper* init)
        : d(M->d), L(M->T), s(init->s), dig(!M->lattice), eta(init->eta, init->eta + M->d),
          B(init->B, init->B + size_t(M->T) * init->s), t(init->t, init->t + M->T), xi(init->xi, init->xi + M->T) {
        h = *init;
        rebind();
    }
    void rebind() {
        h.eta = eta.data();
        h.B = B.data();
        h.t = t.data();
        h.xi = xi.data();
        h.s = s;
    }
    int count() const { return 1 + d + L * s + L + (dig ? 4 : 0); }
    std::vector<double> pack() const {
        std::vector<double> th;
        th.push_back(std::log(h.gamma));
        for (double v : eta) th.push_back(std::log(v));
        for (double v : B) th.push_back(v);
        for (double v : t) th.push_back(std::log(v));
        if (dig)
            for (int a = 0; a < 4; ++a) th.push_back(std::log(h.b[a]));
        return th;
    }
    void unpack(const std::vector<double>& th) {
        int k = 0;
        h.gamma = std::exp(th[k++]);
        for (auto& v : eta) v = std::exp(th[k++]);
        for (auto& v : B) v = th[k++];
        for (auto& v : t) v = std::exp(th[k++]);
        if (dig)
            for (int a = 0; a < 4; ++a) h.b[a] = std::exp(th[k++]);
        rebind();
    }
};

// loss at the packed point (guarded_loss, gp_core.cpp:306-313: escalation failure -> +inf), with
// the gradient w.r.t. theta when grad != nullptr.  Walsh weights: the DSI base kernel is linear in
// b, so with a single non-zero order b_k d/dlog b_k = sum_j eta_j d/deta_j exactly; a zero weight
// sits at log 0 = -inf where the reference's difference quotient is not finite (gradient 0); with
// several non-zero orders the log b_k components use the reference's own central difference.
double fit_loss(fmtgp_model* M, PackedHyper& P, const std::vector<double>& th, std::vector<double>* grad) {
    P.unpack(th);
    fmtgp_result r{};
    try {
        nll_batch_impl(M, 1, &P.h, grad != nullptr, &r, false);
    } catch (const Fail& f) {  // unequal n reports an exhausted escalation by throwing
        if (f.code != FMTGP_ERR_SCHUR) throw;
        r.status = FMTGP_ERR_SCHUR;
    }
    if (r.status == FMTGP_ERR_NONREAL) throw Fail{FMTGP_ERR_NONREAL, "invert_and_logdet: non-real Schur complement"};
    const bool ok = r.status == FMTGP_OK && std::isfinite(r.nll);
    if (!grad) return ok ? r.nll : INFINITY;
    grad->assign(th.size(), 0.0);
    if (!ok) {
        // infeasible point (escalation exhausted): the reference still differences its guarded
        // loss here and moves off it where a probe is finite (gp_core.cpp:343-351)
        for (size_t i = 0; i < th.size(); ++i) {
            const double hstep = 1e-4 * std::max(1.0, std::abs(th[i]));
            std::vector<double> tp = th;
            tp[i] = th[i] + hstep;
            const double fp = fit_loss(M, P, tp, nullptr);
            tp[i] = th[i] - hstep;
            const double fm = fit_loss(M, P, tp, nullptr);
            (*grad)[i] = (std::isfinite(fp) && std::isfinite(fm)) ? (fp - fm) / (2.0 * hstep) : 0.0;
        }
        P.unpack(th);
        return INFINITY;
    }
    auto& g = *grad;
    int k = 0;
    g[k++] = P.h.gamma * r.dgamma;
    double eta_deta = 0.0;
    for (int j = 0; j < P.d; ++j) {
        g[k++] = P.eta[j] * r.deta[j];
        eta_deta += P.eta[j] * r.deta[j];
    }
    for (int l = 0; l < P.L; ++l)
        for (int q = 0; q < P.s; ++q) g[k++] = r.dB[l * P.s + q];
    for (int l = 0; l < P.L; ++l) g[k++] = P.t[l] * r.dt[l];
    if (P.dig) {
        int nz = 0;
        for (int a = 0; a < 4; ++a) nz += P.h.b[a] != 0.0;
        if (nz == 1) {
            for (int a = 0; a < 4; ++a) g[k + a] = P.h.b[a] != 0.0 ? eta_deta : 0.0;
        } else {
            const std::vector<double> base = th;
            for (int a = 0; a < 4; ++a) {
                if (P.h.b[a] == 0.0) continue;
                const double hstep = 1e-4 * std::max(1.0, std::abs(base[k + a]));
                std::vector<double> tp = base;
                tp[k + a] = base[k + a] + hstep;
                const double fp = fit_loss(M, P, tp, nullptr);
                tp[k + a] = base[k + a] - hstep;
                const double fm = fit_loss(M, P, tp, nullptr);
                g[k + a] = (std::isfinite(fp) && std::isfinite(fm)) ? (fp - fm) / (2.0 * hstep) : 0.0;
            }
            P.unpack(base);
        }
    }
    return r.nll;
}

// fit (gp_core.cpp:317-382): iRprop- on theta.  The loss at the updated theta is the value the
// next step's gradient evaluation returns, so each step costs one NLL+gradient evaluation.
void fit_impl(fmtgp_model* M, const fmtgp_hyper* init, int steps, double* theta_best, double* loss_trace,
              double* step_seconds, fmtgp_fit_report* rep) {
    using clock = std::chrono::steady_clock;
    PackedHyper P(M, init);
    std::vector<double> theta = P.pack();
    const int np = int(theta.size());
    std::vector<double> grad, grad_prev(np, 0.0), step(np, 0.1);
    constexpr double kUp = 1.2, kDown = 0.5, kMax = 1.0, kMin = 1e-6;
    double cur = fit_loss(M, P, theta, &grad);
    if (!std::isfinite(cur)) throw Fail{FMTGP_ERR_INVALID, "fit: initial loss is not finite"};
    double best = cur;
    std::vector<double> best_theta = theta;
    for (int it = 0; it < steps; ++it) {
        const auto tic = clock::now();
        for (int i = 0; i < np; ++i) {
            double gi = grad[i];
            const double sgn = gi * grad_prev[i];
            if (sgn > 0.0) {
                step[i] = std::min(step[i] * kUp, kMax);
            } else if (sgn < 0.0) {
                step[i] = std::max(step[i] * kDown, kMin);
                gi = 0.0;  // iRprop-: skip the update after a sign flip
            }
            if (gi > 0.0) theta[i] -= step[i];
            else if (gi < 0.0) theta[i] += step[i];
            grad_prev[i] = gi;
        }
        // the loss at the new theta; its gradient drives the next step (not needed after the last)
        cur = fit_loss(M, P, theta, it + 1 < steps ? &grad : nullptr);
        if (cur < best) {
            best = cur;
            best_theta = theta;
        }
        loss_trace[it] = best;
        if (step_seconds) step_seconds[it] = std::chrono::duration<double>(clock::now() - tic).count();
    }
    P.unpack(best_theta);
    fmtgp_result r{};
    nll_public(M, &P.h, false, &r);  // model.refresh() at the best parameters
    if (theta_best)
        for (int i = 0; i < np; ++i) theta_best[i] = best_theta[i];
    std::memset(rep, 0, sizeof(*rep));
    rep->steps = steps;
    rep->n_params = np;
    rep->escalations = r.escalations;
    rep->final_loss = best;
    for (int l = 0; l < M->T; ++l) rep->tau[l] = r.tau[l];
}

// ===================================================================== C ABI
extern "C" {

const char* fmtgp_last_error(void) { return g_err.c_str(); }
int fmtgp_abi_version(void) { return 1; }

int fmtgp_model_create(const fmtgp_design* design, int device, int max_candidates, fmtgp_model_t* out) {
    return guarded([&] { model_create_impl(design, device, max_candidates, out); });
}

int fmtgp_model_destroy(fmtgp_model_t M) {
    if (!M) return FMTGP_OK;
    cudaSetDevice(M->dev);
    if (M->st) cudaStreamSynchronize(M->st);
    auto F = [](void* p) {
        if (p) cudaFree(p);
    };
    for (auto& g : M->groups) {
        F(g.d_vec_pair);
        F(g.d_voff);
    }
    for (auto& tg : M->tgroups) {
        F(tg.d_yoff);
        F(tg.d_soff);
    }
    F(M->d_g);
    F(M->d_cols);
    F(M->d_offs);
    F(M->d_shifts);
    F(M->d_fit);
    F(M->d_c);
    F(M->d_pa);
    F(M->d_pb);
    F(M->d_y);
    F(M->d_yhat);
    F(M->d_yperm);
    F(M->d_hyp);
    for (auto& ge : M->graphs) {
        if (ge.exec) cudaGraphExecDestroy(ge.exec);
        if (ge.graph) cudaGraphDestroy(ge.graph);
    }
    if (M->h_hyp) cudaFreeHost(M->h_hyp);
    if (M->h_done) cudaFreeHost(const_cast<unsigned long long*>(M->h_done));
    F(M->d_lam);
    F(M->d_M);
    F(M->d_work);
    F(M->d_gen);
    F(M->d_part_mid);
    F(M->d_part_dot);
    F(M->d_counter);
    F(M->d_trace);
    F(M->d_vec_sum);
    F(M->d_pair_ofs);
    F(M->d_scratch);
    F(M->d_iota);
    F(M->d_cvoff);
    F(M->d_ones);
    F(M->d_zeros);
    F(M->d_ofs);
    F(M->d_kap);
    F(M->d_laminv);
    F(M->d_chat);
    F(M->d_psolve);
    F(M->d_pgrad);
    F(M->d_res);
    if (M->h_res) cudaFreeHost(M->h_res);
    if (M->ev_h2d) cudaEventDestroy(M->ev_h2d);
    if (M->ev_set) cudaEventDestroy(M->ev_set);
    for (int t = 0; t < MAXT; ++t)
        if (M->ev_task[t]) cudaEventDestroy(M->ev_task[t]);
    if (M->st_copy) cudaStreamDestroy(M->st_copy);
    F(M->d_vecA);
    F(M->d_vecB);
    F(M->d_sA);
    F(M->d_sB);
    if (M->uneq) unequal::destroy(M->uneq);

    if (M->st) cudaStreamDestroy(M->st);
    delete M;
    return FMTGP_OK;
}

void* fmtgp_model_stream(fmtgp_model_t M) { return M ? static_cast<void*>(M->st) : nullptr; }

int fmtgp_model_set_y(fmtgp_model_t M, const double* y) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !y) invalid("set_y: null argument");
        CK(cudaSetDevice(M->dev));
        // (splitting one copy over several copy engines measured slower at these sizes; the per-task
        // pipeline overlaps the transforms instead)
        if (M->T > 1 && M->N >= (1ll << 20)) {
            upload_yhat_tau(M, y);
        } else {
            CK(cudaMemcpyAsync(M->d_y, y, sizeof(double) * M->N, cudaMemcpyHostToDevice, M->st));
            CK(cudaEventRecord(M->ev_h2d, M->st));
            compute_yhat_tau(M);
        }
        // the caller may reuse y on return: wait for the copy only (the transform runs on)
        CK(cudaEventSynchronize(M->ev_h2d));
        M->have_fit = false;
        M->fit_lazy = false;
    });
}

// Benchmark observations on the device (bench.cpp:84-101 with problems.cpp): y = problem at the
// design points (level user + 1) + noise; then the same yhat / tau as set_y.  y_host optional.
int fmtgp_model_problem_y(fmtgp_model_t M, const char* problem, const int* user_of_internal, double noise,
                          uint64_t seed, double* y_host) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !problem || !user_of_internal) invalid("problem_y: null argument");
        int pd_d = 0, levels = 0;
        const int k = problem_index(problem, &pd_d, &levels);
        if (k < 0) invalid(std::string("problem_y: unknown problem ") + problem);
        if (pd_d != M->d) invalid("problem_y: the problem's dimension differs from the design's");
        for (int l = 0; l < M->T; ++l)
            if (user_of_internal[l] < 0 || user_of_internal[l] >= levels)
                invalid("problem_y: more tasks than the problem has fidelities");
        CK(cudaSetDevice(M->dev));
        ProblemDesign pd{};
        pd.d = M->d;
        pd.T = M->T;
        pd.lattice = M->lattice ? 1 : 0;
        pd.mgen = M->mgen;
        pd.m_cols = M->m_cols;
        pd.n_max = M->n_max;
        pd.g = M->d_g;
        pd.cols = M->d_cols;
        pd.shifts = M->d_shifts;
        for (int l = 0; l <= M->T; ++l) pd.off[l] = M->off[l];
        problem_y(k, pd, user_of_internal, noise, seed, M->d_y, M->st);
        CK(cudaGetLastError());
        compute_yhat_tau(M);
        if (y_host) {
            CK(cudaMemcpyAsync(y_host, M->d_y, sizeof(double) * M->N, cudaMemcpyDeviceToHost, M->st));
            CK(cudaStreamSynchronize(M->st));
        }
        M->have_fit = false;
        M->fit_lazy = false;
    });
}

int fmtgp_problem_eval(const char* problem, int level, const double* X, uint64_t count, double* out, int device) {
    return guarded([&] {
        if (!problem || (count && (!X || !out))) invalid("problem_eval: null argument");
        int pd_d = 0, levels = 0;
        const int k = problem_index(problem, &pd_d, &levels);
        if (k < 0) invalid(std::string("problem_eval: unknown problem ") + problem);
        if (level < 1 || level > levels) invalid("problem_eval: level out of range");
        if (count == 0) return;
        CK(cudaSetDevice(device));
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        double* d_buf = nullptr;
        const size_t nx = size_t(count) * pd_d;
        cudaError_t e = cudaMallocAsync(&d_buf, sizeof(double) * (nx + count), s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_buf, X, sizeof(double) * nx, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
            problem_eval(k, level, pd_d, d_buf, count, d_buf + nx, s);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_buf + nx, sizeof(double) * count, cudaMemcpyDeviceToHost, s);
        if (d_buf) cudaFreeAsync(d_buf, s);
        const cudaError_t e2 = cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        CK(e);
        CK(e2);
    });
}

int fmtgp_model_set_y_device(fmtgp_model_t M, const double* y) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !y) invalid("set_y_device: null argument");
        CK(cudaSetDevice(M->dev));
        CK(cudaMemcpyAsync(M->d_y, y, sizeof(double) * M->N, cudaMemcpyDeviceToDevice, M->st));
        compute_yhat_tau(M);
        M->have_fit = false;
        M->fit_lazy = false;
    });
}

int fmtgp_build_spectrum(fmtgp_model_t M, const fmtgp_hyper* h) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M) invalid("build_spectrum: null model");
        CK(cudaSetDevice(M->dev));
        validate_hyper(M, h);
        ensure_fit_state(M);  // a pending fit keeps its chat / coefficients
        const double one = 1.0;
        const fmtgp_hyper* hs[1] = {h};
        upload_hyper(M, 1, hs, &one);
        build_spectra(M, 1, h->si_alpha, h->b);
        CK(cudaStreamSynchronize(M->st));
        remember_hyper(M, h);
        M->have_spec = true;
        M->have_inv = false;
    });
}

// build_spectrum(design, R_internal, spatial, xi_internal) with an explicit task Gram matrix
// (the exact fast_gram.hpp:34-36 signature): R is any symmetric L x L (row-major).
int fmtgp_build_spectrum_R(fmtgp_model_t M, const double* R, const fmtgp_spatial* sp, const double* xi) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !R || !sp || !sp->eta || !xi) invalid("build_spectrum: null argument");
        if (M->lattice && sp->si_alpha != 1 && sp->si_alpha != 2) invalid("si_bernoulli_1d: alpha must be 1 or 2");
        CK(cudaSetDevice(M->dev));
        ensure_fit_state(M);
        // express R through the hyperparameter record: B = 0 (s = 0) is not general, so load the
        // packed block directly: coefficients are R_ab * sqrt(n_b / n_a)
        const int T = M->T;
        std::vector<double> Bf(size_t(T) * T, 0.0), tv(T, 1.0);
        fmtgp_hyper h{};
        h.gamma = sp->gamma;
        h.eta = sp->eta;
        h.si_alpha = sp->si_alpha;
        for (int i = 0; i < 4; ++i) h.b[i] = sp->b[i];
        h.B = Bf.data();
        h.s = T;
        h.t = tv.data();
        h.xi = xi;
        const double one = 1.0;
        const fmtgp_hyper* hs[1] = {&h};
        fill_hyper(M, 1, hs, &one);
        // overwrite Rpair and the per-group coefficients with the explicit R
        double* Rp = M->h_hyp + size_t(M->max_cand) * (M->d + 1);
        for (int p = 0; p < M->P; ++p) Rp[p] = R[M->pa[p] * T + M->pb[p]];
        double* cur = Rp + size_t(M->max_cand) * M->P;
        for (auto& g : M->groups) {
            const int np = int(g.pairs.size());
            for (int q = 0; q < np; ++q) {
                const int p = g.pairs[q];
                cur[q] = R[M->pa[p] * T + M->pb[p]] * std::sqrt(double(M->n[M->pb[p]]) / double(M->n[M->pa[p]]));
            }
            cur += 2 * size_t(M->max_cand) * np;
        }
        copy_hyper(M);
        build_spectra(M, 1, sp->si_alpha, sp->b);
        CK(cudaStreamSynchronize(M->st));
        M->last_gamma = sp->gamma;
        M->last_eta.assign(sp->eta, sp->eta + M->d);
        M->last_R.assign(R, R + size_t(T) * T);
        M->last_alpha = sp->si_alpha;
        for (int i = 0; i < 4; ++i) M->last_b[i] = sp->b[i];
        M->fit_dirty = true;
        M->have_spec = true;
        M->have_inv = false;
    });
}

int fmtgp_spectrum_read(fmtgp_model_t M, int l, int lp, double* re, double* im) {
    return guarded([&] {
        if (!M || !re || !im) invalid("spectrum_read: null argument");
        if (!M->have_spec) invalid("spectrum_read: no spectrum built");
        ensure_fit_state(M);
        if (l < 0 || lp < l || lp >= M->T) invalid("pair_index: need 0 <= l <= lp < L");
        const int p = pair_index(M->T, l, lp);
        const long long ns = M->pslots[p], n = M->n[l];
        std::vector<double> buf(size_t(ns) * (M->lattice ? 2 : 1));
        CK(cudaMemcpy(buf.data(), static_cast<char*>(M->d_lam) + M->poff[p] * elem_size(M), buf.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
        if (!M->lattice) {
            for (long long k = 0; k < n; ++k) {
                re[k] = buf[k];
                im[k] = 0.0;
            }
            return;
        }
        const Geo g = M->geo_m[M->m[l]];
        for (long long k = 0; k < n; ++k) {
            if (n == 1) {
                re[0] = buf[0];
                im[0] = 0.0;
                break;
            }
            const long long half = n / 2;
            if (k == 0) {
                re[k] = buf[0];
                im[k] = 0.0;
            } else if (k == half) {
                re[k] = buf[1];
                im[k] = 0.0;
            } else if (k < half) {
                const long long q = g.pos_of(k);
                re[k] = buf[2 * q];
                im[k] = buf[2 * q + 1];
            } else {
                const long long q = g.pos_of(n - k);
                re[k] = buf[2 * q];
                im[k] = -buf[2 * q + 1];
            }
        }
    });
}

int fmtgp_invert_and_logdet(fmtgp_model_t M, double* logdet) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !logdet) invalid("invert_and_logdet: null argument");
        if (!M->have_spec) invalid("invert_and_logdet: no spectrum built");
        ensure_fit_state(M);
        CK(cudaSetDevice(M->dev));
        if (!M->equal) {
            unequal::invert(M->uneq, M, logdet);
            M->have_inv = true;
            return;
        }
        CK(cudaMemsetAsync(M->d_bad, 0x7f, sizeof(int), M->st));
        CK(cudaMemsetAsync(M->d_bad + 1, 0, sizeof(int), M->st));
        SolveArgs sa{};
        sa.T = M->T;
        sa.P = M->P;
        sa.lattice = M->lattice;
        sa.nslots = M->pslots[0];
    sa.has_nyq = M->n[0] >= 2;
        sa.cstride = M->total_slots;
        sa.lam = M->d_lam;
        sa.yhat = M->d_sA;  // zero right-hand side: logdet and the inverse only
        CK(cudaMemsetAsync(M->d_sA, 0, M->task_slots * elem_size(M), M->st));
        sa.lam_inv = M->d_laminv;
        sa.partial = M->d_psolve;
        sa.bad = M->d_bad;
        sa.imre = M->d_imre;
        CK(cudaMemsetAsync(M->d_imre, 0, sizeof(unsigned long long) * 2 * MAXT, M->st));
        sa.nblk = M->nblk_solve;
        solve_equal(sa, 1, M->st);
        FinalArgs fa{};
        fa.T = M->T;
        fa.P = M->P;
        fa.d = M->d;
        fa.ncand = 1;
        fa.nblk_solve = M->nblk_solve;
        fa.solve_partial = M->d_psolve;
        fa.out = M->d_out;
        finalize(fa, M->st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(M->h_out, M->d_out, sizeof(double) * NOUT, cudaMemcpyDeviceToHost, M->st));
        CK(cudaMemcpyAsync(M->h_bad, M->d_bad, sizeof(int) * 2, cudaMemcpyDeviceToHost, M->st));
        CK(cudaMemcpyAsync(M->h_imre, M->d_imre, sizeof(double) * 2 * MAXT, cudaMemcpyDeviceToHost, M->st));
        CK(cudaStreamSynchronize(M->st));
        if (nonreal_of(M, 0)) throw Fail{FMTGP_ERR_NONREAL, "invert_and_logdet: non-real Schur complement"};
        if (M->h_bad[0] != BAD_NONE)
            throw Fail{FMTGP_ERR_SCHUR, "non-positive Schur entry at slot " + std::to_string(M->h_bad[0])};
        M->last_logdet = M->h_out[OUT_LOGDET];
        *logdet = M->last_logdet;
        M->have_inv = true;
    });
}

int fmtgp_solve(fmtgp_model_t M, const double* b, double* x) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !b || !x) invalid("solve: null argument");
        if (!M->have_inv) invalid("solve: no factorisation (invert_and_logdet)");
        CK(cudaSetDevice(M->dev));
        CK(cudaMemcpyAsync(M->d_vecA, b, sizeof(double) * M->N, cudaMemcpyHostToDevice, M->st));
        forward_vector(M, M->d_vecA, M->d_sA);
        if (M->equal) apply_hermitian(M->lattice, M->T, M->pslots[0], M->d_laminv, M->d_sA, M->d_sB, M->st);
        else unequal::apply_inverse(M->uneq, M, M->d_sA, M->d_sB);
        inverse_vector(M, M->d_sB, M->d_vecB);
        CK(cudaMemcpyAsync(x, M->d_vecB, sizeof(double) * M->N, cudaMemcpyDeviceToHost, M->st));
        CK(cudaStreamSynchronize(M->st));
    });
}

int fmtgp_gram_matvec(fmtgp_model_t M, const double* b, double* out) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !b || !out) invalid("gram_matvec: null argument");
        if (!M->have_spec) invalid("gram_matvec: no spectrum built");
        ensure_fit_state(M);
        CK(cudaSetDevice(M->dev));
        CK(cudaMemcpyAsync(M->d_vecA, b, sizeof(double) * M->N, cudaMemcpyHostToDevice, M->st));
        forward_vector(M, M->d_vecA, M->d_sA);
        if (M->equal) apply_hermitian(M->lattice, M->T, M->pslots[0], M->d_lam, M->d_sA, M->d_sB, M->st);
        else unequal::apply_gram(M->uneq, M, M->d_sA, M->d_sB);
        inverse_vector(M, M->d_sB, M->d_vecB);
        CK(cudaMemcpyAsync(out, M->d_vecB, sizeof(double) * M->N, cudaMemcpyDeviceToHost, M->st));
        CK(cudaStreamSynchronize(M->st));
    });
}

int fmtgp_extract_pi(fmtgp_model_t M, double* Pi) {
    return guarded([&] {
        if (!M || !Pi) invalid("extract_pi: null argument");
        if (!M->have_inv) invalid("extract_pi: no factorisation");
        CK(cudaSetDevice(M->dev));
        if (!M->equal) {
            unequal::extract_pi(M->uneq, M, Pi);
            return;
        }
        // Pi = n Lam(0)^-1 (fast_gram.cpp:311-335 with V̄ 1 = sqrt(n) e_0)
        const int T = M->T;
        for (int a = 0; a < T; ++a)
            for (int b = a; b < T; ++b) {
                const int p = pair_index(T, a, b);
                double v = 0.0;
                CK(cudaMemcpy(&v, static_cast<char*>(M->d_laminv) + M->poff[p] * elem_size(M), sizeof(double),
                              cudaMemcpyDeviceToHost));
                Pi[a * T + b] = Pi[b * T + a] = double(M->n[a]) * v;
            }
    });
}

int fmtgp_extract_h(fmtgp_model_t M, double* H_re, double* H_im) {
    return guarded([&] {
        if (!M || !H_re || !H_im) invalid("extract_h: null argument");
        if (!M->have_inv) invalid("extract_h: no factorisation");
        CK(cudaSetDevice(M->dev));
        if (!M->equal) {
            unequal::extract_h(M->uneq, M, H_re, H_im);
            return;
        }
        // equal n: r = L, base = n and H_lk = sqrt(n) Lam(0)^-1_lk = Pi_lk / sqrt(n) (real)
        const int T = M->T;
        std::vector<double> Pi(size_t(T) * T);
        const int rc = fmtgp_extract_pi(M, Pi.data());
        if (rc != FMTGP_OK) throw Fail{rc, fmtgp_last_error()};
        const double s = 1.0 / std::sqrt(double(M->n[0]));
        for (int k = 0; k < T * T; ++k) H_re[k] = Pi[k] * s, H_im[k] = 0.0;
    });
}

int fmtgp_spectrum_read_range(fmtgp_model_t M, int l, int lp, int64_t k0, int64_t count, double* re, double* im) {
    return guarded([&] {
        if (!M || ((!re || !im) && count > 0)) invalid("spectrum_read_range: null argument");
        if (!M->have_spec) invalid("spectrum_read_range: no spectrum built");
        ensure_fit_state(M);
        if (l < 0 || lp < l || lp >= M->T) invalid("pair_index: need 0 <= l <= lp < L");
        const long long n = M->n[l];
        if (k0 < 0 || count < 0 || k0 + count > n) invalid("spectrum_read_range: frequency range outside the pair vector");
        CK(cudaSetDevice(M->dev));
        const int p = pair_index(M->T, l, lp);
        const char* base = static_cast<const char*>(M->d_lam) + M->poff[p] * elem_size(M);
        auto word = [&](long long w) {  // w-th double of the pair's slot vector
            double v = 0.0;
            CK(cudaMemcpy(&v, base + w * sizeof(double), sizeof(double), cudaMemcpyDeviceToHost));
            return v;
        };
        const Geo g = M->geo_m[M->m[l]];
        for (long long k = k0; k < k0 + count; ++k) {
            const long long o = k - k0;
            if (!M->lattice || n == 1) {
                re[o] = word(k), im[o] = 0.0;
            } else if (k == 0 || k == n / 2) {
                re[o] = word(k == 0 ? 0 : 1), im[o] = 0.0;
            } else {
                const bool mirror = k > n / 2;
                const long long q = g.pos_of(mirror ? n - k : k);
                re[o] = word(2 * q);
                im[o] = mirror ? -word(2 * q + 1) : word(2 * q + 1);
            }
        }
    });
}

int fmtgp_trace_inverse(fmtgp_model_t M, double* tr) {
    return guarded([&] {
        if (!M || !tr) invalid("trace_inverse: null argument");
        if (!M->have_inv) invalid("trace_inverse: no factorisation");
        CK(cudaSetDevice(M->dev));
        if (!M->equal) {
            *tr = unequal::trace_inverse(M->uneq, M);
            return;
        }
        const long long ns = M->pslots[0];
        const int T = M->T;
        double acc = 0.0;
        std::vector<double> buf(size_t(ns) * (M->lattice ? 2 : 1));
        for (int a = 0; a < T; ++a) {
            const int p = pair_index(T, a, a);
            CK(cudaMemcpy(buf.data(), static_cast<char*>(M->d_laminv) + M->poff[p] * elem_size(M),
                          buf.size() * sizeof(double), cudaMemcpyDeviceToHost));
            if (M->lattice) {
                acc += buf[0] + (M->n[a] > 1 ? buf[1] : 0.0);
                for (long long q = 1; q < ns; ++q) acc += 2.0 * buf[2 * q];
            } else {
                for (long long q = 0; q < ns; ++q) acc += buf[q];
            }
        }
        *tr = acc;
    });
}

int fmtgp_nll(fmtgp_model_t M, const fmtgp_hyper* h, int want_grad, fmtgp_result* out) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !h || !out) invalid("nll: null argument");
        CK(cudaSetDevice(M->dev));
        nll_public(M, h, want_grad != 0, out);
    });
}

// Measurement: `iters` fmtgp_nll calls from a C loop (no interpreter between calls), each bracketed
// by CUDA events on the model's stream after an optional L2 flush (a cudaMemsetAsync of
// flush_bytes outside the events).  ms[i] = device time of call i, wall_us = mean host wall time
// per call (the API cost the events see as gaps).
int fmtgp_bench_nll(fmtgp_model_t M, const fmtgp_hyper* h, int want_grad, int iters, size_t flush_bytes, double* ms,
                    double* wall_us) {
    return guarded([&] {
        if (!M || !h || iters < 1 || !ms) invalid("bench_nll: bad argument");
        CK(cudaSetDevice(M->dev));
        void* flush = nullptr;
        if (flush_bytes) CK(cudaMalloc(&flush, flush_bytes));
        std::vector<cudaEvent_t> ev(2 * size_t(iters));
        for (auto& e : ev) CK(cudaEventCreate(&e));
        fmtgp_result r{};
        double wall = 0.0;
        int rc = FMTGP_OK;
        for (int i = 0; i < iters && rc == FMTGP_OK; ++i) {
            if (flush) CK(cudaMemsetAsync(flush, i & 0xff, flush_bytes, M->st));
            CK(cudaEventRecord(ev[2 * i], M->st));
            const auto t0 = std::chrono::steady_clock::now();
            rc = fmtgp_nll(M, h, want_grad, &r);
            wall += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            CK(cudaEventRecord(ev[2 * i + 1], M->st));
        }
        CK(cudaStreamSynchronize(M->st));
        for (int i = 0; i < iters; ++i) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]));
            ms[i] = t;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        if (flush) cudaFree(flush);
        if (wall_us) *wall_us = 1e6 * wall / iters;
        if (rc != FMTGP_OK) throw Fail{rc, fmtgp_last_error()};
    });
}

// GCV loss (loss_value with LossKind::gcv, gp_core.cpp:213-226) = ||c||^2 / (tr K^-1)^2 at the
// refreshed (escalated) nugget, c = K^-1 (y - E tau_GCV).  Equal n: the tau_GCV normal equations
// (HH^ tau = E^T K^-2 y, gp_core.cpp:84-87) collapse at frequency 0 to the sample mean, i.e. the
// NMLL tau, so c is the fit's coefficient vector.  Unequal n: tau_GCV from H (extract_pi_h) and two
// solves, the trace by selected inversion of the fold.  Composed of the seam calls.
int fmtgp_gcv(fmtgp_model_t M, const fmtgp_hyper* h, double* loss, double* num, double* tr) {
    int rc = guarded([&] {
        if (!M || !h || !loss) invalid("gcv: null argument");
    });
    if (rc) return rc;
    fmtgp_result r{};
    if ((rc = fmtgp_nll(M, h, 0, &r))) return rc;
    std::vector<double> c(size_t(M->N));
    if (M->equal && (rc = fmtgp_coefficients(M, c.data()))) return rc;
    std::vector<double> xi(h->xi, h->xi + M->T);
    for (int t = 0; t < M->T; ++t) {
        xi[t] = h->xi[t] * r.xi_scale;
        if (r.xi_scale > 1.0 && h->xi[t] == 0.0) xi[t] = 1e-12 * r.xi_scale;  // gp_core.cpp:103-105
    }
    fmtgp_hyper h2 = *h;
    h2.xi = xi.data();
    double ld = 0.0, trace = 0.0;
    if ((rc = fmtgp_build_spectrum(M, &h2))) return rc;
    if ((rc = fmtgp_invert_and_logdet(M, &ld))) return rc;
    if ((rc = fmtgp_trace_inverse(M, &trace))) return rc;
    if (!M->equal) {
        rc = guarded([&] {
            const int T = M->T;
            const long long r_ = M->N / M->n[T - 1];
            std::vector<double> Hre(size_t(T) * r_), Him(Hre.size()), y(size_t(M->N)), w(y.size()), w2(y.size());
            int e = fmtgp_extract_h(M, Hre.data(), Him.data());
            if (e) throw Fail{e, fmtgp_last_error()};
            CK(cudaMemcpy(y.data(), M->d_y, sizeof(double) * M->N, cudaMemcpyDeviceToHost));
            if ((e = fmtgp_solve(M, y.data(), w.data())) || (e = fmtgp_solve(M, w.data(), w2.data())))
                throw Fail{e, fmtgp_last_error()};
            // HHbar tau = E^T K^-2 y (compute_tau_internal, gp_core.cpp:84-87)
            std::vector<double> HH(size_t(T) * T, 0.0), rhs(T, 0.0);
            for (int a = 0; a < T; ++a)
                for (int b = 0; b < T; ++b)
                    for (long long k = 0; k < r_; ++k)
                        HH[a * T + b] += Hre[a * r_ + k] * Hre[b * r_ + k] + Him[a * r_ + k] * Him[b * r_ + k];
            for (int a = 0; a < T; ++a)
                for (long long k = M->off[a]; k < M->off[a + 1]; ++k) rhs[a] += w2[k];
            const std::vector<double> tau = unequal::small_solve(T, HH, rhs);
            for (int a = 0; a < T; ++a)
                for (long long k = M->off[a]; k < M->off[a + 1]; ++k) y[k] -= tau[a];
            if ((e = fmtgp_solve(M, y.data(), c.data()))) throw Fail{e, fmtgp_last_error()};
        });
        if (rc) return rc;
    }
    double s = 0.0;
    for (double v : c) s += v * v;
    *loss = s / (trace * trace);
    if (num) *num = s;
    if (tr) *tr = trace;
    return FMTGP_OK;
}

int fmtgp_fit_param_count(fmtgp_model_t M, int s, int* n) {
    return guarded([&] {
        if (!M || !n || s < 0) invalid("fit_param_count: bad argument");
        *n = 1 + M->d + M->T * s + M->T + (M->lattice ? 0 : 4);
    });
}

int fmtgp_fit(fmtgp_model_t M, const fmtgp_hyper* init, int steps, double* theta_best, double* loss_trace,
              double* step_seconds, fmtgp_fit_report* rep) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !init || !rep || steps < 0 || (steps > 0 && !loss_trace)) invalid("fit: bad argument");
        CK(cudaSetDevice(M->dev));
        validate_hyper(M, init);
        fit_impl(M, init, steps, theta_best, loss_trace, step_seconds, rep);
    });
}

// ---- frequency-sharded lattice fit: one rank's three phases; the caller runs
// the two all-to-alls of the exchange blocks between them and sums the records over ranks.
int fmtgp_shard_setup(fmtgp_model_t M, int rank, int world, int64_t* exchange_elems) {
    return guarded([&] {
        if (!M || !exchange_elems) invalid("shard_setup: null argument");
        if (!M->lat)
            throw Fail{FMTGP_ERR_UNSUPPORTED, "shard_setup: only the fused equal-n lattice fit shards (n >= 2^17, T <= 4)"};
        const LatGeo& g = M->lgeo;
        const int clusters = (1 << g.l1) / 2;
        if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world || clusters % world ||
            g.nblk_col % world || (1 << g.l2) % world)
            invalid("shard_setup: the world size must be a power of two dividing the row clusters and column blocks");
        M->sh_G = world;
        M->sh_g = rank;
        M->sh_lkc = 0;
        *exchange_elems = (int64_t)M->nofs * M->pslots[0] / world;
    });
}

int fmtgp_shard_chunks(fmtgp_model_t M, int chunks) {
    return guarded([&] {
        if (!M) invalid("shard_chunks: null argument");
        if (!M->lat) invalid("shard_chunks: model is not sharded (fmtgp_shard_setup)");
        const LatGeo& g = M->lgeo;
        const int rows = (1 << g.l1) / M->sh_G, ncb = g.nblk_col / M->sh_G;  // rows R, column blocks per rank
        if (chunks < 1 || (chunks & (chunks - 1)) || ncb % chunks || rows % (2 * chunks))
            invalid("shard_chunks: chunks must be a power of two dividing the rank's column blocks and row pairs");
        int l = 0;
        while ((1 << l) < chunks) ++l;
        M->sh_lkc = l;
    });
}

// one column chunk of L1 (chunk 0 also stages the hyperparameters); Y: the forward send buffer
int fmtgp_shard_begin_chunk(fmtgp_model_t M, const fmtgp_hyper* h, int want_grad, double xi_scale, void* Y,
                            int chunk) {
    return guarded([&] {
        if (!M || !h || !Y) invalid("shard_begin_chunk: null argument");
        if (!M->lat) invalid("shard_begin_chunk: model is not sharded (fmtgp_shard_setup)");
        if (chunk < 0 || chunk >= (1 << M->sh_lkc)) invalid("shard_begin_chunk: chunk out of range");
        CK(cudaSetDevice(M->dev));
        if (chunk == 0) {
            if (!M->have_y) invalid("nll: observations not set (fmtgp_model_set_y)");
            validate_hyper(M, h);
            const fmtgp_hyper* hs[1] = {h};
            fill_hyper(M, 1, hs, &xi_scale);
            copy_hyper(M);
            M->sh_args = lat_args(M, 1, h->si_alpha, want_grad != 0);
            M->sh_grad = want_grad != 0;
        }
        M->sh_args.Y = static_cast<double2*>(Y);
        M->sh_args.chunk = chunk;
        lat_phase(M->lgeo, M->sh_args, 1, M->st);
        CK(cudaGetLastError());
    });
}

// one row chunk of L2: reads the forward receive buffer Y, writes the return send buffer Yout
int fmtgp_shard_mid_chunk(fmtgp_model_t M, void* Y, void* Yout, int chunk) {
    return guarded([&] {
        if (!M || !Y || !Yout) invalid("shard_mid_chunk: null argument");
        if (chunk < 0 || chunk >= (1 << M->sh_lkc)) invalid("shard_mid_chunk: chunk out of range");
        if (Y == Yout && M->sh_lkc > 0) invalid("shard_mid_chunk: chunked L2 cannot work in place");
        CK(cudaSetDevice(M->dev));
        M->sh_args.Y = static_cast<double2*>(Y);
        M->sh_args.Yout = static_cast<double2*>(Yout);
        M->sh_args.chunk = chunk;
        lat_phase(M->lgeo, M->sh_args, 2, M->st);
        CK(cudaGetLastError());
    });
}

int fmtgp_shard_begin(fmtgp_model_t M, const fmtgp_hyper* h, int want_grad, double xi_scale, void* Y) {
    return guarded([&] {
        if (!M || !h || !Y) invalid("shard_begin: null argument");
        if (!M->lat) invalid("shard_begin: model is not sharded (fmtgp_shard_setup)");
        if (!M->have_y) invalid("nll: observations not set (fmtgp_model_set_y)");
        validate_hyper(M, h);
        CK(cudaSetDevice(M->dev));
        const fmtgp_hyper* hs[1] = {h};
        fill_hyper(M, 1, hs, &xi_scale);
        copy_hyper(M);
        if (M->sh_lkc) invalid("shard_begin: the exchange is chunked (fmtgp_shard_begin_chunk)");
        M->sh_args = lat_args(M, 1, h->si_alpha, want_grad != 0);
        M->sh_args.Y = static_cast<double2*>(Y);
        M->sh_grad = want_grad != 0;
        lat_phase(M->lgeo, M->sh_args, 1, M->st);
        CK(cudaGetLastError());
    });
}

int fmtgp_shard_mid(fmtgp_model_t M, void* Y) {
    return guarded([&] {
        if (!M || !Y) invalid("shard_mid: null argument");
        CK(cudaSetDevice(M->dev));
        if (M->sh_lkc) invalid("shard_mid: the exchange is chunked (fmtgp_shard_mid_chunk)");
        M->sh_args.Y = static_cast<double2*>(Y);
        M->sh_args.Yout = nullptr;
        M->sh_args.chunk = -1;
        lat_phase(M->lgeo, M->sh_args, 2, M->st);
        CK(cudaGetLastError());
    });
}

int fmtgp_shard_end(fmtgp_model_t M, const void* Cbuf, double* rec) {
    return guarded([&] {
        if (!M || !Cbuf || !rec) invalid("shard_end: null argument");
        CK(cudaSetDevice(M->dev));
        M->sh_args.Cbuf = static_cast<const double2*>(Cbuf);
        if (M->sh_grad) lat_phase(M->lgeo, M->sh_args, 3, M->st);
        else lat_finalize_nograd(M, 1);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(M->h_res, M->d_res, sizeof(double) * M->res_len, cudaMemcpyDeviceToHost, M->st));
        CK(cudaStreamSynchronize(M->st));
        for (int x = 0; x < NOUT; ++x) rec[x] = M->h_out[x];
        rec[NOUT] = double(M->h_bad[0]);
        for (int x = 0; x < 2 * MAXT; ++x) rec[NOUT + 1 + x] = M->h_imre[x];
    });
}

int fmtgp_shard_finish(fmtgp_model_t M, const fmtgp_hyper* h, const double* rec, int want_grad, double xi_scale,
                       int escalations, fmtgp_result* out) {
    return guarded([&] {
        if (!M || !h || !rec || !out) invalid("shard_finish: null argument");
        for (int x = 0; x < NOUT; ++x) M->h_out[x] = rec[x];
        M->h_bad[0] = int(rec[NOUT]);
        for (int x = 0; x < 2 * MAXT; ++x) M->h_imre[x] = rec[NOUT + 1 + x];
        const fmtgp_hyper* hs[1] = {h};
        finish_results(M, 1, hs, want_grad != 0, out, &xi_scale, &escalations);
        out->status = nonreal_of(M, 0) ? FMTGP_ERR_NONREAL : (M->h_bad[0] != BAD_NONE ? FMTGP_ERR_SCHUR : FMTGP_OK);
    });
}

int fmtgp_nll_batch(fmtgp_model_t M, int ncand, const fmtgp_hyper* h, int want_grad, fmtgp_result* out) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !h || !out || ncand < 1) invalid("nll_batch: bad argument");
        CK(cudaSetDevice(M->dev));
        M->fit_lazy = false;
        nll_batch_impl(M, ncand, h, want_grad != 0, out, false);
        M->have_fit = false;
        M->have_spec = false;
        M->have_inv = false;
    });
}

int fmtgp_coefficients(fmtgp_model_t M, double* c) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !c) invalid("coefficients: null argument");
        if (!M->have_fit) invalid("coefficients: model not refreshed (call fmtgp_nll)");
        CK(cudaSetDevice(M->dev));
        ensure_coefficients(M);
        CK(cudaMemcpyAsync(c, M->d_c, sizeof(double) * M->N, cudaMemcpyDeviceToHost, M->st));
        CK(cudaStreamSynchronize(M->st));
    });
}

int fmtgp_posterior_mean(fmtgp_model_t M, int task, const double* X, int64_t count, double* out) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || (!X && count > 0) || (!out && count > 0)) invalid("posterior_mean: null argument");
        if (!M->have_fit) invalid("posterior_mean: model not refreshed");
        if (task < 0 || task >= M->T) invalid("posterior_mean: task out of range");
        if (count <= 0) return;
        CK(cudaSetDevice(M->dev));
        ensure_coefficients(M);
        upload_fit(M);
        int nsplit;
        long long chunk;
        posterior_split(count, M->N, nsplit, chunk);
        double* dX = scratch(M, size_t(count) * (M->d + 1 + nsplit));
        double* dO = dX + size_t(count) * M->d;
        {
            CK(cudaMemcpyAsync(dX, X, sizeof(double) * count * M->d, cudaMemcpyHostToDevice, M->st));
            PostArgs a{};
            a.part = dO + count;
            a.nsplit = nsplit;
            a.chunk = chunk;
            a.lattice = M->lattice;
            a.d = M->d;
            a.T = M->T;
            a.task = task;
            a.si_alpha = M->last_alpha;
            a.mgen = M->mgen;
            a.m_cols = M->m_cols;
            a.n_max = M->n_max;
            a.g = M->d_g;
            a.cols = M->d_cols;
            a.shifts = M->d_shifts;
            for (int i = 0; i < 4; ++i) a.b[i] = M->last_b[i];
            a.eta = M->d_fit;
            a.R = M->d_fit + MAXD;
            a.gamma = M->last_gamma;
            a.tau = M->tau[task];
            for (int l = 0; l < M->T; ++l) {
                a.n[l] = M->n[l];
                a.off[l] = M->off[l];
            }
            a.c = M->d_c;
            a.X = dX;
            a.count = count;
            a.out = dO;
            posterior_mean(a, M->st);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(out, dO, sizeof(double) * count, cudaMemcpyDeviceToHost, M->st));
            CK(cudaStreamSynchronize(M->st));
        }
    });
}

int fmtgp_posterior_var(fmtgp_model_t M, int task, const double* X, int64_t count, double* out) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || (!X && count > 0) || (!out && count > 0)) invalid("posterior_var: null argument");
        if (!M->have_fit) invalid("posterior_var: model not refreshed");
        ensure_fit_state(M);
        if (task < 0 || task >= M->T) invalid("posterior_var: task out of range");
        CK(cudaSetDevice(M->dev));
        if (!M->uneq) throw Fail{FMTGP_ERR_UNSUPPORTED, "posterior_var: needs the fold plan"};
        unequal::posterior_var(M->uneq, M, task, X, count, out);
    });
}

int fmtgp_posterior_cov(fmtgp_model_t M, int task, const double* X, int task2, const double* Xp, int64_t count,
                        double* out) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || (count > 0 && (!X || !Xp || !out))) invalid("posterior_cov: null argument");
        if (!M->have_fit) invalid("posterior_cov: model not refreshed");
        ensure_fit_state(M);
        if (task < 0 || task >= M->T || task2 < 0 || task2 >= M->T) invalid("posterior_cov: task out of range");
        CK(cudaSetDevice(M->dev));
        if (!M->uneq) throw Fail{FMTGP_ERR_UNSUPPORTED, "posterior_cov: needs the fold plan"};
        unequal::posterior_cov(M->uneq, M, task, X, task2, Xp, count, out);
    });
}

// multitask_cubature (cubature.cpp:52-75): mu = tau + gamma R (E^T c), Sigma = gamma R - gamma^2 R Pi R
int fmtgp_cubature(fmtgp_model_t M, double* mu, double* Sigma) {
    return guarded([&] {
        ProfGuard pg_(M);
        if (!M || !mu || !Sigma) invalid("cubature: null argument");
        if (!M->have_fit) invalid("cubature: model not refreshed");
        ensure_fit_state(M);
        CK(cudaSetDevice(M->dev));
        const int T = M->T;
        std::vector<double> Pi(size_t(T) * T), etc(T, 0.0);
        if (M->equal) {
            // Pi = n Lam(0)^-1 from the fitted spectrum's frequency-0 entries; E^T c = sqrt(n) chat(0)
            std::vector<double> A(size_t(T) * T);
            for (int a = 0; a < T; ++a)
                for (int b = a; b < T; ++b) {
                    double v = 0.0;
                    CK(cudaMemcpy(&v, static_cast<char*>(M->d_lam) + M->poff[pair_index(T, a, b)] * elem_size(M),
                                  sizeof(double), cudaMemcpyDeviceToHost));
                    A[a * T + b] = A[b * T + a] = v;
                }
            // Gauss-Jordan inverse (T <= 8)
            std::vector<double> I(size_t(T) * T, 0.0);
            for (int a = 0; a < T; ++a) I[a * T + a] = 1.0;
            for (int k = 0; k < T; ++k) {
                int piv = k;
                for (int i = k + 1; i < T; ++i)
                    if (std::fabs(A[i * T + k]) > std::fabs(A[piv * T + k])) piv = i;
                for (int j = 0; j < T; ++j) {
                    std::swap(A[k * T + j], A[piv * T + j]);
                    std::swap(I[k * T + j], I[piv * T + j]);
                }
                const double dk = A[k * T + k];
                for (int j = 0; j < T; ++j) {
                    A[k * T + j] /= dk;
                    I[k * T + j] /= dk;
                }
                for (int i = 0; i < T; ++i)
                    if (i != k) {
                        const double f = A[i * T + k];
                        for (int j = 0; j < T; ++j) {
                            A[i * T + j] -= f * A[k * T + j];
                            I[i * T + j] -= f * I[k * T + j];
                        }
                    }
            }
            for (int a = 0; a < T; ++a)
                for (int b = 0; b < T; ++b) Pi[a * T + b] = double(M->n[0]) * I[a * T + b];
            ensure_coefficients(M);
            std::vector<double> c(M->N);
            CK(cudaMemcpy(c.data(), M->d_c, sizeof(double) * M->N, cudaMemcpyDeviceToHost));
            for (int l = 0; l < T; ++l)
                for (long long k = M->off[l]; k < M->off[l + 1]; ++k) etc[l] += c[k];
        } else {
            unequal::cubature_terms(M->uneq, M, Pi.data(), etc.data());
        }
        const std::vector<double>& R = M->last_R;
        const double g = M->last_gamma;
        for (int a = 0; a < T; ++a) {
            double s = 0.0;
            for (int b = 0; b < T; ++b) s += R[a * T + b] * etc[b];
            mu[a] = M->tau[a] + g * s;
        }
        std::vector<double> RP(size_t(T) * T, 0.0);
        for (int a = 0; a < T; ++a)
            for (int b = 0; b < T; ++b)
                for (int k = 0; k < T; ++k) RP[a * T + b] += R[a * T + k] * Pi[k * T + b];
        for (int a = 0; a < T; ++a)
            for (int b = 0; b < T; ++b) {
                double s = 0.0;
                for (int k = 0; k < T; ++k) s += RP[a * T + k] * R[k * T + b];
                Sigma[a * T + b] = g * R[a * T + b] - g * g * s;
            }
        for (int a = 0; a < T; ++a)
            for (int b = a + 1; b < T; ++b) Sigma[a * T + b] = Sigma[b * T + a] = 0.5 * (Sigma[a * T + b] + Sigma[b * T + a]);
        for (int a = 0; a < T; ++a)
            if (Sigma[a * T + a] < 0.0 && Sigma[a * T + a] > -1e-12) Sigma[a * T + a] = 0.0;
    });
}

int fmtgp_profile_enable(fmtgp_model_t M, int on) {
    return guarded([&] {
        if (!M) invalid("profile_enable: null model");
        M->prof.reset();
        M->profiling = on != 0;
    });
}

int fmtgp_profile_read(fmtgp_model_t M, int idx, char* name, int name_len, double* total_ms, int* launches) {
    return guarded([&] {
        if (!M || !name || name_len < 1 || !total_ms || !launches) invalid("profile_read: bad argument");
        M->prof.collect();
        if (idx < 0 || idx >= int(M->prof.agg.size())) invalid("profile_read: index out of range");
        const auto& e = M->prof.agg[idx];
        std::snprintf(name, size_t(name_len), "%s", e.first.c_str());
        *total_ms = e.second.first;
        *launches = e.second.second;
    });
}

}  // extern "C"
