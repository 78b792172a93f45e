// extern "C" shim over the UNMODIFIED reference sources (/root/reference/proj/src),
// compiled into oracle/_ref/libfmtgp_ref.so by oracle/Makefile.
//
// TEST INFRASTRUCTURE ONLY.  Used by tests/ (parity checker), by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference leg.
// The product path never loads this library.
//
// Designs are built by hand from explicit generators (the reference's
// make_design only knows its shipped tables; BASELINE configs need seeded
// generating vectors, n_max up to 2^26 and scrambled digital nets), exactly as
// SURVEY.md §8c(4) prescribes: LdDesign is a public aggregate
// (ld_sequences.hpp:56-77) and X is materialised with the reference's own
// lattice_points / digital_net_points (ld_sequences.cpp:31-87).
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "fastmtgp/common.hpp"
#include "fastmtgp/cubature.hpp"
#include "fastmtgp/fast_gram.hpp"
#include "fastmtgp/gp_core.hpp"
#include "fastmtgp/kernels.hpp"
#include "fastmtgp/ld_sequences.hpp"
#include "fastmtgp/problems.hpp"
#include "fastmtgp/rng.hpp"
#include "fastmtgp/transforms.hpp"

// The shipped generator tables are only reached through default_lattice /
// default_digital (make_design), which the oracle never calls.
namespace fastmtgp::embedded {
extern const char* const lattice_table = "";
extern const char* const sobol_table = "";
extern const char* const reference_json = "{}";  // problems.cpp's integral table (not used here)
}  // namespace fastmtgp::embedded

using namespace fastmtgp;

extern "C" {

struct RefDesign {
    int kind;  // 0 lattice, 1 digital
    int d;
    int L;
    const int* m;                  // [L] internal order, descending
    const std::uint64_t* g;        // lattice: [d]
    std::uint64_t n_max;           // lattice: power of two >= 2^m[0]
    const std::uint64_t* columns;  // digital: [d * m_cols], 53-bit msb-aligned
    int m_cols;                    // digital
    const std::uint64_t* shift_bits;  // [L * d] 53-bit fractions
};

struct RefHyper {
    double gamma;
    const double* eta;  // [d]
    int si_alpha;
    double b[4];
    const double* B;  // [L * s] row-major
    int s;
    const double* t;   // [L]
    const double* xi;  // [L]
};

}  // extern "C"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const SchurBreakdown& e) {
        return fail(e, 2);
    } catch (const FastMtgpError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 3);
    }
}

LdDesign make_ld(const RefDesign& rd) {
    LdDesign dz;
    dz.kind = rd.kind == 0 ? SeqKind::lattice : SeqKind::digital;
    dz.d = rd.d;
    dz.L = rd.L;
    dz.seed = 0;
    dz.m.assign(rd.m, rd.m + rd.L);
    dz.n.resize(rd.L);
    dz.offset.assign(rd.L + 1, 0);
    for (int l = 0; l < rd.L; ++l) {
        dz.n[l] = std::uint64_t{1} << rd.m[l];
        dz.offset[l + 1] = dz.offset[l] + dz.n[l];
    }
    dz.N = dz.offset[rd.L];
    dz.internal_to_user.resize(rd.L);
    dz.user_to_internal.resize(rd.L);
    for (int l = 0; l < rd.L; ++l) dz.internal_to_user[l] = dz.user_to_internal[l] = l;
    dz.shift.resize(rd.L);
    dz.shift_bits.resize(rd.L);
    dz.X.resize(rd.L);
    LatticeGenerator lg;
    DigitalGenerator dg;
    if (rd.kind == 0) {
        lg.d = rd.d;
        lg.g.assign(rd.g, rd.g + rd.d);
        lg.n_max = rd.n_max;
    } else {
        dg.d = rd.d;
        dg.t = kDigitalBits;
        dg.m_max = rd.m_cols;
        dg.columns.resize(rd.d);
        for (int j = 0; j < rd.d; ++j)
            dg.columns[j].assign(rd.columns + j * rd.m_cols, rd.columns + (j + 1) * rd.m_cols);
    }
    for (int l = 0; l < rd.L; ++l) {
        dz.shift_bits[l].assign(rd.shift_bits + l * rd.d, rd.shift_bits + (l + 1) * rd.d);
        dz.shift[l].resize(rd.d);
        for (int j = 0; j < rd.d; ++j) dz.shift[l][j] = bits_to_frac(dz.shift_bits[l][j]);
        if (rd.kind == 0)
            dz.X[l] = lattice_points(lg, dz.shift[l], 0, dz.n[l]);
        else
            dz.X[l] = digital_net_points(dg, dz.shift_bits[l], 0, dz.n[l]);
    }
    return dz;
}

Hyperparams make_hyper(const RefDesign& rd, const RefHyper& rh) {
    Hyperparams h;
    h.gamma = rh.gamma;
    h.eta.assign(rh.eta, rh.eta + rd.d);
    h.si_alpha = rh.si_alpha;
    for (int a = 0; a < 4; ++a) h.b[a] = rh.b[a];
    h.B.resize(rd.L, rh.s);
    for (int l = 0; l < rd.L; ++l)
        for (int k = 0; k < rh.s; ++k) h.B(l, k) = rh.B[l * rh.s + k];
    h.t.assign(rh.t, rh.t + rd.L);
    h.xi.assign(rh.xi, rh.xi + rd.L);
    h.tau.assign(rd.L, 0.0);
    h.lengthscales.assign(rd.d, 0.25);
    return h;
}

KernelFamily family_of(const RefDesign& rd) {
    return rd.kind == 0 ? KernelFamily::si_lattice : KernelFamily::dsi_digital;
}

struct RefModel {
    GpModel model;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng.hpp (counter RNG: every seeded input in the reference's tests)
std::uint64_t ref_rand_u64(std::uint64_t seed, std::uint64_t stream, std::uint64_t counter) {
    return rng::rand_u64(seed, stream, counter);
}
double ref_normal(std::uint64_t seed, std::uint64_t stream, std::uint64_t k) { return rng::normal(seed, stream, k); }

// ---- transforms / kernels / points (transforms.cpp, kernels.cpp, ld_sequences.cpp)
std::uint64_t ref_bit_reverse(std::uint64_t i, int m) { return bit_reverse(i, m); }
int ref_fwht(double* a, std::size_t n) {
    return guarded([&] { fwht(a, n); });
}
int ref_fft_bitrev(double* a_interleaved, std::size_t n) {
    return guarded([&] { fft_bitrev(reinterpret_cast<cplx*>(a_interleaved), n); });
}
int ref_fft_bitrev_inv(double* a_interleaved, std::size_t n) {
    return guarded([&] { fft_bitrev_inv(reinterpret_cast<cplx*>(a_interleaved), n); });
}
double ref_si_bernoulli_1d(double x, double xp, int alpha) { return si_bernoulli_1d(x, xp, alpha); }
double ref_dsi_order_1d(int alpha, double x, double xp) { return dsi_order_1d(alpha, x, xp); }

int ref_design_points(const RefDesign* rd, double* out /* N x d, internal order */) {
    return guarded([&] {
        LdDesign dz = make_ld(*rd);
        for (int l = 0; l < dz.L; ++l)
            std::memcpy(out + dz.offset[l] * dz.d, dz.X[l].data(), dz.X[l].size() * sizeof(double));
    });
}

// ---- fast_gram.hpp seam ---------------------------------------------------------
// lam_re/lam_im: pairs (l<=lp) row by row, each of length n_l, concatenated.
int ref_build_spectrum(const RefDesign* rd, const RefHyper* rh, double* lam_re, double* lam_im) {
    return guarded([&] {
        LdDesign dz = make_ld(*rd);
        Hyperparams h = make_hyper(*rd, *rh);
        const Eigen::MatrixXd R = task_gram(h.B, h.t);
        SpatialKernel q = SpatialKernel::from(h, family_of(*rd));
        BlockSpectrum spec = build_spectrum(dz, R, q, h.xi);
        std::size_t o = 0;
        for (const auto& v : spec.lam)
            for (const auto& z : v) {
                lam_re[o] = z.real();
                lam_im[o] = z.imag();
                ++o;
            }
    });
}

// logdet, solve(b) -> x, trace_inverse, Pi (L x L row-major), gram_matvec(b) -> kb.
int ref_invert_solve(const RefDesign* rd, const RefHyper* rh, const double* b, double* x,
                     double* kb, double* logdet, double* trace, double* Pi) {
    return guarded([&] {
        LdDesign dz = make_ld(*rd);
        Hyperparams h = make_hyper(*rd, *rh);
        const Eigen::MatrixXd R = task_gram(h.B, h.t);
        SpatialKernel q = SpatialKernel::from(h, family_of(*rd));
        BlockSpectrum spec = build_spectrum(dz, R, q, h.xi);
        BlockInverse inv = invert_and_logdet(spec);
        *logdet = inv.logdet;
        std::vector<double> bv(b, b + dz.N);
        if (x) {
            std::vector<double> xs = solve(inv, bv);
            std::memcpy(x, xs.data(), xs.size() * sizeof(double));
        }
        if (kb) {
            std::vector<double> ks = gram_matvec(spec, bv);
            std::memcpy(kb, ks.data(), ks.size() * sizeof(double));
        }
        if (trace) *trace = trace_inverse(inv);  // callers pass nullptr to skip it
        if (Pi) {
            PiH ph = extract_pi_h(inv);
            for (int l = 0; l < dz.L; ++l)
                for (int lp = 0; lp < dz.L; ++lp) Pi[l * dz.L + lp] = ph.Pi(l, lp);
        }
    });
}

// Pi (L x L) and H (L x r row-major, r = N / n_{L-1}) of extract_pi_h (fast_gram.cpp:311-335).
int ref_pi_h(const RefDesign* rd, const RefHyper* rh, double* Pi, double* H_re, double* H_im) {
    return guarded([&] {
        LdDesign dz = make_ld(*rd);
        Hyperparams h = make_hyper(*rd, *rh);
        const Eigen::MatrixXd R = task_gram(h.B, h.t);
        SpatialKernel q = SpatialKernel::from(h, family_of(*rd));
        BlockSpectrum spec = build_spectrum(dz, R, q, h.xi);
        BlockInverse inv = invert_and_logdet(spec);
        PiH ph = extract_pi_h(inv);
        for (int l = 0; l < dz.L; ++l) {
            for (int lp = 0; lp < dz.L; ++lp) Pi[l * dz.L + lp] = ph.Pi(l, lp);
            for (std::size_t k = 0; k < inv.r; ++k) {
                H_re[l * inv.r + k] = ph.H(l, static_cast<Eigen::Index>(k)).real();
                H_im[l * inv.r + k] = ph.H(l, static_cast<Eigen::Index>(k)).imag();
            }
        }
    });
}

static double (*problem_fn(const std::string& nm))(int, const double*) {
    double (*f)(int, const double*) = nm == "rosenbrock" ? &rosenbrock
                                      : nm == "ackley"   ? &ackley
                                      : nm == "borehole" ? &borehole
                                      : nm == "elliptic" ? &elliptic_pde
                                                         : nullptr;
    if (!f) throw FastMtgpError("unknown problem " + nm);
    return f;
}

// problem(level, X[i]) at arbitrary points (eval_batch's loop, problems.cpp), X [count][d]
int ref_problem_eval(const char* name, int level, int d, const double* X, std::size_t count, double* out) {
    return guarded([&] {
        double (*f)(int, const double*) = problem_fn(name);
        for (std::size_t i = 0; i < count; ++i) out[i] = f(level, X + i * static_cast<std::size_t>(d));
    });
}

// Benchmark observations as bench.cpp:84-101 makes them: problem(level user + 1, x) + noise *
// rng::normal(seed, 0x401 + user, i) at the design points (internal order, users[l] = user task of l).
int ref_problem_y(const RefDesign* rd, const char* name, const int* users, double noise, std::uint64_t seed,
                  double* y) {
    return guarded([&] {
        LdDesign dz = make_ld(*rd);
        const std::string nm(name);
        double (*f)(int, const double*) = problem_fn(nm);
        for (int l = 0; l < dz.L; ++l)
            for (std::size_t i = 0; i < dz.n[l]; ++i) {
                double v = f(users[l] + 1, dz.point(l, i));
                if (noise > 0.0) v += noise * rng::normal(seed, 0x401 + static_cast<std::uint64_t>(users[l]), i);
                y[dz.offset[l] + i] = v;
            }
    });
}

// ---- gp_core.hpp model ------------------------------------------------------------
void* ref_model_create(const RefDesign* rd, const RefHyper* rh, const double* y) {
    try {
        auto* rm = new RefModel;
        LdDesign dz = make_ld(*rd);
        std::vector<std::vector<double>> yu(dz.L);
        for (int l = 0; l < dz.L; ++l) yu[l].assign(y + dz.offset[l], y + dz.offset[l + 1]);
        rm->model = make_model(std::move(dz), family_of(*rd), make_hyper(*rd, *rh), yu, LossKind::nmll);
        return rm;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

// Replace the kernel hyperparameters (FD probes); invalidates the caches.
int ref_model_set_hyper(void* h, const RefDesign* rd, const RefHyper* rh) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        m.hyper = make_hyper(*rd, *rh);
        m.invalidate();
    });
}

// loss_value (gp_core.cpp:197-227); kind 0 = NMLL, 1 = GCV.
int ref_model_loss(void* h, int kind, double* loss) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        *loss = loss_value(m, kind == 0 ? LossKind::nmll : LossKind::gcv);
    });
}

// After a loss evaluation: logdet, tau (internal order), c (length N), escalations.
int ref_model_state(void* h, double* logdet, double* tau, double* c, int* escalations) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        if (!m.fresh()) throw FastMtgpError("ref_model_state: model not refreshed");
        if (logdet) *logdet = m.inv->logdet;
        if (tau)
            for (int l = 0; l < m.design.L; ++l) tau[l] = m.tau_internal[l];
        if (c) std::memcpy(c, m.c.data(), m.c.size() * sizeof(double));
        if (escalations) *escalations = m.jitter_escalations;
    });
}

int ref_model_posterior_mean(void* h, int task, const double* X, std::size_t count, double* out) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        if (!m.fresh()) m.refresh();
        std::vector<double> xs(X, X + count * m.design.d);
        std::vector<double> r = posterior_mean_batch(m, task, xs, count);
        std::memcpy(out, r.data(), count * sizeof(double));
    });
}

int ref_model_posterior_cov(void* h, int task, const double* x, int task2, const double* xp,
                            double* out) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        if (!m.fresh()) m.refresh();
        *out = posterior_cov(m, task, x, task2, xp);
    });
}

int ref_model_cubature(void* h, double* mu, double* Sigma) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        CubatureResult r = multitask_cubature(m);
        const int L = m.design.L;
        for (int l = 0; l < L; ++l) {
            mu[l] = r.mu[l];
            for (int lp = 0; lp < L; ++lp) Sigma[l * L + lp] = r.Sigma(l, lp);
        }
    });
}

int ref_model_single_cubature(void* h, double* mu, double* var) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        auto r = single_task_cubature(m);
        *mu = r.first;
        *var = r.second;
    });
}

// fit (gp_core.cpp:317-382): iRprop- with central-FD gradients.
int ref_model_fit(void* h, int steps, double* final_loss, double* trace) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        FitReport rep = fit(m, steps, LossKind::nmll);
        *final_loss = rep.final_loss;
        if (trace)
            for (std::size_t i = 0; i < rep.loss_trace.size(); ++i) trace[i] = rep.loss_trace[i];
    });
}

// fit with the reference's own per-step timer (FitReport::step_seconds, gp_core.cpp:340-372): one
// step = the central-FD gradient (2 P_theta loss evaluations) + the iRprop- update + the loss at the
// new theta — the reference's cost of one NLL + gradient.  The CPU baseline of bench.py.
int ref_model_fit_timed(void* h, int steps, double* final_loss, double* trace, double* step_seconds,
                        int* n_params) {
    return guarded([&] {
        auto& m = static_cast<RefModel*>(h)->model;
        FitReport rep = fit(m, steps, LossKind::nmll);
        *final_loss = rep.final_loss;
        for (std::size_t i = 0; i < rep.loss_trace.size(); ++i) {
            if (trace) trace[i] = rep.loss_trace[i];
            if (step_seconds) step_seconds[i] = rep.step_seconds[i];
        }
        if (n_params) {
            // ParamPack::layout (gp_core.cpp:243-304): log gamma, log eta, B, log t, log b (DSI)
            *n_params = 1 + m.design.d + int(m.hyper.B.rows() * m.hyper.B.cols()) + m.design.L +
                        (m.family == KernelFamily::dsi_digital ? 4 : 0);
        }
    });
}

int ref_thread_count() { return thread_count(); }

}  // extern "C"
