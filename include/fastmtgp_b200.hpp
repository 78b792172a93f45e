// C++ adapter over the C ABI (fastmtgp_b200.h): the reference's fast_gram.hpp seam
// (/root/reference/proj/include/fastmtgp/fast_gram.hpp:34-70) with the same argument
// meaning and exception semantics — SchurBreakdown (retryable, drives the noise escalation of
// GpModel::refresh, gp_core.cpp:98-127) vs FastMtgpError (fatal), common.hpp:16-22.
//
// Header-only; link against paper_2603_16014_b200/libfmtgp_b200.so.  Device memory lives in
// the Session; host vectors are owned by the caller (value semantics like the reference).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastmtgp_b200.h"

namespace fastmtgp_b200 {

struct FastMtgpError : std::runtime_error {
    explicit FastMtgpError(const std::string& w) : std::runtime_error(w) {}
};
struct SchurBreakdown : FastMtgpError {
    explicit SchurBreakdown(const std::string& w) : FastMtgpError(w) {}
};

inline void check(int rc) {
    if (rc == FMTGP_OK) return;
    const std::string msg = fmtgp_last_error();
    if (rc == FMTGP_ERR_SCHUR) throw SchurBreakdown(msg);
    throw FastMtgpError(msg);
}

// LdDesign without materialised points (ld_sequences.hpp:56-77), internal (descending) order.
struct Design {
    int kind = 1;  // 0 lattice, 1 digital
    int d = 0;
    std::vector<int> m;
    std::vector<std::uint64_t> g;        // lattice
    std::uint64_t n_max = 0;             // lattice
    std::vector<std::uint64_t> columns;  // digital [d * m_cols]
    int m_cols = 0;
    std::vector<std::uint64_t> shift_bits;  // [L * d]
    int L() const { return int(m.size()); }
    std::size_t N() const {
        std::size_t s = 0;
        for (int v : m) s += std::size_t(1) << v;
        return s;
    }
};

// SpatialKernel (kernels.hpp:53-66) for the periodic families.
struct Spatial {
    double gamma = 1.0;
    std::vector<double> eta;
    int si_alpha = 1;
    double b[4] = {1, 1, 1, 1};
};

// One device-resident design + workspace (one per GPU / dataset).
class Session {
   public:
    explicit Session(const Design& dz, int device = 0, int max_candidates = 1) : dz_(dz) {
        fmtgp_design cd{};
        cd.kind = dz_.kind;
        cd.d = dz_.d;
        cd.L = dz_.L();
        cd.m = dz_.m.data();
        cd.g = dz_.g.empty() ? nullptr : dz_.g.data();
        cd.n_max = dz_.n_max;
        cd.columns = dz_.columns.empty() ? nullptr : dz_.columns.data();
        cd.m_cols = dz_.m_cols;
        cd.shift_bits = dz_.shift_bits.data();
        check(fmtgp_model_create(&cd, device, max_candidates, &h_));
    }
    ~Session() { fmtgp_model_destroy(h_); }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    fmtgp_model_t handle() const { return h_; }
    const Design& design() const { return dz_; }

    // ---- fast_gram.hpp seam (internal task order) ------------------------------------
    // build_spectrum(design, R_internal, spatial, xi_internal)  fast_gram.hpp:34-36
    void build_spectrum(const std::vector<double>& R_internal, const Spatial& q, const std::vector<double>& xi) {
        if (int(R_internal.size()) != dz_.L() * dz_.L()) throw FastMtgpError("build_spectrum: task kernel size mismatch");
        if (int(xi.size()) != dz_.L()) throw FastMtgpError("build_spectrum: xi size mismatch");
        if (int(q.eta.size()) != dz_.d) throw FastMtgpError("product kernel: eta dimension mismatch");
        fmtgp_spatial sp{q.gamma, q.eta.data(), q.si_alpha, {q.b[0], q.b[1], q.b[2], q.b[3]}};
        check(fmtgp_build_spectrum_R(h_, R_internal.data(), &sp, xi.data()));
    }
    // invert_and_logdet  fast_gram.hpp:56-57 (throws SchurBreakdown on a non-positive pivot)
    double invert_and_logdet() {
        double ld = 0.0;
        check(fmtgp_invert_and_logdet(h_, &ld));
        return ld;
    }
    // solve  fast_gram.hpp:59-60
    std::vector<double> solve(const std::vector<double>& y) {
        if (y.size() != dz_.N()) throw FastMtgpError("solve: length mismatch");
        std::vector<double> x(y.size());
        check(fmtgp_solve(h_, y.data(), x.data()));
        return x;
    }
    // gram_matvec  fast_gram.hpp:38-39
    std::vector<double> gram_matvec(const std::vector<double>& y) {
        if (y.size() != dz_.N()) throw FastMtgpError("gram_matvec: length mismatch");
        std::vector<double> out(y.size());
        check(fmtgp_gram_matvec(h_, y.data(), out.data()));
        return out;
    }
    // trace_inverse  fast_gram.hpp:62
    double trace_inverse() {
        double tr = 0.0;
        check(fmtgp_trace_inverse(h_, &tr));
        return tr;
    }
    // extract_pi_h(...).Pi  fast_gram.hpp:64-70
    std::vector<double> extract_pi() {
        std::vector<double> Pi(std::size_t(dz_.L()) * dz_.L());
        check(fmtgp_extract_pi(h_, Pi.data()));
        return Pi;
    }

    // ---- gp_core hot path ------------------------------------------------------------
    void set_y(const std::vector<double>& y) {
        if (y.size() != dz_.N()) throw FastMtgpError("make_model: observation size mismatch");
        check(fmtgp_model_set_y(h_, y.data()));
    }
    fmtgp_result nll(const fmtgp_hyper& h, bool grad = true) {
        fmtgp_result r{};
        check(fmtgp_nll(h_, &h, grad ? 1 : 0, &r));
        return r;
    }
    // loss_value(model, LossKind::gcv)  gp_core.cpp:213-226 (equal n)
    double gcv(const fmtgp_hyper& h) {
        double loss = 0.0;
        check(fmtgp_gcv(h_, &h, &loss, nullptr, nullptr));
        return loss;
    }
    std::vector<double> coefficients() {
        std::vector<double> c(dz_.N());
        check(fmtgp_coefficients(h_, c.data()));
        return c;
    }

   private:
    Design dz_;
    fmtgp_model_t h_ = nullptr;
};

}  // namespace fastmtgp_b200
