// Unequal sample sizes: stage-wise LDL^H "fold" of the transformed Gram (Algorithm 1,
// PAPER.md:390-419, in factored form).  Declarations only; the
// implementation (unequal_impl.inc) is compiled inside model.cu.
#pragma once

#include "../../include/fastmtgp_b200.h"

struct fmtgp_model;

namespace fmtgp::unequal {
struct Plan;
Plan* create(fmtgp_model* M);
void destroy(Plan* P);
void nll(Plan* P, fmtgp_model* M, const fmtgp_hyper* h, bool grad, fmtgp_result* out);
void invert(Plan* P, fmtgp_model* M, double* logdet);
void apply_inverse(Plan* P, fmtgp_model* M, const void* in_slots, void* out_slots);
void apply_gram(Plan* P, fmtgp_model* M, const void* in_slots, void* out_slots);
void extract_pi(Plan* P, fmtgp_model* M, double* Pi);
void extract_h(Plan* P, fmtgp_model* M, double* Hre, double* Him);
double trace_inverse(Plan* P, fmtgp_model* M);
void coefficients(Plan* P, fmtgp_model* M, double* d_out);
void posterior_var(Plan* P, fmtgp_model* M, int task, const double* X, int64_t count, double* out);
void posterior_cov(Plan* P, fmtgp_model* M, int task, const double* X, int task2, const double* Xp, int64_t count,
                   double* out);
void cubature_terms(Plan* P, fmtgp_model* M, double* Pi, double* etc);
}  // namespace fmtgp::unequal
