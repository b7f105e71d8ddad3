// alsncg/ncg.hpp -- drop-in declaration of the objective, gradient and the
// ALS-NCG driver (/root/reference/proj/include/alsncg/ncg.hpp:23-65).  The
// driver runs device-resident (paper_1508_03110_b200/csrc/solver.cpp).
#pragma once

#include <optional>

#include "alsncg/config.hpp"
#include "alsncg/factors.hpp"
#include "alsncg/ratings.hpp"

namespace alsncg::ncg {

double loss(const FlatVector& x, const RatingsMatrix& ratings, double lambda);

/// n_workers is accepted for API parity; rows are independent, so the
/// device result does not depend on it.
FlatVector gradient(const FlatVector& x, const RatingsMatrix& ratings, double lambda,
                    int n_workers = 1);

/// gbar_next'(g_next - g_prev) / (gbar_prev' g_prev); 0 on |den| < 1e-30 or
/// a non-finite quotient.
double beta_bar(const FlatVector& g_next, const FlatVector& g_prev,
                const FlatVector& gbar_next, const FlatVector& gbar_prev);

double normalized_grad_norm(const FlatVector& g);

struct NcgOverrides {
  std::optional<double> fixed_alpha;
  bool force_beta_zero = false;
};

SolveResult als_ncg_solve(const RatingsMatrix& ratings, const SolverConfig& config,
                          const SnapshotSink& snapshot = {},
                          const NcgOverrides& overrides = {});

}  // namespace alsncg::ncg
