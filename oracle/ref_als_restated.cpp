// ref_als_restated.cpp -- TEST INFRASTRUCTURE (oracle/_ref build only).
//
// The reference's als.cpp cannot compile here: it includes <Eigen/Dense>
// (als.cpp:17) and Eigen3 is absent.  This unit
// supplies the alsncg::als API declared in the reference header
// /root/reference/proj/include/alsncg/als.hpp so the other reference sources
// (ncg.cpp, parallel.cpp, linesearch.cpp, ...) link unmodified.  The column
// solve delegates to the oracle's Eigen-free restatement
// (orc_solve_normal_column in alsncg_oracle.c: same Gram/rhs order and shift
// as als.cpp:49-61, unblocked Cholesky for Eigen::LLT, pseudo-inverse for the
// COD fallback); the drivers restate als.cpp:85-195.
#include "alsncg/als.hpp"

#include "alsncg/ncg.hpp"
#include "alsncg/parallel.hpp"
#include "stopwatch.hpp"

extern "C" {
#include "alsncg_oracle.h"
}

namespace alsncg::als {

void solve_normal_column(const int* idx, const double* vals, int count,
                         const double* const* cols, int n_f, double lambda,
                         double* out, SolveStats& stats) {
  int fb = 0;
  orc_solve_normal_column(idx, vals, count, cols, n_f, lambda, out, &fb);
  stats.fallback_columns += fb;
}

namespace {
std::vector<double> update_side(const FactorModel& model, const RatingsMatrix& ratings,
                                double lambda, SolveStats* stats, bool users) {
  const int n_f = model.n_f;
  const int n_dest = users ? ratings.n_users() : ratings.n_items();
  const int n_src = users ? ratings.n_items() : ratings.n_users();
  std::vector<double> out(static_cast<std::size_t>(n_f) * n_dest, 0.0);
  std::vector<const double*> cols(static_cast<std::size_t>(n_src));
  for (int j = 0; j < n_src; ++j) cols[j] = users ? model.item_col(j) : model.user_col(j);
  SolveStats local;
  for (int c = 0; c < n_dest; ++c) {  // als.cpp:93-99 / :112-118
    const auto idx = users ? ratings.user_items(c) : ratings.item_users(c);
    const auto val = users ? ratings.user_values(c) : ratings.item_values(c);
    if (idx.empty()) continue;
    solve_normal_column(idx.data(), val.data(), static_cast<int>(idx.size()), cols.data(),
                        n_f, lambda, out.data() + static_cast<std::size_t>(c) * n_f, local);
  }
  if (stats) stats->fallback_columns += local.fallback_columns;
  return out;
}
}  // namespace

std::vector<double> update_users(const FactorModel& model, const RatingsMatrix& ratings,
                                 double lambda, SolveStats* stats) {
  return update_side(model, ratings, lambda, stats, true);
}

std::vector<double> update_items(const FactorModel& model, const RatingsMatrix& ratings,
                                 double lambda, SolveStats* stats) {
  return update_side(model, ratings, lambda, stats, false);
}

FlatVector als_sweep(const FlatVector& x, const RatingsMatrix& ratings, double lambda) {
  FactorModel model = unflatten(x);  // als.cpp:123-128
  model.user_data = update_users(model, ratings, lambda);
  model.item_data = update_items(model, ratings, lambda);
  return flatten(model);
}

SolveResult als_solve(const RatingsMatrix& ratings, const SolverConfig& config,
                      const SnapshotSink& snapshot) {
  config.validate();  // als.cpp:130-195
  const auto plan = parallel::SweepPlan::build(ratings, config.resolved_blocks());
  const std::int64_t sweep_columns = plan.t_m.total_columns() + plan.t_u.total_columns();
  SolveResult result;
  result.model = random_init(config.n_f, ratings.n_users(), ratings.n_items(), config.seed);
  Stopwatch watch;
  auto instrumented = [&](auto&& fn) {
    if (config.paper_timing) watch.stop();
    fn();
    if (config.paper_timing) watch.start();
  };
  FlatVector x = flatten(result.model);
  double grad_norm =
      ncg::normalized_grad_norm(ncg::gradient(x, ratings, config.lambda, config.n_workers));
  result.trace.append({0, ncg::loss(x, ratings, config.lambda), grad_norm, 0.0, 0, 0, false});
  if (snapshot && config.snapshot_every > 0) snapshot(result.model, 0);
  bool converged = config.tol > 0.0 && grad_norm < config.tol;
  int k = 0;
  watch.start();
  while (!converged && k < config.max_iters) {
    auto users = parallel::parallel_half_sweep(parallel::HalfSweepKind::kUsers, result.model,
                                               ratings, config.lambda, plan, config.n_workers);
    result.model.user_data = std::move(users.columns);
    auto items = parallel::parallel_half_sweep(parallel::HalfSweepKind::kItems, result.model,
                                               ratings, config.lambda, plan, config.n_workers);
    result.model.item_data = std::move(items.columns);
    result.fallback_columns +=
        users.solve_stats.fallback_columns + items.solve_stats.fallback_columns;
    ++k;
    instrumented([&] {
      x = flatten(result.model);
      grad_norm =
          ncg::normalized_grad_norm(ncg::gradient(x, ratings, config.lambda, config.n_workers));
    });
    converged = config.tol > 0.0 && grad_norm < config.tol;
    if (k % config.trace_every == 0 || converged || k == config.max_iters) {
      double loss_value = 0.0;
      instrumented([&] { loss_value = ncg::loss(x, ratings, config.lambda); });
      result.trace.append({k, loss_value, grad_norm, watch.seconds(), 0, sweep_columns, false});
    }
    if (snapshot && config.snapshot_every > 0 && k % config.snapshot_every == 0)
      snapshot(result.model, k);
  }
  watch.stop();
  result.converged = converged;
  result.iterations = k;
  result.final_grad_norm = grad_norm;
  result.final_loss = ncg::loss(flatten(result.model), ratings, config.lambda);
  return result;
}

}  // namespace alsncg::als
