// ref_capi.cpp -- TEST INFRASTRUCTURE (oracle/_ref build only).
//
// extern "C" wrapper over the REFERENCE C++ API (the reference sources under
// /root/reference/proj/src compiled in place by oracle/Makefile), so pytest
// can drive the real reference through ctypes with the same argument
// conventions as the oracle port (alsncg_oracle.h).  Used to pin the port and
// to generate tests/golden fixtures; also the "reference" CPU baseline.
#include <cstring>
#include <string>
#include <vector>

#include "alsncg/als.hpp"
#include "alsncg/config.hpp"
#include "alsncg/factors.hpp"
#include "alsncg/harness.hpp"
#include "alsncg/ranking.hpp"
#include "alsncg/linesearch.hpp"
#include "alsncg/ncg.hpp"
#include "alsncg/parallel.hpp"
#include "alsncg/ratings.hpp"
#include "alsncg/rng.hpp"

extern "C" {
#include "alsncg_oracle.h"
}

using namespace alsncg;

namespace {

FlatVector make_flat(int n_f, int n_u, int n_m, const double* u, const double* m) {
  FlatVector v = FlatVector::zeros(n_f, n_u, n_m);
  if (u) std::memcpy(v.user_part.data(), u, sizeof(double) * v.user_part.size());
  if (m) std::memcpy(v.item_part.data(), m, sizeof(double) * v.item_part.size());
  return v;
}

void copy_out(const FlatVector& v, double* u, double* m) {
  std::memcpy(u, v.user_part.data(), sizeof(double) * v.user_part.size());
  std::memcpy(m, v.item_part.data(), sizeof(double) * v.item_part.size());
}

SolverConfig to_config(const orc_config* c) {
  SolverConfig s;
  s.lambda = c->lambda;
  s.n_f = c->n_f;
  s.max_iters = c->max_iters;
  s.tol = c->tol;
  s.seed = c->seed;
  s.alpha0 = c->alpha0;
  s.armijo_c = c->armijo_c;
  s.tau = c->tau;
  s.max_backtracks = c->max_backtracks;
  s.n_blocks = c->n_blocks;
  s.n_workers = c->n_workers;
  s.trace_every = c->trace_every;
  s.snapshot_every = c->snapshot_every;
  s.paper_timing = c->paper_timing != 0;
  return s;
}

void export_result(const SolveResult& r, double* mu, double* mm, orc_trace_rec* trace,
                   int cap, int* len, orc_result* out) {
  std::memcpy(mu, r.model.user_data.data(), sizeof(double) * r.model.user_data.size());
  std::memcpy(mm, r.model.item_data.data(), sizeof(double) * r.model.item_data.size());
  *len = static_cast<int>(r.trace.size());
  for (int k = 0; k < *len && k < cap; ++k) {
    const TraceRecord& t = r.trace[k];
    trace[k] = {t.iter, t.loss, t.grad_norm, t.elapsed_seconds, t.backtracks,
                t.shuffled_columns, t.restarted ? 1 : 0};
  }
  *out = {r.converged ? 1 : 0, r.iterations, r.final_loss, r.final_grad_norm,
          r.restarts, r.fallback_steps, r.fallback_columns};
}

}  // namespace

extern "C" {

// Builds a reference RatingsMatrix from triples; returns an opaque handle or
// null with *status = 1 (range), 2 (non-finite), 3 (duplicate).
void* ref_ratings_from_triples(int n_u, int n_m, std::int64_t nnz, const int* users,
                               const int* items, const double* values, int single,
                               int* status, int* dup_user, int* dup_item) {
  std::vector<Rating> t(static_cast<std::size_t>(nnz));
  for (std::int64_t k = 0; k < nnz; ++k) t[k] = {users[k], items[k], values[k]};
  try {
    auto* r = new RatingsMatrix(RatingsMatrix::from_triples(n_u, n_m, std::move(t), single != 0));
    *status = 0;
    return r;
  } catch (const DuplicateRatingError& e) {
    *status = 3;
    if (dup_user) *dup_user = e.user;
    if (dup_item) *dup_item = e.item;
  } catch (const DataError& e) {
    *status = std::string(e.what()).find("non-finite") != std::string::npos ? 2 : 1;
  }
  return nullptr;
}

void ref_ratings_free(void* h) { delete static_cast<RatingsMatrix*>(h); }

// Exports the CSR/CSC arrays through the public spans (the views are
// contiguous: user_items(0).data() is the base of the index array).
void ref_ratings_export(void* h, std::int64_t* uptr, int* uidx, double* uval,
                        std::int64_t* iptr, int* iidx, double* ival) {
  const RatingsMatrix& r = *static_cast<RatingsMatrix*>(h);
  uptr[0] = 0;
  for (int i = 0; i < r.n_users(); ++i) uptr[i + 1] = uptr[i] + r.user_count(i);
  iptr[0] = 0;
  for (int j = 0; j < r.n_items(); ++j) iptr[j + 1] = iptr[j] + r.item_count(j);
  for (int i = 0; i < r.n_users(); ++i) {
    auto a = r.user_items(i);
    auto b = r.user_values(i);
    std::memcpy(uidx + uptr[i], a.data(), sizeof(int) * a.size());
    std::memcpy(uval + uptr[i], b.data(), sizeof(double) * b.size());
  }
  for (int j = 0; j < r.n_items(); ++j) {
    auto a = r.item_users(j);
    auto b = r.item_values(j);
    std::memcpy(iidx + iptr[j], a.data(), sizeof(int) * a.size());
    std::memcpy(ival + iptr[j], b.data(), sizeof(double) * b.size());
  }
}

void ref_random_init(int n_f, int n_u, int n_m, std::uint64_t seed, double* user, double* item) {
  FactorModel m = random_init(n_f, n_u, n_m, seed);
  std::memcpy(user, m.user_data.data(), sizeof(double) * m.user_data.size());
  std::memcpy(item, m.item_data.data(), sizeof(double) * m.item_data.size());
}

void ref_rng_draws(std::uint64_t seed, int n, std::uint64_t* raw, double* uni, double* nrm) {
  Rng a(seed), b(seed), c(seed);
  for (int k = 0; k < n; ++k) {
    raw[k] = a.next_u64();
    uni[k] = b.uniform();
    nrm[k] = c.normal();
  }
}

double ref_loss(void* h, int n_f, const double* xu, const double* xm, double lambda) {
  const RatingsMatrix& r = *static_cast<RatingsMatrix*>(h);
  return ncg::loss(make_flat(n_f, r.n_users(), r.n_items(), xu, xm), r, lambda);
}

void ref_gradient(void* h, int n_f, const double* xu, const double* xm, double lambda,
                  int n_workers, double* gu, double* gm) {
  const RatingsMatrix& r = *static_cast<RatingsMatrix*>(h);
  copy_out(ncg::gradient(make_flat(n_f, r.n_users(), r.n_items(), xu, xm), r, lambda, n_workers),
           gu, gm);
}

void ref_quartic(void* h, int n_f, const double* xu, const double* xm, const double* pu,
                 const double* pm, double lambda, int n_chunks, int n_workers, double c[5]) {
  const RatingsMatrix& r = *static_cast<RatingsMatrix*>(h);
  const QuarticPoly q = linesearch::quartic_coefficients(
      make_flat(n_f, r.n_users(), r.n_items(), xu, xm),
      make_flat(n_f, r.n_users(), r.n_items(), pu, pm), r, lambda, n_chunks, n_workers);
  for (int n = 0; n < 5; ++n) c[n] = q.c[n];
}

int ref_backtracking(const double c[5], double slope, double alpha0, double cc, double tau,
                     int max_backtracks, double* alpha, int* backtracks) {
  QuarticPoly q;
  for (int n = 0; n < 5; ++n) q.c[n] = c[n];
  const auto res = linesearch::backtracking_search(q, slope, alpha0, cc, tau, max_backtracks);
  *alpha = res.alpha;
  *backtracks = res.backtracks;
  return static_cast<int>(res.status);
}

double ref_beta_bar(int n_f, int n_u, int n_m, const double* gnu, const double* gnm,
                    const double* gpu, const double* gpm, const double* bnu, const double* bnm,
                    const double* bpu, const double* bpm) {
  return ncg::beta_bar(make_flat(n_f, n_u, n_m, gnu, gnm), make_flat(n_f, n_u, n_m, gpu, gpm),
                       make_flat(n_f, n_u, n_m, bnu, bnm), make_flat(n_f, n_u, n_m, bpu, bpm));
}

double ref_dot(int n_f, int n_u, int n_m, const double* xu, const double* xm, const double* yu,
               const double* ym) {
  return dot(make_flat(n_f, n_u, n_m, xu, xm), make_flat(n_f, n_u, n_m, yu, ym));
}

// Half-sweep through parallel_half_sweep (the reference's data-parallel path).
void ref_half_sweep(void* h, int users, int n_f, const double* src, double lambda, int n_blocks,
                    int n_workers, double* out, int* fallback_columns) {
  const RatingsMatrix& r = *static_cast<RatingsMatrix*>(h);
  FactorModel m(n_f, r.n_users(), r.n_items());
  if (users)
    std::memcpy(m.item_data.data(), src, sizeof(double) * m.item_data.size());
  else
    std::memcpy(m.user_data.data(), src, sizeof(double) * m.user_data.size());
  const auto plan = parallel::SweepPlan::build(r, n_blocks);
  auto o = parallel::parallel_half_sweep(
      users ? parallel::HalfSweepKind::kUsers : parallel::HalfSweepKind::kItems, m, r, lambda,
      plan, n_workers);
  std::memcpy(out, o.columns.data(), sizeof(double) * o.columns.size());
  *fallback_columns = o.solve_stats.fallback_columns;
}

void ref_routing_totals(void* h, int n_blocks, std::int64_t* tu, std::int64_t* tm) {
  const auto plan = parallel::SweepPlan::build(*static_cast<RatingsMatrix*>(h), n_blocks);
  *tu = plan.t_u.total_columns();
  *tm = plan.t_m.total_columns();
}

int ref_ncg_solve(void* h, const orc_config* cfg, double* mu, double* mm, orc_trace_rec* trace,
                  int cap, int* len, orc_result* out) {
  try {
    ncg::NcgOverrides ov;
    if (cfg->has_fixed_alpha) ov.fixed_alpha = cfg->fixed_alpha;
    ov.force_beta_zero = cfg->force_beta_zero != 0;
    const SolveResult r =
        ncg::als_ncg_solve(*static_cast<RatingsMatrix*>(h), to_config(cfg), {}, ov);
    export_result(r, mu, mm, trace, cap, len, out);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

int ref_als_solve(void* h, const orc_config* cfg, double* mu, double* mm, orc_trace_rec* trace,
                  int cap, int* len, orc_result* out) {
  try {
    const SolveResult r = als::als_solve(*static_cast<RatingsMatrix*>(h), to_config(cfg));
    export_result(r, mu, mm, trace, cap, len, out);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

}  // extern "C"

// ---- off-path pins: trace CSV (harness.cpp:80-118) and ranking evaluation
// (ranking.cpp:40-109), through the reference's own functions.
extern "C" int ref_write_trace_csv(const char* path, int n, const int* iter, const double* loss,
                                   const double* grad_norm, const double* elapsed, const int* backtracks,
                                   const long long* shuffled) {
  try {
    ConvergenceTrace t;
    for (int i = 0; i < n; ++i) {
      TraceRecord r;
      r.iter = iter[i];
      r.loss = loss[i];
      r.grad_norm = grad_norm[i];
      r.elapsed_seconds = elapsed[i];
      r.backtracks = backtracks[i];
      r.shuffled_columns = shuffled[i];
      t.records.push_back(r);
    }
    harness::write_trace_csv(path, t);
    return 0;
  } catch (...) {
    return 1;
  }
}

extern "C" double ref_mean_ranking_accuracy(int n_f, int n_u, int n_m, const double* uk, const double* mk,
                                            const double* uf, const double* mf, int t, int n_workers) {
  FactorModel a(n_f, n_u, n_m), b(n_f, n_u, n_m);
  std::memcpy(a.user_data.data(), uk, sizeof(double) * a.user_data.size());
  std::memcpy(a.item_data.data(), mk, sizeof(double) * a.item_data.size());
  std::memcpy(b.user_data.data(), uf, sizeof(double) * b.user_data.size());
  std::memcpy(b.item_data.data(), mf, sizeof(double) * b.item_data.size());
  return ranking::mean_ranking_accuracy(a, b, t, n_workers);
}
