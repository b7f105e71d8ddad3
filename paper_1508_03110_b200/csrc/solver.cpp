// solver.cpp -- device-resident drivers.  Branch structure, counters, trace
// and snapshot cadence follow ncg.cpp:138-307 and als.cpp:130-195 line for
// line; every vector lives in HBM, each iteration moves ~10 doubles over PCIe.
#include "solver.h"

#include <cstdio>
#include <cstdlib>

#include <cmath>
#include <cstring>
#include <stdexcept>

#include "host_data.h"

namespace ab2 {

namespace {
// d_scalars slots
constexpr int kSlotQuartic = 0;  // 5
constexpr int kSlotLoss = 5;
constexpr int kSlotGbar = 8;     // 4
constexpr int kSlotDir = 12;
constexpr int kSlotDot = 16;
// d_counters slot accumulating least-norm fallback columns over the solve
constexpr int kCounterFallback = 16;

void validate(const alsncg_config& c) {  // config.cpp:21-34
  auto bad = [](const char* what) {
    throw Error(ALSNCG_EINVAL, std::string("SolverConfig: ") + what);
  };
  if (c.lambda < 0.0) bad("lambda must be >= 0");
  if (c.n_f < 1) bad("n_f must be >= 1");
  if (c.max_iters < 0) bad("max_iters must be >= 0");
  if (c.alpha0 <= 0.0) bad("alpha0 must be > 0");
  if (!(c.armijo_c > 0.0 && c.armijo_c < 1.0)) bad("armijo_c must be in (0,1)");
  if (!(c.tau > 0.0 && c.tau < 1.0)) bad("tau must be in (0,1)");
  if (c.max_backtracks < 0) bad("max_backtracks must be >= 0");
  if (c.n_blocks < 0) bad("n_blocks must be >= 0 (0 = use n_workers)");
  if (c.n_workers < 1) bad("n_workers must be >= 1");
  if (c.trace_every < 1) bad("trace_every must be >= 1");
  if (c.snapshot_every < 0) bad("snapshot_every must be >= 0");
}

int resolved_blocks(const alsncg_config& c) {  // config.hpp:48
  return c.n_blocks > 0 ? c.n_blocks : (c.n_workers > 0 ? c.n_workers : 1);
}
}  // namespace

Solver::Solver(DevRatings* R, const alsncg_config& cfg, bool ncg, alsncg_snapshot_fn snap,
               void* user)
    : R_(R), ctx_(R->ctx), cfg_(cfg), ncg_(ncg), snap_(snap), user_(user) {
  static const bool tsetup = std::getenv("ALSNCG_SETUP_TIMING") != nullptr;
  Watch tw;
  tw.start();
  auto mark = [&](const char* what) {
    if (!tsetup) return;
    ctx_->sync();
    std::fprintf(stderr, "[setup] %-22s %8.2f ms\n", what, tw.seconds() * 1e3);
  };
  validate(cfg_);
  AB2_CUDA(cudaSetDevice(ctx_->device));
  n_f_ = cfg_.n_f;
  if (n_f_ > kMaxRank) throw Error(ALSNCG_EUNSUPPORTED, "n_f exceeds the compiled kernel range");
  ld_ = row_stride(n_f_);
  rows_ = static_cast<int64_t>(R_->n_u) + R_->n_m;
  N_ = rows_ * ld_;
  Nlog_ = rows_ * n_f_;
  const auto tot = R_->routing_totals(resolved_blocks(cfg_));
  sweep_columns_ = tot.first + tot.second;  // ncg.cpp:143-151
  gradient_columns_ = sweep_columns_;
  quartic_columns_ = 2 * tot.second;
  mark("routing");
  const int nbuf = ncg_ ? 10 : 2;
  buf_ = static_cast<double*>(ctx_->alloc(sizeof(double) * std::max<int64_t>(N_, 1) * nbuf));
  double* b = buf_;
  auto take = [&]() {
    double* p = b;
    b += std::max<int64_t>(N_, 1);
    return p;
  };
  x_ = take();
  g_ = take();
  if (ncg_) {
    gbar_ = take();
    p_ = take();
    px_ = take();
    xn_ = take();
    gn_ = take();
    gbn_ = take();
    pn_ = take();
    pxn_ = take();
  } else {
    gbar_ = p_ = px_ = xn_ = gn_ = gbn_ = pn_ = pxn_ = nullptr;
  }
  AB2_CUDA(cudaMemsetAsync(ctx_->d_counters + kCounterFallback, 0, sizeof(unsigned), ctx_->stream));
  use_graphs_ = std::getenv("ALSNCG_GRAPH") != nullptr;
  mark("malloc");

  // x0 = flatten(random_init(seed)) (ncg.cpp:154-155), generated on the
  // device in padded rows (bitwise the host stream, k_vec.cu).
  launch_random_init(ctx_, n_f_, R_->n_u, R_->n_m, cfg_.seed, x_);
  mark("random_init+upload");
  // ncg.cpp:178-181 / als.cpp:150-154
  gradient(x_, g_);
  mark("gradient(x0)");
  launch_vec(ctx_, kDot, N_, g_, g_, nullptr, nullptr, 0.0, nullptr, kSlotDot);
  ctx_->fetch_scalars(kSlotDot + 1);
  grad_norm_ = std::sqrt(ctx_->h_scalars[kSlotDot]) / static_cast<double>(Nlog_);
  append({0, loss(x_), grad_norm_, 0.0, 0, 0, 0});
  mark("loss(x0)");
  if (snap_ && cfg_.snapshot_every > 0) snapshot(0);
  converged_ = cfg_.tol > 0.0 && grad_norm_ < cfg_.tol;
  if (!ncg_) {
    watch_.start();  // als.cpp:157
    started_ = true;
    return;
  }
  if (!converged_ && cfg_.max_iters > 0) {  // ncg.cpp:184-193
    watch_.start();
    apply_als(x_, px_);
    launch_vec(ctx_, kGbarFused, N_, x_, px_, g_, g_, 0.0, gbar_, kSlotGbar);
    launch_vec(ctx_, kDirFused, N_, gbar_, gbar_, g_, nullptr, 0.0, p_, kSlotDir);
    ctx_->fetch_scalars(kSlotDir + 1);
    den_ = ctx_->h_scalars[kSlotGbar + 1];
    slope_ = ctx_->h_scalars[kSlotDir];
    p_is_neg_gbar_ = true;
    restart_pending_ = false;
    step_columns_ = sweep_columns_ + gradient_columns_;
    started_ = true;
    mark("P(x0)+vec");
  }
}

// ncg.cpp:253-257 on the device: gradient at x_{k+1}, P(x_{k+1}), and the
// fused pass (gbar_next, beta parts, ||g_next||^2, g_next.(-gbar_next)).  No
// host decision falls inside this sequence, so with ALSNCG_GRAPH=1 it is
// captured once per rotation of its buffers and replayed as a CUDA graph --
// for launch-bound sizes (config 0: ~20 launches of a few microseconds each).
// Capture starts at the third iteration, when every plan, scratch buffer and
// kernel attribute the sequence needs already exists (nothing may allocate or
// synchronise while the stream is capturing).
void Solver::gradient_als_gbar() {
  auto run = [&]() {
    gradient(xn_, gn_);
    apply_als(xn_, pxn_);
    launch_vec(ctx_, kGbarFused, N_, xn_, pxn_, gn_, g_, 0.0, gbn_, kSlotGbar);
  };
  if (!use_graphs_ || ctx_->world > 1 || ctx_->profiling || k_ < 2) return run();
  const std::array<const void*, 5> key = {xn_, gn_, pxn_, g_, gbn_};
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    const long before = ctx_->launches;
    cudaGraph_t graph = nullptr;
    AB2_CUDA(cudaStreamBeginCapture(ctx_->stream, cudaStreamCaptureModeRelaxed));
    try {
      run();
    } catch (...) {
      cudaStreamEndCapture(ctx_->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    AB2_CUDA(cudaStreamEndCapture(ctx_->stream, &graph));
    IterGraph g;
    g.launches = ctx_->launches - before;
    ctx_->launches = before;
    AB2_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
    it = graphs_.emplace(key, g).first;
  }
  AB2_CUDA(cudaGraphLaunch(it->second.exec, ctx_->stream));
  ctx_->launches += it->second.launches;
}

Solver::~Solver() {
  for (auto& kv : graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (buf_) {
    cudaSetDevice(ctx_->device);
    ctx_->release(buf_);  // stream-ordered: back to the pool after the last use
  }
}

void Solver::append(const alsncg_trace_record& rec) {  // config.cpp:36-44
  if (!trace_.empty()) {
    if (rec.iter <= trace_.back().iter)
      throw Error(ALSNCG_ELOGIC, "ConvergenceTrace: iterations must be strictly increasing");
    if (rec.elapsed_seconds < trace_.back().elapsed_seconds)
      throw Error(ALSNCG_ELOGIC, "ConvergenceTrace: elapsed time must be non-decreasing");
  }
  trace_.push_back(rec);
}

double Solver::loss(const double* x) {
  launch_loss(*R_, n_f_, x, cfg_.lambda, kSlotLoss);
  ctx_->fetch_scalars(kSlotLoss + 1);
  return ctx_->h_scalars[kSlotLoss];
}

void Solver::gradient(const double* x, double* g) {
  launch_gradient(*R_, n_f_, x, cfg_.lambda, g);
  if (ctx_->world > 1) {
    allgather_rows(ctx_, g, R_->ub, ld_);
    std::vector<int> mb(R_->mb);
    for (int& v : mb) v += R_->n_u;
    allgather_rows(ctx_, g, mb, ld_);
  }
}

// P(v) = items(users(v)) (ncg.cpp:165-176, als.cpp:123-128).
void Solver::apply_als(const double* v, double* out) {
  const int64_t item_off = static_cast<int64_t>(R_->n_u) * ld_;
  launch_half_sweep(*R_, 0, n_f_, v + item_off, cfg_.lambda, out, kCounterFallback);
  allgather_rows(ctx_, out, R_->ub, ld_);
  launch_half_sweep(*R_, 1, n_f_, out, cfg_.lambda, out, kCounterFallback);
  if (ctx_->world > 1) {
    std::vector<int> mb(R_->mb);
    for (int& b : mb) b += R_->n_u;
    allgather_rows(ctx_, out, mb, ld_);
  }
}

void Solver::snapshot(int iter) {
  std::vector<double> host(static_cast<size_t>(Nlog_));
  model(host.data());
  snap_(iter, n_f_, R_->n_u, R_->n_m, host.data(), host.data() + static_cast<size_t>(n_f_) * R_->n_u,
        user_);
}

void Solver::model(double* host_packed) {
  double* d_packed = static_cast<double*>(ctx_->scratch(6, sizeof(double) * std::max<int64_t>(Nlog_, 1)));
  launch_unpad_rows(ctx_, rows_, n_f_, x_, d_packed);
  AB2_CUDA(cudaMemcpyAsync(host_packed, d_packed, sizeof(double) * Nlog_, cudaMemcpyDeviceToHost,
                           ctx_->stream));
  ctx_->sync();
}

int Solver::fallback_columns() {
  return static_cast<int>(ctx_->counter_total(kCounterFallback));  // summed over the ranks
}

void Solver::record(int backtracks, bool restarted) {
  // ncg.cpp:287-294: the trace loss runs outside the clock under paper_timing.
  double lv;
  if (cfg_.paper_timing) {
    ctx_->sync();
    watch_.stop();
    lv = loss(x_);
    watch_.start();
  } else {
    lv = loss(x_);
  }
  append({k_, lv, grad_norm_, watch_.seconds(), backtracks, step_columns_, restarted ? 1 : 0});
}

void Solver::ncg_iteration() {
  bool restarted = restart_pending_;  // ncg.cpp:195-205
  restart_pending_ = false;
  double slope = slope_;
  if (slope >= 0.0 && !p_is_neg_gbar_) {
    launch_vec(ctx_, kDirFused, N_, gbar_, gbar_, g_, nullptr, 0.0, p_, kSlotDir);
    ctx_->fetch_scalars(kSlotDir + 1);
    p_is_neg_gbar_ = true;
    restarted = true;
    slope = ctx_->h_scalars[kSlotDir];
  }
  bool pure = false;  // ncg.cpp:207-226
  double alpha = 0.0;
  int backtracks = 0;
  if (cfg_.has_fixed_alpha) {
    alpha = cfg_.fixed_alpha;
  } else if (slope >= 0.0) {
    pure = true;
  } else {
    launch_quartic(*R_, n_f_, x_, p_, cfg_.lambda, kSlotQuartic);
    ctx_->fetch_scalars(kSlotQuartic + 5);
    double c[5];
    std::memcpy(c, ctx_->h_scalars + kSlotQuartic, sizeof c);
    step_columns_ += quartic_columns_;
    double a = 0.0;
    int bt = 0;
    const int st = backtracking_search(c, slope, cfg_.alpha0, cfg_.armijo_c, cfg_.tau,
                                       cfg_.max_backtracks, &a, &bt);
    if (st == 0) {
      alpha = a;
      backtracks = bt;
    } else {
      pure = true;
    }
  }
  if (pure) {  // ncg.cpp:228-241
    std::swap(xn_, px_);
    restarted = true;
    ++fallback_steps_;
  } else if (p_is_neg_gbar_ && alpha == 1.0) {
    std::swap(xn_, px_);
  } else {
    launch_axpby(ctx_, N_, 1.0, x_, alpha, p_, xn_);
  }
  // ncg.cpp:253-255: the gradient at x_{k+1} and P(x_{k+1}) only read
  // x_{k+1}; on one GPU the gradient runs on the side stream beside the two
  // half-sweeps (latency-bound solves leave the SMs room for its gathers).
  // With NCCL exchanges in both, the multi-GPU path keeps them in order.
  // Opt-in (ALSNCG_OVERLAP=1): measured neutral-to-slightly-negative on one
  // B200 at n_f = 25..100 (the gradient's FP64 gathers and the latency-bound
  // solve contend for the same sub-partitions), so the default keeps order.
  static const bool overlap = std::getenv("ALSNCG_OVERLAP") != nullptr;
  if (ctx_->world == 1 && overlap) {
    // enqueued by the first half-sweep batch after its Gram launch (ev_fork
    // recorded there), joined before the next Gram (k_hs_inst.cu run_hs)
    ctx_->side_work = [this]() {
      AB2_CUDA(cudaStreamWaitEvent(ctx_->side, ctx_->ev_fork, 0));
      std::swap(ctx_->stream, ctx_->side);
      gradient(xn_, gn_);
      std::swap(ctx_->stream, ctx_->side);
      AB2_CUDA(cudaEventRecord(ctx_->ev_join, ctx_->side));
    };
    apply_als(xn_, pxn_);
    if (ctx_->side_work) {  // no split half-sweep consumed it (small ranks): run it in order
      AB2_CUDA(cudaEventRecord(ctx_->ev_fork, ctx_->stream));
      auto w = std::move(ctx_->side_work);
      ctx_->side_work = nullptr;
      w();
      ctx_->side_join = true;
    }
    if (ctx_->side_join) {
      AB2_CUDA(cudaStreamWaitEvent(ctx_->stream, ctx_->ev_join, 0));
      ctx_->side_join = false;
    }
    launch_vec(ctx_, kGbarFused, N_, xn_, pxn_, gn_, g_, 0.0, gbn_, kSlotGbar);
  } else {
    gradient_als_gbar();
  }
  step_columns_ += gradient_columns_;
  step_columns_ += sweep_columns_;
  ctx_->fetch_scalars(kSlotGbar + 4);
  const double num = ctx_->h_scalars[kSlotGbar];
  const double den_next = ctx_->h_scalars[kSlotGbar + 1];
  const double gg = ctx_->h_scalars[kSlotGbar + 2];
  const double slope_neg = ctx_->h_scalars[kSlotGbar + 3];
  double beta = 0.0;  // ncg.cpp:259-261, beta_bar ncg.cpp:118-132
  if (!cfg_.force_beta_zero && !pure) {
    if (std::abs(den_) < 1e-30) {
      beta = 0.0;
    } else {
      beta = num / den_;
      if (!std::isfinite(beta)) beta = 0.0;
    }
  }
  double slope_next;
  if (beta == 0.0) {  // ncg.cpp:263-275
    launch_vec(ctx_, kDirFused, N_, gbn_, gbn_, gn_, nullptr, 0.0, pn_, kSlotDir);
    p_is_neg_gbar_ = true;
    slope_next = slope_neg;
  } else {
    launch_vec(ctx_, kDirFused, N_, gbn_, p_, gn_, nullptr, beta, pn_, kSlotDir);
    ctx_->fetch_scalars(kSlotDir + 1);
    p_is_neg_gbar_ = false;
    slope_next = ctx_->h_scalars[kSlotDir];
    if (slope_next >= 0.0) {
      launch_vec(ctx_, kDirFused, N_, gbn_, gbn_, gn_, nullptr, 0.0, pn_, kSlotDir);
      p_is_neg_gbar_ = true;
      restart_pending_ = true;
      slope_next = slope_neg;
    }
  }
  std::swap(x_, xn_);  // ncg.cpp:277-281
  std::swap(g_, gn_);
  std::swap(gbar_, gbn_);
  std::swap(px_, pxn_);
  std::swap(p_, pn_);
  den_ = den_next;
  slope_ = slope_next;
  ++k_;
  if (restarted) ++restarts_;
  grad_norm_ = std::sqrt(gg) / static_cast<double>(Nlog_);  // ncg.cpp:284-286
  converged_ = cfg_.tol > 0.0 && grad_norm_ < cfg_.tol;
  const bool rec = k_ % cfg_.trace_every == 0 || converged_ || k_ == cfg_.max_iters;
  if (rec) {
    record(backtracks, restarted);
    step_columns_ = 0;
  }
  if (snap_ && cfg_.snapshot_every > 0 && k_ % cfg_.snapshot_every == 0) snapshot(k_);
}

void Solver::als_iteration() {  // als.cpp:159-191
  const int64_t item_off = static_cast<int64_t>(R_->n_u) * ld_;
  launch_half_sweep(*R_, 0, n_f_, x_ + item_off, cfg_.lambda, x_, kCounterFallback);
  allgather_rows(ctx_, x_, R_->ub, ld_);
  launch_half_sweep(*R_, 1, n_f_, x_, cfg_.lambda, x_, kCounterFallback);
  if (ctx_->world > 1) {
    std::vector<int> mb(R_->mb);
    for (int& b : mb) b += R_->n_u;
    allgather_rows(ctx_, x_, mb, ld_);
  }
  ++k_;
  if (cfg_.paper_timing) {
    ctx_->sync();
    watch_.stop();
  }
  gradient(x_, g_);
  launch_vec(ctx_, kDot, N_, g_, g_, nullptr, nullptr, 0.0, nullptr, kSlotDot);
  ctx_->fetch_scalars(kSlotDot + 1);
  grad_norm_ = std::sqrt(ctx_->h_scalars[kSlotDot]) / static_cast<double>(Nlog_);
  if (cfg_.paper_timing) watch_.start();
  converged_ = cfg_.tol > 0.0 && grad_norm_ < cfg_.tol;
  if (k_ % cfg_.trace_every == 0 || converged_ || k_ == cfg_.max_iters) {
    double lv;
    if (cfg_.paper_timing) {
      ctx_->sync();
      watch_.stop();
      lv = loss(x_);
      watch_.start();
    } else {
      lv = loss(x_);
    }
    append({k_, lv, grad_norm_, watch_.seconds(), 0, sweep_columns_, 0});
  }
  if (snap_ && cfg_.snapshot_every > 0 && k_ % cfg_.snapshot_every == 0) snapshot(k_);
}

int Solver::step(int n) {
  int ran = 0;
  while (ran < n && started_ && !done()) {
    if (ncg_)
      ncg_iteration();
    else
      als_iteration();
    ++ran;
  }
  return ran;
}

void Solver::finish(alsncg_result* res, double* model_out) {
  ctx_->sync();
  watch_.stop();
  res->converged = converged_ ? 1 : 0;
  res->iterations = k_;
  res->final_grad_norm = grad_norm_;
  res->final_loss = loss(x_);
  res->restarts = restarts_;
  res->fallback_steps = fallback_steps_;
  res->fallback_columns = fallback_columns();
  if (model_out) model(model_out);
}

}  // namespace ab2
