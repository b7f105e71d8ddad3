// solver.h -- device-resident ALS-NCG / ALS drivers (ncg.cpp:138-307,
// als.cpp:130-195).  Host control flow mirrors the reference branch for
// branch; only scalars cross PCIe per iteration.
#pragma once

#include <array>
#include <chrono>
#include <map>
#include <vector>

#include "engine.h"

namespace ab2 {

struct Watch {  // src/stopwatch.hpp:23-45 semantics
  using clock = std::chrono::steady_clock;
  clock::time_point t0;
  double total = 0.0;
  bool running = false;
  void start() {
    if (!running) {
      t0 = clock::now();
      running = true;
    }
  }
  void stop() {
    if (running) {
      total += std::chrono::duration<double>(clock::now() - t0).count();
      running = false;
    }
  }
  double seconds() const {
    return running ? total + std::chrono::duration<double>(clock::now() - t0).count() : total;
  }
};

class Solver {
 public:
  Solver(DevRatings* R, const alsncg_config& cfg, bool ncg, alsncg_snapshot_fn snap, void* user);
  ~Solver();
  // Runs up to n outer iterations; returns how many ran.
  int step(int n);
  bool done() const { return converged_ || k_ >= cfg_.max_iters; }
  void finish(alsncg_result* res, double* model_out);
  void model(double* host_packed);
  const std::vector<alsncg_trace_record>& trace() const { return trace_; }
  int iterations() const { return k_; }
  bool converged() const { return converged_; }
  double grad_norm() const { return grad_norm_; }
  int restarts() const { return restarts_; }
  int fallback_steps() const { return fallback_steps_; }
  int fallback_columns();

 private:
  void ncg_iteration();
  void als_iteration();
  double loss(const double* x);
  void gradient(const double* x, double* g);
  void apply_als(const double* x, double* out);
  void record(int backtracks, bool restarted);
  void snapshot(int iter);
  void append(const alsncg_trace_record& rec);

  DevRatings* R_;
  Ctx* ctx_;
  alsncg_config cfg_;
  bool ncg_;
  alsncg_snapshot_fn snap_;
  void* user_;
  int n_f_, ld_;
  int64_t rows_, N_, Nlog_;
  double* buf_ = nullptr;
  double *x_, *g_, *gbar_, *p_, *px_, *xn_, *gn_, *gbn_, *pn_, *pxn_;
  int k_ = 0;
  bool converged_ = false;
  bool started_ = false;
  double grad_norm_ = 0.0;
  double slope_ = 0.0;  // g.p for the current p
  double den_ = 0.0;    // gbar.g for the current pair (beta denominator)
  bool p_is_neg_gbar_ = true;
  bool restart_pending_ = false;
  // CUDA graphs of the launch sequence between two host decisions (gradient,
  // P(x), fused gbar pass), one per rotation of the buffers it touches.
  struct IterGraph {
    cudaGraphExec_t exec = nullptr;
    long launches = 0;
  };
  std::map<std::array<const void*, 5>, IterGraph> graphs_;
  bool use_graphs_ = false;
  void gradient_als_gbar();
  int restarts_ = 0, fallback_steps_ = 0;
  int64_t sweep_columns_ = 0, gradient_columns_ = 0, quartic_columns_ = 0, step_columns_ = 0;
  Watch watch_;
  std::vector<alsncg_trace_record> trace_;
};

}  // namespace ab2
