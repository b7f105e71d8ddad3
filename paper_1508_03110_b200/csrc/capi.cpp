// capi.cpp -- extern "C" boundary (include/alsncg_capi.h) over the engine.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "alsncg/harness.hpp"
#include "alsncg/ratings.hpp"
#include "alsncg_capi.h"
#include "engine.h"
#include "host_data.h"
#include "solver.h"

struct alsncg_ctx {
  std::unique_ptr<ab2::Ctx> impl;
};
struct alsncg_ratings {
  alsncg_ctx* ctx;
  std::unique_ptr<ab2::DevRatings> impl;
};
struct alsncg_solver {
  std::unique_ptr<ab2::Solver> impl;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ALSNCG_OK;
  } catch (const ab2::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return ALSNCG_ENOMEM;
  } catch (const alsncg::DuplicateRatingError& e) {
    g_last_error = e.what();
    return ALSNCG_EDUP;
  } catch (const alsncg::DataError& e) {
    g_last_error = e.what();
    return ALSNCG_EDATA;
  } catch (const std::logic_error& e) {
    if (dynamic_cast<const std::invalid_argument*>(&e) == nullptr &&
        dynamic_cast<const std::out_of_range*>(&e) == nullptr) {
      g_last_error = e.what();
      return ALSNCG_ELOGIC;
    }
    g_last_error = e.what();
    return ALSNCG_EINVAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ALSNCG_EINVAL;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw ab2::Error(ALSNCG_EINVAL, what);
}

// Stages a packed host flat vector (or one side of it) into a padded device
// flat vector held in a scratch slot.
double* stage_flat(ab2::DevRatings& R, int slot, int n_f, const double* host_u,
                   const double* host_m) {
  ab2::Ctx* ctx = R.ctx;
  const int ld = ab2::row_stride(n_f);
  const int64_t rows = static_cast<int64_t>(R.n_u) + R.n_m;
  double* dev = static_cast<double*>(ctx->scratch(slot, sizeof(double) * std::max<int64_t>(rows * ld, 1)));
  AB2_CUDA(cudaMemsetAsync(dev, 0, sizeof(double) * rows * ld, ctx->stream));
  double* packed = static_cast<double*>(
      ctx->scratch(6, sizeof(double) * std::max<int64_t>(rows * n_f, 1)));
  const int64_t nu = static_cast<int64_t>(n_f) * R.n_u, nm = static_cast<int64_t>(n_f) * R.n_m;
  if (host_u && nu) {
    AB2_CUDA(cudaMemcpyAsync(packed, host_u, sizeof(double) * nu, cudaMemcpyHostToDevice, ctx->stream));
    ab2::launch_pad_rows(ctx, R.n_u, n_f, packed, dev);
  }
  if (host_m && nm) {
    AB2_CUDA(cudaMemcpyAsync(packed + nu, host_m, sizeof(double) * nm, cudaMemcpyHostToDevice,
                             ctx->stream));
    ab2::launch_pad_rows(ctx, R.n_m, n_f, packed + nu, dev + static_cast<int64_t>(R.n_u) * ld);
  }
  return dev;
}

void unstage_rows(ab2::DevRatings& R, int n_f, const double* dev_rows, int64_t rows, double* host) {
  ab2::Ctx* ctx = R.ctx;
  double* packed = static_cast<double*>(
      ctx->scratch(6, sizeof(double) * std::max<int64_t>((static_cast<int64_t>(R.n_u) + R.n_m) * n_f, 1)));
  if (rows == 0) return;
  ab2::launch_unpad_rows(ctx, rows, n_f, dev_rows, packed);
  AB2_CUDA(cudaMemcpyAsync(host, packed, sizeof(double) * rows * n_f, cudaMemcpyDeviceToHost,
                           ctx->stream));
  ctx->sync();
}

void gather_flat(ab2::DevRatings& R, int n_f, double* dev) {
  ab2::Ctx* ctx = R.ctx;
  if (ctx->world <= 1) return;
  const int ld = ab2::row_stride(n_f);
  ab2::allgather_rows(ctx, dev, R.ub, ld);
  std::vector<int> mb(R.mb);
  for (int& b : mb) b += R.n_u;
  ab2::allgather_rows(ctx, dev, mb, ld);
}

void check_rank(int n_f) {
  need(n_f >= 1, "n_f must be >= 1");
  if (n_f > ab2::kMaxRank) throw ab2::Error(ALSNCG_EUNSUPPORTED, "n_f exceeds the compiled kernel range");
}

int run_solve(alsncg_ratings* r, const alsncg_config* cfg, bool ncg, alsncg_snapshot_fn snap,
              void* user, alsncg_result* res, double* model_out, alsncg_trace_record* trace,
              int trace_cap, int* trace_len) {
  return guarded([&] {
    need(r && cfg && res, "null argument");
    AB2_CUDA(cudaSetDevice(r->impl->ctx->device));
    ab2::Solver s(r->impl.get(), *cfg, ncg, snap, user);
    while (!s.done()) s.step(1 << 20);
    s.finish(res, model_out);
    const auto& t = s.trace();
    if (trace_len) *trace_len = static_cast<int>(t.size());
    for (int k = 0; trace && k < static_cast<int>(t.size()) && k < trace_cap; ++k) trace[k] = t[k];
  });
}

}  // namespace

extern "C" {

const char* alsncg_last_error(void) { return g_last_error.c_str(); }
int alsncg_abi_version(void) { return 1; }
int alsncg_row_stride(int n_f) { return ab2::row_stride(n_f); }
int alsncg_max_rank(void) { return ab2::kMaxRank; }

int alsncg_csr_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
                     const double* values, int single, int64_t* uptr, int* uidx, double* uval,
                     int64_t* iptr, int* iidx, double* ival, int* dup_user, int* dup_item) {
  std::string err;
  const int st = ab2::csr_build(n_u, n_m, nnz, users, items, values, single != 0, uptr, uidx, uval,
                                iptr, iidx, ival, dup_user, dup_item, &err);
  if (st) g_last_error = err;
  return st;
}

int alsncg_random_init(int n_f, int n_u, int n_m, uint64_t seed, double* user, double* item) {
  if (n_f < 1) {
    g_last_error = "random_init: n_f must be >= 1";
    return ALSNCG_EINVAL;
  }
  ab2::random_init(n_f, n_u, n_m, seed, user, item);
  return ALSNCG_OK;
}

int alsncg_synth_generate(int n_u, int n_m, int64_t nnz, int min_per_user, uint64_t seed,
                          int* users, int* items, double* values) {
  std::string err;
  const int st = ab2::synth_generate(n_u, n_m, nnz, min_per_user, seed, users, items, values, &err);
  if (st) g_last_error = err;
  return st;
}

int alsncg_backtracking_search(const double c[5], double slope, double alpha0, double armijo_c,
                               double tau, int max_backtracks, double* alpha, int* backtracks) {
  if (alpha0 <= 0.0) {
    g_last_error = "backtracking_search: alpha0 must be > 0";
    return -ALSNCG_EINVAL;
  }
  if (!(armijo_c > 0.0 && armijo_c < 1.0) || !(tau > 0.0 && tau < 1.0)) {
    g_last_error = "backtracking_search: c and tau must be in (0,1)";
    return -ALSNCG_EINVAL;
  }
  return ab2::backtracking_search(c, slope, alpha0, armijo_c, tau, max_backtracks, alpha, backtracks);
}

int alsncg_ctx_create(int device, alsncg_ctx** out) {
  return guarded([&] {
    need(out, "null argument");
    auto c = std::make_unique<alsncg_ctx>();
    c->impl = std::make_unique<ab2::Ctx>(device);
    *out = c.release();
  });
}

int alsncg_nccl_unique_id(unsigned char id[128]) {
  return guarded([&] {
    ncclUniqueId u;
    AB2_NCCL(ab2::nccl().GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
  });
}

int alsncg_ctx_create_dist(int device, int rank, int world, const unsigned char id[128],
                           alsncg_ctx** out) {
  return guarded([&] {
    need(out && world >= 1 && rank >= 0 && rank < world, "bad rank/world");
    auto c = std::make_unique<alsncg_ctx>();
    c->impl = std::make_unique<ab2::Ctx>(device);
    c->impl->rank = rank;
    c->impl->world = world;
    if (world > 1) {
      ncclUniqueId u;
      std::memcpy(&u, id, 128);
      AB2_NCCL(ab2::nccl().CommInitRank(&c->impl->comm, world, u, rank));
    }
    *out = c.release();
  });
}

int alsncg_mean_ranking_accuracy(alsncg_ctx* ctx, int n_f, int n_u, int n_m, const double* user_k,
                                 const double* item_k, const double* user_final, const double* item_final,
                                 int t, double* out) {
  return guarded([&] {
    need(ctx && out && n_f >= 1 && n_u >= 0 && n_m >= 0, "mean_ranking_accuracy: bad arguments");
    if (n_u == 0) throw std::invalid_argument("mean_ranking_accuracy: no users");  // ranking.cpp:95
    if (t < 1 || t > n_m) throw std::invalid_argument("ranking_accuracy: t out of range");  // ranking.cpp:63
    need(user_k && item_k && user_final && item_final, "null argument");
    ab2::Ctx* c = ctx->impl.get();
    AB2_CUDA(cudaSetDevice(c->device));
    const size_t nu = static_cast<size_t>(n_f) * n_u, nm = static_cast<size_t>(n_f) * n_m;
    double* d = static_cast<double*>(c->alloc(sizeof(double) * (2 * nu + 2 * nm + n_u)));
    AB2_CUDA(cudaMemcpyAsync(d, user_k, sizeof(double) * nu, cudaMemcpyHostToDevice, c->stream));
    AB2_CUDA(cudaMemcpyAsync(d + nu, item_k, sizeof(double) * nm, cudaMemcpyHostToDevice, c->stream));
    AB2_CUDA(cudaMemcpyAsync(d + nu + nm, user_final, sizeof(double) * nu, cudaMemcpyHostToDevice, c->stream));
    AB2_CUDA(cudaMemcpyAsync(d + 2 * nu + nm, item_final, sizeof(double) * nm, cudaMemcpyHostToDevice, c->stream));
    double* dq = d + 2 * nu + 2 * nm;
    ab2::launch_mean_ranking(c, n_f, n_u, n_m, d, d + nu, d + nu + nm, d + 2 * nu + nm, t, dq);
    std::vector<double> q(n_u);
    AB2_CUDA(cudaMemcpyAsync(q.data(), dq, sizeof(double) * n_u, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    c->release(d);
    double sum = 0.0;  // ranking.cpp:104-107: sequential in user order
    for (double v : q) sum += v;
    *out = sum / static_cast<double>(n_u);
  });
}

int alsncg_write_trace_csv(const char* path, const alsncg_trace_record* recs, int n) {
  return guarded([&] {
    need(path && (recs || n == 0) && n >= 0, "null argument");
    alsncg::ConvergenceTrace t;
    for (int i = 0; i < n; ++i) {
      alsncg::TraceRecord r;
      r.iter = recs[i].iter;
      r.loss = recs[i].loss;
      r.grad_norm = recs[i].grad_norm;
      r.elapsed_seconds = recs[i].elapsed_seconds;
      r.backtracks = recs[i].backtracks;
      r.shuffled_columns = recs[i].shuffled_columns;
      r.restarted = recs[i].restarted != 0;
      t.records.push_back(r);
    }
    alsncg::harness::write_trace_csv(path, t);
  });
}

int alsncg_read_trace_csv(const char* path, alsncg_trace_record* recs, int cap, int* n) {
  return guarded([&] {
    need(path && n && (recs || cap == 0), "null argument");
    const alsncg::ConvergenceTrace t = alsncg::harness::read_trace_csv(path);
    *n = static_cast<int>(t.records.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      const alsncg::TraceRecord& r = t.records[i];
      recs[i] = {r.iter, r.loss, r.grad_norm, r.elapsed_seconds, r.backtracks, r.shuffled_columns,
                 r.restarted ? 1 : 0};
    }
  });
}

int alsncg_loopgroup_create(int world, alsncg_loopgroup** out) {
  return guarded([&] {
    need(out && world >= 1, "bad world");
    *out = reinterpret_cast<alsncg_loopgroup*>(new ab2::LoopGroup(world));
  });
}

int alsncg_loopgroup_destroy(alsncg_loopgroup* g) {
  return guarded([&] { delete reinterpret_cast<ab2::LoopGroup*>(g); });
}

int alsncg_ctx_create_loopback(int device, int rank, alsncg_loopgroup* group, alsncg_ctx** out) {
  return guarded([&] {
    auto* G = reinterpret_cast<ab2::LoopGroup*>(group);
    need(out && G && rank >= 0 && rank < G->world, "bad rank/group");
    auto c = std::make_unique<alsncg_ctx>();
    c->impl = std::make_unique<ab2::Ctx>(device);
    c->impl->rank = rank;
    c->impl->world = G->world;
    c->impl->loop = G;
    G->ranks[rank] = c->impl.get();
    *out = c.release();
  });
}

int alsncg_ctx_destroy(alsncg_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int alsncg_ctx_info(alsncg_ctx* ctx, int* device, int* rank, int* world) {
  return guarded([&] {
    need(ctx, "null context");
    if (device) *device = ctx->impl->device;
    if (rank) *rank = ctx->impl->rank;
    if (world) *world = ctx->impl->world;
  });
}

void* alsncg_ctx_stream(alsncg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->impl->stream) : nullptr; }

int alsncg_ctx_synchronize(alsncg_ctx* ctx) {
  return guarded([&] { ctx->impl->sync(); });
}

int alsncg_ctx_set_profiling(alsncg_ctx* ctx, int on) {
  return guarded([&] {
    ctx->impl->collect_stats();
    ctx->impl->profiling = on != 0;
  });
}

int alsncg_ctx_reset_stats(alsncg_ctx* ctx) {
  return guarded([&] {
    ctx->impl->collect_stats();
    ctx->impl->stats.clear();
    ctx->impl->launches = 0;
  });
}

int alsncg_ctx_stat_count(alsncg_ctx* ctx) {
  int n = -1;
  guarded([&] {
    ctx->impl->collect_stats();
    n = static_cast<int>(ctx->impl->stats.size());
  });
  return n;
}

int alsncg_ctx_stat(alsncg_ctx* ctx, int k, const char** name, int64_t* launches, double* ms) {
  return guarded([&] {
    ctx->impl->collect_stats();
    need(k >= 0 && k < static_cast<int>(ctx->impl->stats.size()), "stat index");
    const auto& s = ctx->impl->stats[k];
    if (name) *name = s.name.c_str();
    if (launches) *launches = s.launches;
    if (ms) *ms = s.ms;
  });
}

int64_t alsncg_ctx_launches(alsncg_ctx* ctx) { return ctx ? ctx->impl->launches : -1; }

int alsncg_ratings_upload(alsncg_ctx* ctx, int n_u, int n_m, int64_t nnz, const int64_t* uptr,
                          const int* uidx, const double* uval, const int64_t* iptr, const int* iidx,
                          const double* ival, alsncg_ratings** out) {
  return guarded([&] {
    need(ctx && out && uptr && iptr, "null argument");
    auto r = std::make_unique<alsncg_ratings>();
    r->ctx = ctx;
    r->impl.reset(ab2::upload_ratings(ctx->impl.get(), n_u, n_m, nnz, uptr, uidx, uval, iptr, iidx, ival));
    *out = r.release();
  });
}

int alsncg_ratings_download(alsncg_ratings* r, int64_t* uptr, int* uidx, double* uval,
                            int64_t* iptr, int* iidx, double* ival) {
  return guarded([&] {
    need(r, "null ratings");
    ab2::DevRatings& R = *r->impl;
    need(R.ctx->world == 1, "download needs a single-GPU context");
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    const cudaStream_t s = R.ctx->stream;
    AB2_CUDA(cudaMemcpyAsync(uptr, R.users.ptr, sizeof(int64_t) * (R.n_u + 1), cudaMemcpyDeviceToHost, s));
    AB2_CUDA(cudaMemcpyAsync(iptr, R.items.ptr, sizeof(int64_t) * (R.n_m + 1), cudaMemcpyDeviceToHost, s));
    if (R.nnz) {
      AB2_CUDA(cudaMemcpyAsync(uidx, R.users.idx, sizeof(int) * R.nnz, cudaMemcpyDeviceToHost, s));
      AB2_CUDA(cudaMemcpyAsync(uval, R.users.val, sizeof(double) * R.nnz, cudaMemcpyDeviceToHost, s));
      AB2_CUDA(cudaMemcpyAsync(iidx, R.items.idx, sizeof(int) * R.nnz, cudaMemcpyDeviceToHost, s));
      AB2_CUDA(cudaMemcpyAsync(ival, R.items.val, sizeof(double) * R.nnz, cudaMemcpyDeviceToHost, s));
    }
    R.ctx->sync();
  });
}

int alsncg_ratings_shard(alsncg_ratings* r, int* u0, int* u1, int* m0, int* m1) {
  return guarded([&] {
    const ab2::DevRatings& R = *r->impl;
    *u0 = R.users.row0;
    *u1 = R.users.row0 + R.users.nrows;
    *m0 = R.items.row0;
    *m1 = R.items.row0 + R.items.nrows;
  });
}

int alsncg_partition_rows(int n_rows, const int64_t* ptr, int world, int align, int* bounds) {
  return guarded([&] {
    if (n_rows < 0 || world < 1 || align < 1 || ptr == nullptr || bounds == nullptr)
      throw ab2::Error(ALSNCG_EINVAL, "alsncg_partition_rows: bad arguments");
    const std::vector<int> b = ab2::partition_rows(n_rows, ptr, world, align);
    std::copy(b.begin(), b.end(), bounds);
  });
}

int alsncg_ratings_free(alsncg_ratings* r) {
  return guarded([&] {
    if (r) AB2_CUDA(cudaSetDevice(r->impl->ctx->device));
    delete r;
  });
}

// ------------------------------------------------------ host-buffer API --
int alsncg_loss(alsncg_ratings* r, int n_f, const double* x, double lambda, double* out) {
  return guarded([&] {
    need(r && x && out, "null argument");
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    double* d = stage_flat(R, 7, n_f, x, x + static_cast<int64_t>(n_f) * R.n_u);
    ab2::launch_loss(R, n_f, d, lambda, 0);
    R.ctx->fetch_scalars(1);
    *out = R.ctx->h_scalars[0];
  });
}

int alsncg_gradient(alsncg_ratings* r, int n_f, const double* x, double lambda, double* g) {
  return guarded([&] {
    need(r && x && g, "null argument");
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    double* d = stage_flat(R, 7, n_f, x, x + static_cast<int64_t>(n_f) * R.n_u);
    double* dg = stage_flat(R, 8, n_f, nullptr, nullptr);
    ab2::launch_gradient(R, n_f, d, lambda, dg);
    gather_flat(R, n_f, dg);
    unstage_rows(R, n_f, dg, static_cast<int64_t>(R.n_u) + R.n_m, g);
  });
}

int alsncg_quartic(alsncg_ratings* r, int n_f, const double* x, const double* p, double lambda,
                   double c[5]) {
  return guarded([&] {
    need(r && x && p && c, "null argument");
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    const int64_t nu = static_cast<int64_t>(n_f) * R.n_u;
    double* dx = stage_flat(R, 7, n_f, x, x + nu);
    double* dp = stage_flat(R, 8, n_f, p, p + nu);
    ab2::launch_quartic(R, n_f, dx, dp, lambda, 0);
    R.ctx->fetch_scalars(5);
    std::memcpy(c, R.ctx->h_scalars, sizeof(double) * 5);
  });
}

int alsncg_half_sweep(alsncg_ratings* r, int kind, int n_f, const double* src, double lambda,
                      double* out, int* fallback_columns) {
  return guarded([&] {
    need(r && src && out && (kind == 0 || kind == 1), "bad argument");
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    ab2::Ctx* ctx = R.ctx;
    AB2_CUDA(cudaSetDevice(ctx->device));
    const int ld = ab2::row_stride(n_f);
    double* d = stage_flat(R, 7, n_f, kind == 0 ? nullptr : src, kind == 0 ? src : nullptr);
    const int64_t item_off = static_cast<int64_t>(R.n_u) * ld;
    AB2_CUDA(cudaMemsetAsync(ctx->d_counters + 17, 0, sizeof(unsigned), ctx->stream));
    ab2::launch_half_sweep(R, kind, n_f, kind == 0 ? d + item_off : d, lambda, d, 17);
    if (kind == 0) {
      ab2::allgather_rows(ctx, d, R.ub, ld);
      unstage_rows(R, n_f, d, R.n_u, out);
    } else {
      std::vector<int> mb(R.mb);
      for (int& b : mb) b += R.n_u;
      ab2::allgather_rows(ctx, d, mb, ld);
      unstage_rows(R, n_f, d + item_off, R.n_m, out);
    }
    if (fallback_columns) *fallback_columns = static_cast<int>(ctx->counter_total(17));
  });
}

int alsncg_als_sweep(alsncg_ratings* r, int n_f, const double* x, double lambda, double* out,
                     int* fallback_columns) {
  return guarded([&] {
    need(r && x && out, "null argument");
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    ab2::Ctx* ctx = R.ctx;
    AB2_CUDA(cudaSetDevice(ctx->device));
    const int ld = ab2::row_stride(n_f);
    const int64_t item_off = static_cast<int64_t>(R.n_u) * ld;
    double* d = stage_flat(R, 7, n_f, nullptr, x + static_cast<int64_t>(n_f) * R.n_u);
    AB2_CUDA(cudaMemsetAsync(ctx->d_counters + 17, 0, sizeof(unsigned), ctx->stream));
    ab2::launch_half_sweep(R, 0, n_f, d + item_off, lambda, d, 17);
    ab2::allgather_rows(ctx, d, R.ub, ld);
    ab2::launch_half_sweep(R, 1, n_f, d, lambda, d, 17);
    gather_flat(R, n_f, d);
    unstage_rows(R, n_f, d, static_cast<int64_t>(R.n_u) + R.n_m, out);
    if (fallback_columns) *fallback_columns = static_cast<int>(ctx->counter_total(17));
  });
}

// ---------------------------------------------------- device-buffer API --
int alsncg_dev_loss(alsncg_ratings* r, int n_f, const double* d_x, double lambda, double* out) {
  return guarded([&] {
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    ab2::launch_loss(R, n_f, d_x, lambda, 0);
    R.ctx->fetch_scalars(1);
    *out = R.ctx->h_scalars[0];
  });
}

int alsncg_dev_gradient(alsncg_ratings* r, int n_f, const double* d_x, double lambda, double* d_g) {
  return guarded([&] {
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    ab2::launch_gradient(R, n_f, d_x, lambda, d_g);
    gather_flat(R, n_f, d_g);
  });
}

int alsncg_dev_quartic(alsncg_ratings* r, int n_f, const double* d_x, const double* d_p,
                       double lambda, double c[5]) {
  return guarded([&] {
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    AB2_CUDA(cudaSetDevice(R.ctx->device));
    ab2::launch_quartic(R, n_f, d_x, d_p, lambda, 0);
    R.ctx->fetch_scalars(5);
    std::memcpy(c, R.ctx->h_scalars, sizeof(double) * 5);
  });
}

int alsncg_dev_half_sweep(alsncg_ratings* r, int kind, int n_f, const double* d_src, double lambda,
                          double* d_out, int* fallback_columns) {
  return guarded([&] {
    need(kind == 0 || kind == 1, "kind must be 0 or 1");
    check_rank(n_f);
    ab2::DevRatings& R = *r->impl;
    ab2::Ctx* ctx = R.ctx;
    AB2_CUDA(cudaSetDevice(ctx->device));
    const int ld = ab2::row_stride(n_f);
    const int64_t item_off = static_cast<int64_t>(R.n_u) * ld;
    AB2_CUDA(cudaMemsetAsync(ctx->d_counters + 17, 0, sizeof(unsigned), ctx->stream));
    // d_src / d_out are flat vectors; the half-sweep reads the other side.
    ab2::launch_half_sweep(R, kind, n_f, kind == 0 ? d_src + item_off : d_src, lambda, d_out, 17);
    if (kind == 0) {
      ab2::allgather_rows(ctx, d_out, R.ub, ld);
    } else {
      std::vector<int> mb(R.mb);
      for (int& b : mb) b += R.n_u;
      ab2::allgather_rows(ctx, d_out, mb, ld);
    }
    if (fallback_columns) *fallback_columns = static_cast<int>(ctx->counter_total(17));
  });
}

int alsncg_dev_dot(alsncg_ctx* ctx, int64_t n, const double* d_x, const double* d_y, double* out) {
  return guarded([&] {
    ab2::launch_vec(ctx->impl.get(), ab2::kDot, n, d_x, d_y, nullptr, nullptr, 0.0, nullptr, 0);
    ctx->impl->fetch_scalars(1);
    *out = ctx->impl->h_scalars[0];
  });
}

int alsncg_dev_dot_seq(alsncg_ctx* ctx, int64_t n, const double* d_x, const double* d_y, double* out) {
  return guarded([&] {
    ab2::launch_seq_dots(ctx->impl.get(), n, d_x, d_y, nullptr, nullptr, 0);
    ctx->impl->fetch_scalars(1);
    *out = ctx->impl->h_scalars[0];
  });
}

int alsncg_dev_beta_bar_seq(alsncg_ctx* ctx, int64_t n, const double* d_gn, const double* d_gp,
                            const double* d_bn, const double* d_bp, double* out) {
  return guarded([&] {
    // num = sum bn*(gn - gp), den = sum bp*gp, each in index order (ncg.cpp:123-131)
    ab2::launch_seq_dots(ctx->impl.get(), n, d_bn, d_gn, d_gp, d_bp, 0);
    ctx->impl->fetch_scalars(2);
    const double num = ctx->impl->h_scalars[0], den = ctx->impl->h_scalars[1];
    double beta = 0.0;
    if (!(std::abs(den) < 1e-30)) {
      beta = num / den;
      if (!std::isfinite(beta)) beta = 0.0;
    }
    *out = beta;
  });
}

int alsncg_dev_axpby(alsncg_ctx* ctx, int64_t n, double a, const double* d_x, double b,
                     const double* d_y, double* d_out) {
  return guarded([&] { ab2::launch_axpby(ctx->impl.get(), n, a, d_x, b, d_y, d_out); });
}

int alsncg_dev_beta_bar(alsncg_ctx* ctx, int64_t n, const double* d_gn, const double* d_gp,
                        const double* d_bn, const double* d_bp, double* out) {
  return guarded([&] {
    ab2::launch_vec(ctx->impl.get(), ab2::kBetaParts, n, d_bn, d_gn, d_gp, d_bp, 0.0, nullptr, 0);
    ctx->impl->fetch_scalars(2);
    const double num = ctx->impl->h_scalars[0], den = ctx->impl->h_scalars[1];
    double beta = 0.0;  // ncg.cpp:123-131
    if (!(std::abs(den) < 1e-30)) {
      beta = num / den;
      if (!std::isfinite(beta)) beta = 0.0;
    }
    *out = beta;
  });
}

int alsncg_dev_malloc(alsncg_ctx* ctx, size_t bytes, void** ptr) {
  return guarded([&] {
    AB2_CUDA(cudaSetDevice(ctx->impl->device));
    AB2_CUDA(cudaMalloc(ptr, std::max<size_t>(bytes, 16)));
  });
}

int alsncg_dev_free(alsncg_ctx* ctx, void* ptr) {
  return guarded([&] {
    AB2_CUDA(cudaSetDevice(ctx->impl->device));
    ctx->impl->sync();
    AB2_CUDA(cudaFree(ptr));
  });
}

int alsncg_memcpy_h2d(alsncg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    AB2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->impl->stream));
    ctx->impl->sync();
  });
}

int alsncg_memcpy_d2h(alsncg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    AB2_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->impl->stream));
    ctx->impl->sync();
  });
}

int alsncg_flat_h2d(alsncg_ctx* ctx, int n_f, int n_u, int n_m, const double* host, double* d_dev) {
  return guarded([&] {
    ab2::Ctx* c = ctx->impl.get();
    const int64_t rows = static_cast<int64_t>(n_u) + n_m;
    double* packed = static_cast<double*>(c->scratch(6, sizeof(double) * std::max<int64_t>(rows * n_f, 1)));
    AB2_CUDA(cudaMemcpyAsync(packed, host, sizeof(double) * rows * n_f, cudaMemcpyHostToDevice, c->stream));
    ab2::launch_pad_rows(c, rows, n_f, packed, d_dev);
    c->sync();
  });
}

int alsncg_flat_d2h(alsncg_ctx* ctx, int n_f, int n_u, int n_m, const double* d_dev, double* host) {
  return guarded([&] {
    ab2::Ctx* c = ctx->impl.get();
    const int64_t rows = static_cast<int64_t>(n_u) + n_m;
    double* packed = static_cast<double*>(c->scratch(6, sizeof(double) * std::max<int64_t>(rows * n_f, 1)));
    ab2::launch_unpad_rows(c, rows, n_f, d_dev, packed);
    AB2_CUDA(cudaMemcpyAsync(host, packed, sizeof(double) * rows * n_f, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  });
}

// -------------------------------------------------------------- drivers --
int alsncg_ncg_solve(alsncg_ratings* r, const alsncg_config* cfg, alsncg_snapshot_fn snap, void* user,
                     alsncg_result* res, double* model_out, alsncg_trace_record* trace,
                     int trace_cap, int* trace_len) {
  return run_solve(r, cfg, true, snap, user, res, model_out, trace, trace_cap, trace_len);
}

int alsncg_als_solve(alsncg_ratings* r, const alsncg_config* cfg, alsncg_snapshot_fn snap, void* user,
                     alsncg_result* res, double* model_out, alsncg_trace_record* trace,
                     int trace_cap, int* trace_len) {
  return run_solve(r, cfg, false, snap, user, res, model_out, trace, trace_cap, trace_len);
}

int alsncg_solver_create(alsncg_ratings* r, const alsncg_config* cfg, alsncg_solver** out) {
  return guarded([&] {
    need(r && cfg && out, "null argument");
    AB2_CUDA(cudaSetDevice(r->impl->ctx->device));
    auto s = std::make_unique<alsncg_solver>();
    s->impl = std::make_unique<ab2::Solver>(r->impl.get(), *cfg, true, nullptr, nullptr);
    *out = s.release();
  });
}

int alsncg_solver_step(alsncg_solver* s, int n, int* ran) {
  return guarded([&] {
    const int k = s->impl->step(n);
    if (ran) *ran = k;
  });
}

int alsncg_solver_state(alsncg_solver* s, int* iterations, int* converged, double* grad_norm,
                        int* restarts, int* fallback_steps, int* fallback_columns) {
  return guarded([&] {
    ab2::Solver& v = *s->impl;
    if (iterations) *iterations = v.iterations();
    if (converged) *converged = v.converged() ? 1 : 0;
    if (grad_norm) *grad_norm = v.grad_norm();
    if (restarts) *restarts = v.restarts();
    if (fallback_steps) *fallback_steps = v.fallback_steps();
    if (fallback_columns) *fallback_columns = v.fallback_columns();
  });
}

int alsncg_solver_trace(alsncg_solver* s, alsncg_trace_record* trace, int cap, int* len) {
  return guarded([&] {
    const auto& t = s->impl->trace();
    if (len) *len = static_cast<int>(t.size());
    for (int k = 0; trace && k < static_cast<int>(t.size()) && k < cap; ++k) trace[k] = t[k];
  });
}

int alsncg_solver_model(alsncg_solver* s, double* model_out) {
  return guarded([&] { s->impl->model(model_out); });
}

int alsncg_solver_destroy(alsncg_solver* s) {
  return guarded([&] { delete s; });
}

}  // extern "C"
