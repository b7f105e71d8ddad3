// cxx_api.cpp -- the reference's C++ solver API (include/alsncg/*.hpp)
// implemented over the C-ABI (include/alsncg_capi.h).  Host-only logic
// (validation, traces, routing tables, RNG, snapshots) is plain C++; every
// numerical hot-path call goes to the sm_100a kernels through the ABI on a
// process-wide default context (device ALSNCG_DEVICE, default 0).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <fstream>
#include <map>
#include <mutex>
#include <numbers>
#include <numeric>
#include <stdexcept>
#include <thread>

#include "alsncg/als.hpp"
#include "alsncg/config.hpp"
#include "alsncg/factors.hpp"
#include "alsncg/harness.hpp"
#include "alsncg/linesearch.hpp"
#include "alsncg/ncg.hpp"
#include "alsncg/parallel.hpp"
#include "alsncg/ranking.hpp"
#include "alsncg/ratings.hpp"
#include "alsncg/rng.hpp"
#include "alsncg/snapshot.hpp"
#include "alsncg_capi.h"

namespace alsncg {

namespace {

// C-ABI status -> the reference's exception types.
void check(int st) {
  if (st == ALSNCG_OK) return;
  const std::string msg = alsncg_last_error();
  switch (st) {
    case ALSNCG_EINVAL:
      throw std::invalid_argument(msg);
    case ALSNCG_EDATA:
      throw DataError(msg);
    case ALSNCG_ELOGIC:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error("alsncg: " + msg);
  }
}

alsncg_ctx* default_ctx() {
  static std::once_flag once;
  static alsncg_ctx* ctx = nullptr;
  std::call_once(once, [] {
    const char* env = std::getenv("ALSNCG_DEVICE");
    check(alsncg_ctx_create(env ? std::atoi(env) : 0, &ctx));
  });
  return ctx;
}

// RAII device buffer on the default context.
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { check(alsncg_dev_malloc(default_ctx(), bytes, &p)); }
  DevBuf(const void* host, size_t bytes) : DevBuf(bytes) {
    if (bytes) check(alsncg_memcpy_h2d(default_ctx(), p, host, bytes));
  }
  ~DevBuf() { alsncg_dev_free(default_ctx(), p); }
  double* d() const { return static_cast<double*>(p); }
};

std::vector<double> concat(const FlatVector& x) {
  std::vector<double> v(x.user_part);
  v.insert(v.end(), x.item_part.begin(), x.item_part.end());
  return v;
}

FlatVector split(std::vector<double> v, int n_f, int n_u, int n_m) {
  FlatVector x;
  x.n_f = n_f;
  x.n_u = n_u;
  x.n_m = n_m;
  const auto mid = v.begin() + static_cast<std::ptrdiff_t>(n_f) * n_u;
  x.user_part.assign(v.begin(), mid);
  x.item_part.assign(mid, v.end());
  return x;
}

std::mutex g_upload_mu;

}  // namespace

// ------------------------------------------------------------- ratings --
struct RatingsDevice {
  static alsncg_ratings* get(const RatingsMatrix& r) {
    std::lock_guard<std::mutex> lock(g_upload_mu);
    if (!r.device_) {
      alsncg_ratings* h = nullptr;
      check(alsncg_ratings_upload(default_ctx(), r.n_u_, r.n_m_, r.nnz_, r.uptr_.data(), r.uidx_.data(),
                                  r.uval_.data(), r.iptr_.data(), r.iidx_.data(), r.ival_.data(), &h));
      r.device_ = std::shared_ptr<void>(h, [](void* p) { alsncg_ratings_free(static_cast<alsncg_ratings*>(p)); });
    }
    return static_cast<alsncg_ratings*>(r.device_.get());
  }
};

DuplicateRatingError::DuplicateRatingError(int user_in, int item_in)
    : DataError("duplicate rating for user " + std::to_string(user_in) + ", item " +
                std::to_string(item_in)),
      user(user_in),
      item(item_in) {}

RatingsMatrix RatingsMatrix::from_triples(int n_users, int n_items, std::vector<Rating> triples,
                                          bool single_precision_storage) {
  if (n_users < 0 || n_items < 0) throw DataError("negative matrix dimensions");
  const std::int64_t nnz = static_cast<std::int64_t>(triples.size());
  std::vector<int> u(triples.size()), it(triples.size());
  std::vector<double> v(triples.size());
  for (std::size_t k = 0; k < triples.size(); ++k) {
    u[k] = triples[k].user;
    it[k] = triples[k].item;
    v[k] = triples[k].value;
  }
  RatingsMatrix r;
  r.n_u_ = n_users;
  r.n_m_ = n_items;
  r.nnz_ = nnz;
  r.single_ = single_precision_storage;
  r.uptr_.assign(static_cast<std::size_t>(n_users) + 1, 0);
  r.iptr_.assign(static_cast<std::size_t>(n_items) + 1, 0);
  r.uidx_.resize(triples.size());
  r.iidx_.resize(triples.size());
  r.uval_.resize(triples.size());
  r.ival_.resize(triples.size());
  int du = -1, di = -1;
  const int st = alsncg_csr_build(n_users, n_items, nnz, u.data(), it.data(), v.data(),
                                  single_precision_storage ? 1 : 0, r.uptr_.data(), r.uidx_.data(),
                                  r.uval_.data(), r.iptr_.data(), r.iidx_.data(), r.ival_.data(), &du, &di);
  if (st == ALSNCG_EDUP) throw DuplicateRatingError(du, di);
  check(st);
  return r;
}

std::vector<Rating> RatingsMatrix::to_triples() const {
  std::vector<Rating> out;
  out.reserve(static_cast<std::size_t>(nnz_));
  for (int i = 0; i < n_u_; ++i)
    for (std::int64_t t = uptr_[i]; t < uptr_[i + 1]; ++t) out.push_back({i, uidx_[t], uval_[t]});
  return out;
}

void RatingsMatrix::check_consistent() const {  // ratings.cpp:103-132 semantics
  auto fail = [](const std::string& w) { throw std::logic_error("RatingsMatrix: " + w); };
  if (uptr_.size() != static_cast<std::size_t>(n_u_) + 1 || iptr_.size() != static_cast<std::size_t>(n_m_) + 1)
    fail("pointer size");
  if (uptr_.back() != nnz_ || iptr_.back() != nnz_) fail("nnz mismatch");
  for (int i = 0; i < n_u_; ++i)
    for (std::int64_t t = uptr_[i]; t < uptr_[i + 1]; ++t) {
      if (t > uptr_[i] && uidx_[t] <= uidx_[t - 1]) fail("user adjacency not sorted");
      const int j = uidx_[t];
      if (j < 0 || j >= n_m_) fail("item index range");
      const auto users = item_users(j);
      auto pos = std::lower_bound(users.begin(), users.end(), i);
      if (pos == users.end() || *pos != i) fail("entry missing from item view");
      if (item_values(j)[pos - users.begin()] != uval_[t]) fail("value mismatch between views");
    }
  for (int j = 0; j < n_m_; ++j)
    for (std::int64_t t = iptr_[j] + 1; t < iptr_[j + 1]; ++t)
      if (iidx_[t] <= iidx_[t - 1]) fail("item adjacency not sorted");
}

// ------------------------------------------------------------- factors --
FactorModel random_init(int n_f, int n_u, int n_m, std::uint64_t seed) {
  if (n_f < 1) throw std::invalid_argument("random_init: n_f must be >= 1");
  FactorModel m(n_f, n_u, n_m);
  check(alsncg_random_init(n_f, n_u, n_m, seed, m.user_data.data(), m.item_data.data()));
  return m;
}

FlatVector FlatVector::zeros(int n_f, int n_u, int n_m) {
  FlatVector v;
  v.n_f = n_f;
  v.n_u = n_u;
  v.n_m = n_m;
  v.user_part.assign(static_cast<std::size_t>(n_f) * n_u, 0.0);
  v.item_part.assign(static_cast<std::size_t>(n_f) * n_m, 0.0);
  return v;
}

double FlatVector::at(std::int64_t k) const {
  const std::int64_t split_at = static_cast<std::int64_t>(n_f) * n_u;
  if (k < 0 || k >= size()) throw std::out_of_range("FlatVector::at");
  return k < split_at ? user_part[static_cast<std::size_t>(k)] : item_part[static_cast<std::size_t>(k - split_at)];
}

void FlatVector::set(std::int64_t k, double v) {
  const std::int64_t split_at = static_cast<std::int64_t>(n_f) * n_u;
  if (k < 0 || k >= size()) throw std::out_of_range("FlatVector::set");
  (k < split_at ? user_part[static_cast<std::size_t>(k)] : item_part[static_cast<std::size_t>(k - split_at)]) = v;
}

FlatVector flatten(const FactorModel& model) {
  FlatVector v;
  v.n_f = model.n_f;
  v.n_u = model.n_u;
  v.n_m = model.n_m;
  v.user_part = model.user_data;
  v.item_part = model.item_data;
  return v;
}

FactorModel unflatten(const FlatVector& x) {
  FactorModel m;
  m.n_f = x.n_f;
  m.n_u = x.n_u;
  m.n_m = x.n_m;
  m.user_data = x.user_part;
  m.item_data = x.item_part;
  return m;
}

FlatVector axpby(double a, const FlatVector& x, double b, const FlatVector& y) {
  if (!x.same_shape(y)) throw std::invalid_argument("axpby: shape mismatch");
  const std::vector<double> hx = concat(x), hy = concat(y);
  const size_t bytes = hx.size() * sizeof(double);
  DevBuf dx(hx.data(), bytes), dy(hy.data(), bytes), dz(bytes);
  check(alsncg_dev_axpby(default_ctx(), static_cast<std::int64_t>(hx.size()), a, dx.d(), b, dy.d(), dz.d()));
  std::vector<double> out(hx.size());
  if (bytes) check(alsncg_memcpy_d2h(default_ctx(), out.data(), dz.p, bytes));
  return split(std::move(out), x.n_f, x.n_u, x.n_m);
}

double dot(const FlatVector& x, const FlatVector& y) {
  if (!x.same_shape(y)) throw std::invalid_argument("dot: shape mismatch");
  const std::vector<double> hx = concat(x), hy = concat(y);
  const size_t bytes = hx.size() * sizeof(double);
  DevBuf dx(hx.data(), bytes), dy(hy.data(), bytes);
  double out = 0.0;
  check(alsncg_dev_dot_seq(default_ctx(), static_cast<std::int64_t>(hx.size()), dx.d(), dy.d(), &out));
  return out;
}

double norm(const FlatVector& x) { return std::sqrt(dot(x, x)); }

// -------------------------------------------------------------- config --
void SolverConfig::validate() const {  // config.cpp:21-34
  auto bad = [](const char* what) { throw std::invalid_argument(std::string("SolverConfig: ") + what); };
  if (lambda < 0.0) bad("lambda must be >= 0");
  if (n_f < 1) bad("n_f must be >= 1");
  if (max_iters < 0) bad("max_iters must be >= 0");
  if (alpha0 <= 0.0) bad("alpha0 must be > 0");
  if (!(armijo_c > 0.0 && armijo_c < 1.0)) bad("armijo_c must be in (0,1)");
  if (!(tau > 0.0 && tau < 1.0)) bad("tau must be in (0,1)");
  if (max_backtracks < 0) bad("max_backtracks must be >= 0");
  if (n_blocks < 0) bad("n_blocks must be >= 0 (0 = use n_workers)");
  if (n_workers < 1) bad("n_workers must be >= 1");
  if (trace_every < 1) bad("trace_every must be >= 1");
  if (snapshot_every < 0) bad("snapshot_every must be >= 0");
}

void ConvergenceTrace::append(const TraceRecord& rec) {  // config.cpp:36-44
  if (!records.empty()) {
    if (rec.iter <= records.back().iter)
      throw std::logic_error("ConvergenceTrace: iterations must be strictly increasing");
    if (rec.elapsed_seconds < records.back().elapsed_seconds)
      throw std::logic_error("ConvergenceTrace: elapsed time must be non-decreasing");
  }
  records.push_back(rec);
}

// ----------------------------------------------------------------- rng --
std::uint64_t Rng::uniform_below(std::uint64_t n) {  // rng.cpp:25-34 semantics
  if (n == 0) throw std::invalid_argument("uniform_below: n must be positive");
  const std::uint64_t mx = ~std::uint64_t{0};
  const std::uint64_t limit = mx - mx % n;
  std::uint64_t v;
  do {
    v = gen_();
  } while (v >= limit);
  return v % n;
}

double Rng::normal() {  // rng.cpp:36-49 semantics
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double mag = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * std::numbers::pi * u2;
  spare_ = mag * std::sin(ang);
  has_spare_ = true;
  return mag * std::cos(ang);
}

int sample_cumulative(const std::vector<double>& cumulative, double u) {
  if (cumulative.empty() || cumulative.back() <= 0.0)
    throw std::invalid_argument("sample_cumulative: empty or zero-mass distribution");
  auto pos = std::upper_bound(cumulative.begin(), cumulative.end(), u * cumulative.back());
  if (pos == cumulative.end()) --pos;
  return static_cast<int>(pos - cumulative.begin());
}

// ------------------------------------------------------------ snapshot --
void save_model(const std::string& path, const FactorModel& model, std::int64_t iter, std::uint64_t seed) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw DataError("cannot write " + path);
  out.write("ALSNCG01", 8);
  const std::int64_t hdr[5] = {model.n_f, model.n_u, model.n_m, iter, static_cast<std::int64_t>(seed)};
  out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  out.write(reinterpret_cast<const char*>(model.user_data.data()),
            static_cast<std::streamsize>(model.user_data.size() * sizeof(double)));
  out.write(reinterpret_cast<const char*>(model.item_data.data()),
            static_cast<std::streamsize>(model.item_data.size() * sizeof(double)));
  if (!out) throw DataError("failed writing " + path);
}

LoadedModel load_model(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open " + path);
  char magic[8] = {};
  in.read(magic, 8);
  if (!in || std::memcmp(magic, "ALSNCG01", 8) != 0) throw DataError(path + ": not a model snapshot");
  std::int64_t hdr[5] = {};
  in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  if (!in || hdr[0] < 1 || hdr[1] < 0 || hdr[2] < 0 || hdr[0] > (1 << 20) || hdr[1] > (1LL << 32) ||
      hdr[2] > (1LL << 32))
    throw DataError(path + ": malformed snapshot header");
  LoadedModel l;
  l.meta.n_f = static_cast<int>(hdr[0]);
  l.meta.n_u = static_cast<int>(hdr[1]);
  l.meta.n_m = static_cast<int>(hdr[2]);
  l.meta.iter = hdr[3];
  l.meta.seed = static_cast<std::uint64_t>(hdr[4]);
  l.model = FactorModel(l.meta.n_f, l.meta.n_u, l.meta.n_m);
  in.read(reinterpret_cast<char*>(l.model.user_data.data()),
          static_cast<std::streamsize>(l.model.user_data.size() * sizeof(double)));
  in.read(reinterpret_cast<char*>(l.model.item_data.data()),
          static_cast<std::streamsize>(l.model.item_data.size() * sizeof(double)));
  if (!in) throw DataError(path + ": truncated snapshot");
  return l;
}

// ------------------------------------------------------------- ranking --
namespace ranking {

RankingVector rank_items(const FactorModel& model, int user) {
  if (user < 0 || user >= model.n_u) throw std::out_of_range("rank_items: user index");
  const double* u = model.user_col(user);
  std::vector<double> sc(static_cast<size_t>(model.n_m));
  for (int j = 0; j < model.n_m; ++j) {
    const double* m = model.item_col(j);
    double d = 0.0;
    for (int k = 0; k < model.n_f; ++k) d += u[k] * m[k];  // sequential, no FMA (-ffp-contract=off)
    sc[j] = d;
  }
  RankingVector order(static_cast<size_t>(model.n_m));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return sc[a] != sc[b] ? sc[a] > sc[b] : a < b; });
  return order;
}

double ranking_accuracy(const RankingVector& p1, const RankingVector& p2, int t) {
  const int n = static_cast<int>(p1.size());
  auto is_perm = [n](const RankingVector& p) {
    if (static_cast<int>(p.size()) != n) throw std::invalid_argument("ranking_accuracy: size mismatch");
    std::vector<char> seen(static_cast<size_t>(n), 0);
    for (int v : p) {
      if (v < 0 || v >= n || seen[v]) throw std::invalid_argument("ranking_accuracy: not a permutation");
      seen[v] = 1;
    }
  };
  is_perm(p1);
  is_perm(p2);
  if (t < 1 || t > n) throw std::invalid_argument("ranking_accuracy: t out of range");
  // closed form of the swap walk: rank2(p1[r]) minus the earlier picks that
  // p2 ranks ahead of it (the same count the reference's working-copy walk makes)
  std::vector<int> pos(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) pos[p2[r]] = r;
  std::int64_t swaps = 0;
  for (int r = 0; r < t; ++r) {
    int ahead = 0;
    for (int q = 0; q < r; ++q) ahead += pos[p1[q]] < pos[p1[r]] ? 1 : 0;
    swaps += pos[p1[r]] - ahead;
  }
  const std::int64_t smax = static_cast<std::int64_t>(t) * (2 * static_cast<std::int64_t>(n) - t - 1) / 2;
  if (smax == 0) return 1.0;
  return 1.0 - static_cast<double>(swaps) / static_cast<double>(smax);
}

double mean_ranking_accuracy(const FactorModel& model_at_k, const FactorModel& model_final, int t, int n_workers) {
  (void)n_workers;
  if (model_at_k.n_f != model_final.n_f || model_at_k.n_u != model_final.n_u || model_at_k.n_m != model_final.n_m)
    throw std::invalid_argument("mean_ranking_accuracy: model shape mismatch");
  double out = 0.0;
  check(alsncg_mean_ranking_accuracy(default_ctx(), model_at_k.n_f, model_at_k.n_u, model_at_k.n_m,
                                     model_at_k.user_data.data(), model_at_k.item_data.data(),
                                     model_final.user_data.data(), model_final.item_data.data(), t, &out));
  return out;
}

}  // namespace ranking

// ----------------------------------------------------------- trace CSV --
// harness.cpp:80-127 (file format and error behaviour of the reference).
namespace harness {
namespace {

std::string fmt17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

template <typename T>
T parse_field(const std::string& f, const std::string& path, const char* what) {
  T v{};
  const auto r = std::from_chars(f.data(), f.data() + f.size(), v);
  if (r.ec != std::errc() || r.ptr != f.data() + f.size())
    throw DataError(path + ": bad " + what + " field '" + f + "'");
  return v;
}

}  // namespace

void write_trace_csv(const std::string& path, const ConvergenceTrace& trace) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw DataError("cannot write " + path);
  out << "iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns\n";
  for (const TraceRecord& t : trace.records)
    out << t.iter << ',' << fmt17(t.loss) << ',' << fmt17(t.grad_norm) << ',' << fmt17(t.elapsed_seconds)
        << ',' << t.backtracks << ',' << t.shuffled_columns << '\n';
  if (!out) throw DataError("failed writing " + path);
}

ConvergenceTrace read_trace_csv(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open " + path);
  ConvergenceTrace trace;
  std::string line;
  bool header = true;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (header) {
      header = false;
      continue;
    }
    std::vector<std::string> f;
    for (size_t b = 0;;) {
      const size_t c = line.find(',', b);
      f.push_back(line.substr(b, c == std::string::npos ? std::string::npos : c - b));
      if (c == std::string::npos) break;
      b = c + 1;
    }
    if (f.size() != 6) throw DataError(path + ": expected 6 trace columns");
    TraceRecord t;
    t.iter = static_cast<int>(parse_field<std::int64_t>(f[0], path, "integer"));
    t.loss = parse_field<double>(f[1], path, "numeric");
    t.grad_norm = parse_field<double>(f[2], path, "numeric");
    t.elapsed_seconds = parse_field<double>(f[3], path, "numeric");
    t.backtracks = static_cast<int>(parse_field<std::int64_t>(f[4], path, "integer"));
    t.shuffled_columns = parse_field<std::int64_t>(f[5], path, "integer");
    trace.append(t);
  }
  if (trace.empty()) throw DataError(path + ": empty trace");
  return trace;
}

double mean_iteration_seconds(const ConvergenceTrace& trace) {
  if (trace.empty()) throw DataError("mean_iteration_seconds: empty trace");
  const TraceRecord& a = trace.records.front();
  const TraceRecord& b = trace.records.back();
  if (a.iter == b.iter) return 0.0;
  return (b.elapsed_seconds - a.elapsed_seconds) / static_cast<double>(b.iter - a.iter);
}

}  // namespace harness

// ------------------------------------------------------------- drivers --
namespace {

alsncg_config to_c(const SolverConfig& c, const ncg::NcgOverrides* ov) {
  alsncg_config o{};
  o.lambda = c.lambda;
  o.n_f = c.n_f;
  o.max_iters = c.max_iters;
  o.tol = c.tol;
  o.seed = c.seed;
  o.alpha0 = c.alpha0;
  o.armijo_c = c.armijo_c;
  o.tau = c.tau;
  o.max_backtracks = c.max_backtracks;
  o.n_blocks = c.n_blocks;
  o.n_workers = c.n_workers;
  o.trace_every = c.trace_every;
  o.snapshot_every = c.snapshot_every;
  o.paper_timing = c.paper_timing ? 1 : 0;
  if (ov) {
    o.has_fixed_alpha = ov->fixed_alpha.has_value() ? 1 : 0;
    o.fixed_alpha = ov->fixed_alpha.value_or(0.0);
    o.force_beta_zero = ov->force_beta_zero ? 1 : 0;
  }
  return o;
}

struct SinkCtx {
  const SnapshotSink* sink;
  std::exception_ptr err;
};

void sink_tramp(int iter, int n_f, int n_u, int n_m, const double* u, const double* m, void* user) {
  auto* s = static_cast<SinkCtx*>(user);
  if (s->err) return;
  try {
    FactorModel fm(n_f, n_u, n_m);
    std::copy(u, u + fm.user_data.size(), fm.user_data.begin());
    std::copy(m, m + fm.item_data.size(), fm.item_data.begin());
    (*s->sink)(fm, iter);
  } catch (...) {
    s->err = std::current_exception();
  }
}

SolveResult run(bool ncg_mode, const RatingsMatrix& ratings, const SolverConfig& config,
                const SnapshotSink& snapshot, const ncg::NcgOverrides* ov) {
  config.validate();
  const alsncg_config c = to_c(config, ov);
  SolveResult r;
  r.model = FactorModel(config.n_f, ratings.n_users(), ratings.n_items());
  std::vector<double> model(r.model.user_data.size() + r.model.item_data.size());
  std::vector<alsncg_trace_record> tr(static_cast<std::size_t>(config.max_iters) + 2);
  int len = 0;
  alsncg_result res{};
  SinkCtx sctx{&snapshot, nullptr};
  auto fn = ncg_mode ? alsncg_ncg_solve : alsncg_als_solve;
  check(fn(RatingsDevice::get(ratings), &c, snapshot ? sink_tramp : nullptr, &sctx, &res, model.data(),
           tr.data(), static_cast<int>(tr.size()), &len));
  if (sctx.err) std::rethrow_exception(sctx.err);
  std::copy(model.begin(), model.begin() + static_cast<std::ptrdiff_t>(r.model.user_data.size()),
            r.model.user_data.begin());
  std::copy(model.begin() + static_cast<std::ptrdiff_t>(r.model.user_data.size()), model.end(),
            r.model.item_data.begin());
  for (int k = 0; k < len && k < static_cast<int>(tr.size()); ++k)
    r.trace.records.push_back({tr[k].iter, tr[k].loss, tr[k].grad_norm, tr[k].elapsed_seconds,
                               tr[k].backtracks, tr[k].shuffled_columns, tr[k].restarted != 0});
  r.converged = res.converged != 0;
  r.iterations = res.iterations;
  r.final_loss = res.final_loss;
  r.final_grad_norm = res.final_grad_norm;
  r.restarts = res.restarts;
  r.fallback_steps = res.fallback_steps;
  r.fallback_columns = res.fallback_columns;
  return r;
}

void check_shape(const FlatVector& x, const RatingsMatrix& ratings) {
  if (x.n_u != ratings.n_users() || x.n_m != ratings.n_items())
    throw std::invalid_argument("vector/ratings dimension mismatch");
}

std::vector<double> half(const FactorModel& model, const RatingsMatrix& ratings, double lambda,
                         als::SolveStats* stats, int kind) {
  const std::vector<double>& src = kind == 0 ? model.item_data : model.user_data;
  std::vector<double> out(static_cast<std::size_t>(model.n_f) * (kind == 0 ? ratings.n_users() : ratings.n_items()));
  int fb = 0;
  check(alsncg_half_sweep(RatingsDevice::get(ratings), kind, model.n_f, src.data(), lambda, out.data(), &fb));
  if (stats) stats->fallback_columns += fb;
  return out;
}

}  // namespace

namespace als {

void solve_normal_column(const int* idx, const double* vals, int count, const double* const* cols,
                         int n_f, double lambda, double* out, SolveStats& stats) {
  // One-column problem on the device: the referenced columns become a
  // compact item matrix and the column a single user row.
  std::vector<int> uniq(idx, idx + count);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  std::vector<Rating> t(static_cast<std::size_t>(count));
  for (int k = 0; k < count; ++k)
    t[k] = {0, static_cast<int>(std::lower_bound(uniq.begin(), uniq.end(), idx[k]) - uniq.begin()), vals[k]};
  const RatingsMatrix one = RatingsMatrix::from_triples(1, static_cast<int>(uniq.size()), std::move(t));
  FactorModel m(n_f, 1, static_cast<int>(uniq.size()));
  for (std::size_t j = 0; j < uniq.size(); ++j) std::copy(cols[uniq[j]], cols[uniq[j]] + n_f, m.item_col(static_cast<int>(j)));
  const std::vector<double> u = half(m, one, lambda, &stats, 0);
  std::copy(u.begin(), u.end(), out);
}

std::vector<double> update_users(const FactorModel& model, const RatingsMatrix& ratings, double lambda,
                                 SolveStats* stats) {
  return half(model, ratings, lambda, stats, 0);
}

std::vector<double> update_items(const FactorModel& model, const RatingsMatrix& ratings, double lambda,
                                 SolveStats* stats) {
  return half(model, ratings, lambda, stats, 1);
}

FlatVector als_sweep(const FlatVector& x, const RatingsMatrix& ratings, double lambda) {
  check_shape(x, ratings);
  const std::vector<double> hx = concat(x);
  std::vector<double> out(hx.size());
  int fb = 0;
  check(alsncg_als_sweep(RatingsDevice::get(ratings), x.n_f, hx.data(), lambda, out.data(), &fb));
  return split(std::move(out), x.n_f, x.n_u, x.n_m);
}

SolveResult als_solve(const RatingsMatrix& ratings, const SolverConfig& config, const SnapshotSink& snapshot) {
  return run(false, ratings, config, snapshot, nullptr);
}

}  // namespace als

namespace ncg {

double loss(const FlatVector& x, const RatingsMatrix& ratings, double lambda) {
  check_shape(x, ratings);
  const std::vector<double> hx = concat(x);
  double out = 0.0;
  check(alsncg_loss(RatingsDevice::get(ratings), x.n_f, hx.data(), lambda, &out));
  return out;
}

FlatVector gradient(const FlatVector& x, const RatingsMatrix& ratings, double lambda, int /*n_workers*/) {
  check_shape(x, ratings);
  const std::vector<double> hx = concat(x);
  std::vector<double> g(hx.size());
  check(alsncg_gradient(RatingsDevice::get(ratings), x.n_f, hx.data(), lambda, g.data()));
  return split(std::move(g), x.n_f, x.n_u, x.n_m);
}

double beta_bar(const FlatVector& g_next, const FlatVector& g_prev, const FlatVector& gbar_next,
                const FlatVector& gbar_prev) {
  if (!g_next.same_shape(g_prev) || !gbar_next.same_shape(g_next) || !gbar_prev.same_shape(g_next))
    throw std::invalid_argument("beta_bar: shape mismatch");
  const std::vector<double> a = concat(g_next), b = concat(g_prev), c = concat(gbar_next), d = concat(gbar_prev);
  const size_t bytes = a.size() * sizeof(double);
  DevBuf da(a.data(), bytes), db(b.data(), bytes), dc(c.data(), bytes), dd(d.data(), bytes);
  double out = 0.0;
  check(alsncg_dev_beta_bar_seq(default_ctx(), static_cast<std::int64_t>(a.size()), da.d(), db.d(), dc.d(), dd.d(), &out));
  return out;
}

double normalized_grad_norm(const FlatVector& g) {
  const std::int64_t n = g.size();
  return n ? norm(g) / static_cast<double>(n) : 0.0;
}

SolveResult als_ncg_solve(const RatingsMatrix& ratings, const SolverConfig& config, const SnapshotSink& snapshot,
                          const NcgOverrides& overrides) {
  return run(true, ratings, config, snapshot, &overrides);
}

}  // namespace ncg

namespace linesearch {

QuarticPoly quartic_coefficients(const FlatVector& x, const FlatVector& p, const RatingsMatrix& ratings,
                                 double lambda, int /*n_chunks*/, int /*n_workers*/) {
  if (!x.same_shape(p)) throw std::invalid_argument("quartic_coefficients: shape mismatch");
  if (x.n_u != ratings.n_users() || x.n_m != ratings.n_items())
    throw std::invalid_argument("quartic_coefficients: vector/ratings dimension mismatch");
  const std::vector<double> hx = concat(x), hp = concat(p);
  QuarticPoly q;
  check(alsncg_quartic(RatingsDevice::get(ratings), x.n_f, hx.data(), hp.data(), lambda, q.c.data()));
  return q;
}

double armijo_slope(const FlatVector& g, const FlatVector& p) { return dot(g, p); }

LineSearchResult backtracking_search(const QuarticPoly& q, double slope, double alpha0, double c, double tau,
                                     int max_backtracks) {
  LineSearchResult r;
  const int st = alsncg_backtracking_search(q.c.data(), slope, alpha0, c, tau, max_backtracks, &r.alpha,
                                            &r.backtracks);
  if (st < 0) throw std::invalid_argument(alsncg_last_error());
  r.status = static_cast<LineSearchStatus>(st);
  return r;
}

}  // namespace linesearch

namespace parallel {

void parallel_for(int n_tasks, int n_workers, const std::function<void(int)>& fn) {
  if (n_tasks <= 0) return;
  n_workers = std::min(n_workers, n_tasks);
  if (n_workers <= 1) {
    for (int t = 0; t < n_tasks; ++t) fn(t);
    return;
  }
  std::atomic<int> next{0};
  std::exception_ptr first;
  std::mutex mu;
  auto work = [&] {
    for (int t; (t = next.fetch_add(1, std::memory_order_relaxed)) < n_tasks;) {
      try {
        fn(t);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!first) first = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < n_workers; ++w) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (first) std::rethrow_exception(first);
}

Partitioning build_partitioning(int n_columns, int n_blocks) {
  if (n_blocks < 1) throw std::invalid_argument("build_partitioning: n_blocks must be >= 1");
  if (n_columns < 0) throw std::invalid_argument("build_partitioning: negative column count");
  return Partitioning{n_blocks, n_columns};
}

std::int64_t RoutingTable::total_columns() const {
  std::int64_t t = 0;
  for (const auto& l : lists) t += static_cast<std::int64_t>(l.size());
  return t;
}

std::pair<RoutingTable, RoutingTable> build_routing_tables(const RatingsMatrix& ratings, const Partitioning& users,
                                                           const Partitioning& items) {
  if (users.n_columns != ratings.n_users() || items.n_columns != ratings.n_items())
    throw std::invalid_argument("build_routing_tables: partitioning does not cover the ratings");
  RoutingTable tu{users.n_blocks, items.n_blocks, {}}, tm{items.n_blocks, users.n_blocks, {}};
  tu.lists.resize(static_cast<std::size_t>(users.n_blocks) * items.n_blocks);
  tm.lists.resize(static_cast<std::size_t>(items.n_blocks) * users.n_blocks);
  // A column is listed once per distinct destination block among its
  // neighbours; scanning columns in ascending order keeps lists sorted.
  std::vector<int> mark(static_cast<std::size_t>(std::max(users.n_blocks, items.n_blocks)), -1);
  for (int i = 0; i < ratings.n_users(); ++i)
    for (int j : ratings.user_items(i)) {
      const int d = items.block_of(j);
      if (mark[d] != i) {
        mark[d] = i;
        tu.lists[static_cast<std::size_t>(users.block_of(i)) * items.n_blocks + d].push_back(i);
      }
    }
  std::fill(mark.begin(), mark.end(), -1);
  for (int j = 0; j < ratings.n_items(); ++j)
    for (int i : ratings.item_users(j)) {
      const int d = users.block_of(i);
      if (mark[d] != j) {
        mark[d] = j;
        tm.lists[static_cast<std::size_t>(items.block_of(j)) * users.n_blocks + d].push_back(j);
      }
    }
  return {std::move(tu), std::move(tm)};
}

std::int64_t ShuffleStats::cross_block_columns() const {
  std::int64_t t = 0;
  for (int s = 0; s < n_source_blocks; ++s)
    for (int d = 0; d < n_dest_blocks; ++d)
      if (s != d) t += sent_between(s, d);
  return t;
}

ShuffleStats stats_for(const RoutingTable& table, int n_f) {
  ShuffleStats st;
  st.n_source_blocks = table.n_source_blocks;
  st.n_dest_blocks = table.n_dest_blocks;
  st.sent.resize(table.lists.size());
  for (std::size_t k = 0; k < table.lists.size(); ++k) {
    st.sent[k] = static_cast<std::int64_t>(table.lists[k].size());
    st.columns_sent += st.sent[k];
  }
  st.scalar_values_sent = st.columns_sent * n_f;
  return st;
}

SweepPlan SweepPlan::build(const RatingsMatrix& ratings, int n_blocks) {
  SweepPlan p;
  p.users = build_partitioning(ratings.n_users(), n_blocks);
  p.items = build_partitioning(ratings.n_items(), n_blocks);
  auto [tu, tm] = build_routing_tables(ratings, p.users, p.items);
  p.t_u = std::move(tu);
  p.t_m = std::move(tm);
  return p;
}

HalfSweepOutput parallel_half_sweep(HalfSweepKind kind, const FactorModel& model, const RatingsMatrix& ratings,
                                    double lambda, const SweepPlan& plan, int /*n_workers*/) {
  const bool users = kind == HalfSweepKind::kUsers;
  HalfSweepOutput out;
  out.stats = stats_for(users ? plan.t_m : plan.t_u, model.n_f);
  out.columns = half(model, ratings, lambda, &out.solve_stats, users ? 0 : 1);
  return out;
}

}  // namespace parallel

}  // namespace alsncg
