// host_data.cpp -- host-side data path of the product: the dual CSR/CSC
// build (ratings.cpp:28-89 semantics, bit-identical output), random_init
// (factors.cpp:24-32), the seeded BASELINE workload generator and the scalar
// backtracking search (linesearch.cpp:115-131).  No device work here.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

#include "host_data.h"

namespace ab2 {

// ----------------------------------------------------------------- Rng --
// Same stream as alsncg::Rng (rng.hpp:26-45): raw mt19937_64 draws, 53-bit
// uniforms, Box-Muller normals with a cached spare.
double HostRng::uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }

double HostRng::normal() {
  if (has_spare) {
    has_spare = false;
    return spare;
  }
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double mag = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * std::numbers::pi * u2;
  spare = mag * std::sin(ang);
  has_spare = true;
  return mag * std::cos(ang);
}

int sample_cumulative(const double* cum, int n, double u) {
  const double target = u * cum[n - 1];
  const double* it = std::upper_bound(cum, cum + n, target);
  if (it == cum + n) --it;
  return static_cast<int>(it - cum);
}

// ------------------------------------------------------- host threads --
// Static-partition parallel loop over [0, n) on the host's cores (the data
// path for configs 3-4 moves 10^8-10^9 ratings).  f(lo, hi, t).
template <typename F>
void par_ranges(int64_t n, F&& f, int max_threads = 0) {
  int T = static_cast<int>(std::thread::hardware_concurrency());
  if (max_threads > 0) T = std::min(T, max_threads);
  T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(T, n / 65536 + 1)));
  if (T <= 1) {
    f(int64_t(0), n, 0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T, t); });
  for (auto& x : th) x.join();
}

int host_threads(int64_t n) {
  return static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(std::thread::hardware_concurrency(), n / 65536 + 1)));
}

// ---------------------------------------------------------- CSR / CSC --
// ratings.cpp:28-89, multi-threaded and bit-identical: validation reports
// the first bad triple in input order; a per-user bucket fill (atomic
// cursors) followed by a per-user sort by item gives the (user, item) order
// of the reference's std::sort (keys are unique once duplicates are
// rejected, so the fill order inside a bucket does not matter); the first
// duplicate in sorted order is reported; the CSC is the reference's stable
// counting pass, parallelised over contiguous user ranges with per-range
// item offsets (users stay ascending within every item).
int csr_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
              const double* values, bool single, int64_t* uptr, int* uidx, double* uval,
              int64_t* iptr, int* iidx, double* ival, int* dup_user, int* dup_item,
              std::string* err) {
  if (n_u < 0 || n_m < 0) {
    *err = "negative matrix dimensions";
    return ALSNCG_EDATA;
  }
  std::atomic<int64_t> first_bad{nnz};
  par_ranges(nnz, [&](int64_t lo, int64_t hi, int) {  // ratings.cpp:32-42, input order
    for (int64_t t = lo; t < hi && t < first_bad.load(std::memory_order_relaxed); ++t)
      if (users[t] < 0 || users[t] >= n_u || items[t] < 0 || items[t] >= n_m || !std::isfinite(values[t])) {
        int64_t cur = first_bad.load();
        while (t < cur && !first_bad.compare_exchange_weak(cur, t)) {
        }
        break;
      }
  });
  if (first_bad.load() < nnz) {
    const int64_t t = first_bad.load();
    if (users[t] < 0 || users[t] >= n_u || items[t] < 0 || items[t] >= n_m)
      *err = "rating index out of range: user " + std::to_string(users[t]) + ", item " +
             std::to_string(items[t]);
    else
      *err = "non-finite rating value for user " + std::to_string(users[t]) + ", item " +
             std::to_string(items[t]);
    return ALSNCG_EDATA;
  }
  // user counts (atomic histogram) -> uptr
  std::vector<std::atomic<int64_t>> cnt(static_cast<size_t>(n_u) + 1);
  for (auto& c : cnt) c.store(0, std::memory_order_relaxed);
  par_ranges(nnz, [&](int64_t lo, int64_t hi, int) {
    for (int64_t t = lo; t < hi; ++t) cnt[users[t]].fetch_add(1, std::memory_order_relaxed);
  });
  uptr[0] = 0;
  for (int i = 0; i < n_u; ++i) uptr[i + 1] = uptr[i] + cnt[i].load(std::memory_order_relaxed);
  // bucket fill (cursor per user), then per-user sort by item
  for (int i = 0; i < n_u; ++i) cnt[i].store(uptr[i], std::memory_order_relaxed);
  std::vector<std::pair<int, double>> tmp(static_cast<size_t>(nnz));
  par_ranges(nnz, [&](int64_t lo, int64_t hi, int) {
    for (int64_t t = lo; t < hi; ++t)
      tmp[cnt[users[t]].fetch_add(1, std::memory_order_relaxed)] = {items[t], values[t]};
  });
  std::atomic<int> dup_row{n_u};
  par_ranges(n_u, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; ++i) {
      auto b = tmp.begin() + uptr[i], e = tmp.begin() + uptr[i + 1];
      std::sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto it = b + (b != e ? 1 : 0); it < e; ++it)
        if (it->first == (it - 1)->first) {
          int cur = dup_row.load();
          while (i < cur && !dup_row.compare_exchange_weak(cur, static_cast<int>(i))) {
          }
          break;
        }
    }
  });
  if (dup_row.load() < n_u) {  // ratings.cpp:47-51 (first duplicate in sorted order)
    const int i = dup_row.load();
    for (int64_t t = uptr[i] + 1; t < uptr[i + 1]; ++t)
      if (tmp[t].first == tmp[t - 1].first) {
        if (dup_user) *dup_user = i;
        if (dup_item) *dup_item = tmp[t].first;
        *err = "duplicate rating for user " + std::to_string(i) + ", item " + std::to_string(tmp[t].first);
        return ALSNCG_EDUP;
      }
  }
  // CSR arrays + CSC (stable counting by item over contiguous user ranges)
  const int T = host_threads(nnz);
  std::vector<int> ub(T + 1);
  for (int t = 0; t <= T; ++t)  // user ranges with ~equal rating counts
    ub[t] = t == T ? n_u
                   : static_cast<int>(std::lower_bound(uptr, uptr + n_u + 1, nnz * t / T) - uptr);
  std::vector<std::vector<int64_t>> icnt(T, std::vector<int64_t>(static_cast<size_t>(n_m), 0));
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (int64_t k = uptr[ub[t]]; k < uptr[ub[t + 1]]; ++k) ++icnt[t][tmp[k].first];
    });
  for (auto& x : th) x.join();
  th.clear();
  iptr[0] = 0;
  for (int j = 0; j < n_m; ++j) {
    int64_t run = iptr[j];
    for (int t = 0; t < T; ++t) {
      const int64_t c = icnt[t][j];
      icnt[t][j] = run;  // this range's first slot in item j
      run += c;
    }
    iptr[j + 1] = run;
  }
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      std::vector<int64_t>& cur = icnt[t];
      for (int i = ub[t]; i < ub[t + 1]; ++i)
        for (int64_t k = uptr[i]; k < uptr[i + 1]; ++k) {
          double v = tmp[k].second;
          if (single) v = static_cast<double>(static_cast<float>(v));  // ratings.cpp:80
          uidx[k] = tmp[k].first;
          uval[k] = v;
          const int64_t ip = cur[tmp[k].first]++;
          iidx[ip] = i;
          ival[ip] = v;
        }
    });
  for (auto& x : th) x.join();
  return ALSNCG_OK;
}

void random_init(int n_f, int n_u, int n_m, uint64_t seed, double* user, double* item) {
  HostRng rng(seed);
  const double scale = 1.0 / std::sqrt(static_cast<double>(n_f));
  const int64_t nm = static_cast<int64_t>(n_f) * n_m, nu = static_cast<int64_t>(n_f) * n_u;
  for (int64_t k = 0; k < nm; ++k) item[k] = rng.uniform() * scale;
  for (int64_t k = 0; k < nu; ++k) user[k] = rng.uniform() * scale;
}

// ----------------------------------------------------------- generator --
// BASELINE.json configs: rank-10 truth u*, m* ~ N(0, var 1/sqrt(10)) (so
// u*.m* has unit variance); per-user counts >= min_per_user, heavy-tailed
// lognormal(sigma=1) around the mean nnz/n_u, fixed up to sum exactly to nnz;
// items ~ Zipf(s=1) via sample_cumulative with per-user redraws on repeats;
// r = clamp(round_half_away(2*(3.5 + u*.m* + N(0,0.5^2)))/2, 0.5, 5.0).
//
// One mt19937_64 stream defines the output (oracle/alsncg_oracle.c
// orc_synth_generate is the sequential statement; tests pin the two bitwise).
// It is produced on all host cores without changing a bit: the raw stream is
// drawn sequentially in chunks (cheap), the expensive per-draw functions are
// evaluated speculatively in parallel for EVERY position of a chunk -- the
// item index as if the draw were an item draw (binary search over the Zipf
// cumulative weights) and the Box-Muller pair as if a normal started there --
// then a sequential walker replays the exact call sequence (item draw,
// repeat check, normal with its cached spare) picking the precomputed values,
// and a final parallel pass forms the ratings from (user, item, normal).
namespace {

struct Stream {
  std::mt19937_64 gen;
  explicit Stream(uint64_t seed) : gen(seed) {}
  double next() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
};

// Box-Muller of rng.cpp:36-49 from the uniforms (a, b) at stream positions
// (p, p+1): u1 = 1 - a, u2 = b; first call returns cos, caches sin.
inline void box_muller(double a, double b, double* c, double* s) {
  const double u1 = 1.0 - a;
  const double mag = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * std::numbers::pi * b;
  *s = mag * std::sin(ang);
  *c = mag * std::cos(ang);
}

}  // namespace

int synth_generate(int n_u, int n_m, int64_t nnz, int min_per_user, uint64_t seed, int* users,
                   int* items, double* values, std::string* err) {
  constexpr int kRank = 10;
  if (n_u <= 0 || n_m <= 0 || min_per_user < 1 || min_per_user > n_m) {
    *err = "synth_generate: bad dimensions";
    return ALSNCG_EINVAL;
  }
  const int cap = std::max(min_per_user, n_m / 2);
  if (nnz < static_cast<int64_t>(min_per_user) * n_u || nnz > static_cast<int64_t>(cap) * n_u) {
    *err = "synth_generate: nnz outside [min_per_user*n_u, cap*n_u]";
    return ALSNCG_EINVAL;
  }
  Stream rng(seed);
  const double sd = std::pow(10.0, -0.25);
  const double extra = static_cast<double>(nnz) / n_u - min_per_user;
  // ---- normal() calls 0..Na-1 before the first item draw: truth factors
  // (users then items), then one per user count; no uniform() in between, so
  // call c uses the Box-Muller pair c/2 of the stream (cos for even c).
  const int64_t n_truth = static_cast<int64_t>(n_u + n_m) * kRank;
  const int64_t Na = n_truth + (extra > 0.0 ? n_u : 0);
  const int64_t pairs = (Na + 1) / 2;
  std::vector<double> nv(static_cast<size_t>(2 * pairs));
  {
    std::vector<double> raw(static_cast<size_t>(2 * pairs));
    for (double& v : raw) v = rng.next();
    par_ranges(pairs, [&](int64_t lo, int64_t hi, int) {
      for (int64_t k = lo; k < hi; ++k) box_muller(raw[2 * k], raw[2 * k + 1], &nv[2 * k], &nv[2 * k + 1]);
    });
  }
  bool has_spare = (Na & 1) != 0;  // an odd count leaves the sin of the last pair cached
  double spare = has_spare ? nv[static_cast<size_t>(Na)] : 0.0;
  std::vector<double> ut(static_cast<size_t>(n_u) * kRank), mt(static_cast<size_t>(n_m) * kRank);
  par_ranges(n_truth, [&](int64_t lo, int64_t hi, int) {
    for (int64_t k = lo; k < hi; ++k) {
      const double v = sd * nv[k];
      if (k < static_cast<int64_t>(n_u) * kRank) ut[k] = v;
      else mt[k - static_cast<int64_t>(n_u) * kRank] = v;
    }
  });
  std::vector<int> cnt(n_u, min_per_user);
  if (extra > 0.0) {
    for (int i = 0; i < n_u; ++i) {
      const double c = min_per_user + std::round(extra * std::exp(nv[n_truth + i] - 0.5));
      cnt[i] = static_cast<int>(std::min<double>(cap, std::max<double>(min_per_user, c)));
    }
  }
  std::vector<double>().swap(nv);
  int64_t total = 0;
  for (int c : cnt) total += c;
  while (total != nnz) {  // +-1 adjustments in user order
    bool moved = false;
    for (int i = 0; i < n_u && total != nnz; ++i) {
      if (total < nnz && cnt[i] < cap) {
        ++cnt[i];
        ++total;
        moved = true;
      } else if (total > nnz && cnt[i] > min_per_user) {
        --cnt[i];
        --total;
        moved = true;
      }
    }
    if (!moved) {
      *err = "synth_generate: cannot meet nnz";
      return ALSNCG_EINVAL;
    }
  }
  std::vector<double> cum(n_m);
  double run = 0.0;
  for (int j = 0; j < n_m; ++j) {
    run += 1.0 / static_cast<double>(j + 1);
    cum[j] = run;
  }
  // ---- item draws and rating noise, in chunks of the raw stream
  constexpr int64_t kChunk = int64_t(1) << 24;
  std::vector<double> raw(kChunk + 1), bmc(kChunk), bms(kChunk);
  std::vector<int> jv(kChunk);
  int64_t have = 0, p = 0;  // valid speculative positions [0, have); cursor p
  auto refill = [&]() {   // keep the unread tail, draw the rest, recompute
    const int64_t keep = have + 1 - p;  // raw[have] is the look-ahead draw
    std::memmove(raw.data(), raw.data() + p, sizeof(double) * static_cast<size_t>(keep));
    for (int64_t k = keep; k <= kChunk; ++k) raw[k] = rng.next();
    have = kChunk;
    p = 0;
    par_ranges(have, [&](int64_t lo, int64_t hi, int) {
      for (int64_t k = lo; k < hi; ++k) {
        jv[k] = sample_cumulative(cum.data(), n_m, raw[k]);
        box_muller(raw[k], raw[k + 1], &bmc[k], &bms[k]);
      }
    });
  };
  raw[0] = rng.next();  // first look-ahead draw
  have = 0;
  p = 0;
  refill();
  std::vector<double> noise(static_cast<size_t>(nnz));
  std::vector<int> stamp(n_m, -1);
  int64_t pos = 0;
  for (int i = 0; i < n_u; ++i) {
    for (int drawn = 0; drawn < cnt[i];) {
      if (p >= have) refill();
      const int j = jv[p++];  // uniform() -> sample_cumulative
      if (stamp[j] == i) continue;
      stamp[j] = i;
      ++drawn;
      double z;  // normal()
      if (has_spare) {
        has_spare = false;
        z = spare;
      } else {
        if (p + 1 >= have) refill();  // the pair (p, p+1) lies inside [0, have]
        z = bmc[p];
        spare = bms[p];
        has_spare = true;
        p += 2;
      }
      users[pos] = i;
      items[pos] = j;
      noise[pos] = z;
      ++pos;
    }
  }
  par_ranges(nnz, [&](int64_t lo, int64_t hi, int) {
    for (int64_t t = lo; t < hi; ++t) {
      const double* u = ut.data() + static_cast<size_t>(users[t]) * kRank;
      const double* m = mt.data() + static_cast<size_t>(items[t]) * kRank;
      double score = 0.0;
      for (int k = 0; k < kRank; ++k) score += u[k] * m[k];
      const double eps = 0.5 * noise[t];
      const double r = std::round(2.0 * (3.5 + score + eps)) / 2.0;
      values[t] = std::min(5.0, std::max(0.5, r));
    }
  });
  return ALSNCG_OK;
}

// linesearch.cpp:115-131 (host scalar code, O(max_backtracks)).
int backtracking_search(const double c[5], double slope, double alpha0, double armijo_c,
                        double tau, int max_backtracks, double* alpha, int* backtracks) {
  auto q = [&](double a) { return (((c[4] * a + c[3]) * a + c[2]) * a + c[1]) * a + c[0]; };
  if (!(slope < 0.0)) {
    *alpha = 0.0;
    *backtracks = 0;
    return 1;
  }
  const double q0 = q(0.0);
  double a = alpha0;
  for (int k = 0; k <= max_backtracks; ++k) {
    if (q(a) - q0 <= a * armijo_c * slope) {
      *alpha = a;
      *backtracks = k;
      return 0;
    }
    a *= tau;
  }
  *alpha = 0.0;
  *backtracks = max_backtracks;
  return 2;
}

}  // namespace ab2
