// host_data.cpp -- host-side data path of the product: the dual CSR/CSC
// build (ratings.cpp:28-89 semantics, bit-identical output), random_init
// (factors.cpp:24-32), the seeded BASELINE workload generator and the scalar
// backtracking search (linesearch.cpp:115-131).  No device work here.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
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

// ---------------------------------------------------------- CSR / CSC --
// Counting sort by user (stable), then a per-user sort by item; the sorted
// (user,item) keys are unique once duplicates are rejected, so the result
// does not depend on the sort algorithm and equals the reference's std::sort
// output bit for bit.  CSC is the reference's stable counting pass.
int csr_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
              const double* values, bool single, int64_t* uptr, int* uidx, double* uval,
              int64_t* iptr, int* iidx, double* ival, int* dup_user, int* dup_item,
              std::string* err) {
  if (n_u < 0 || n_m < 0) {
    *err = "negative matrix dimensions";
    return ALSNCG_EDATA;
  }
  for (int64_t t = 0; t < nnz; ++t) {  // ratings.cpp:32-42, input order
    if (users[t] < 0 || users[t] >= n_u || items[t] < 0 || items[t] >= n_m) {
      *err = "rating index out of range: user " + std::to_string(users[t]) + ", item " +
             std::to_string(items[t]);
      return ALSNCG_EDATA;
    }
    if (!std::isfinite(values[t])) {
      *err = "non-finite rating value for user " + std::to_string(users[t]) + ", item " +
             std::to_string(items[t]);
      return ALSNCG_EDATA;
    }
  }
  std::fill(uptr, uptr + n_u + 1, 0);
  for (int64_t t = 0; t < nnz; ++t) ++uptr[users[t] + 1];
  for (int i = 0; i < n_u; ++i) uptr[i + 1] += uptr[i];
  std::vector<int64_t> cur(uptr, uptr + n_u);
  std::vector<std::pair<int, double>> tmp(static_cast<size_t>(nnz));
  for (int64_t t = 0; t < nnz; ++t) tmp[cur[users[t]]++] = {items[t], values[t]};
  for (int i = 0; i < n_u; ++i) {
    auto b = tmp.begin() + uptr[i], e = tmp.begin() + uptr[i + 1];
    std::sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
    for (auto it = b + (b != e ? 1 : 0); it < e; ++it)
      if (it->first == (it - 1)->first) {  // ratings.cpp:47-51 (first in sorted order)
        if (dup_user) *dup_user = i;
        if (dup_item) *dup_item = it->first;
        *err = "duplicate rating for user " + std::to_string(i) + ", item " +
               std::to_string(it->first);
        return ALSNCG_EDUP;
      }
  }
  std::fill(iptr, iptr + n_m + 1, 0);
  for (int64_t t = 0; t < nnz; ++t) ++iptr[tmp[t].first + 1];
  for (int j = 0; j < n_m; ++j) iptr[j + 1] += iptr[j];
  std::vector<int64_t> icur(iptr, iptr + n_m);
  for (int i = 0; i < n_u; ++i)
    for (int64_t t = uptr[i]; t < uptr[i + 1]; ++t) {
      double v = tmp[t].second;
      if (single) v = static_cast<double>(static_cast<float>(v));  // ratings.cpp:80
      uidx[t] = tmp[t].first;
      uval[t] = v;
      const int64_t ip = icur[tmp[t].first]++;
      iidx[ip] = i;
      ival[ip] = v;
    }
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
  HostRng rng(seed);
  const double sd = std::pow(10.0, -0.25);
  std::vector<double> ut(static_cast<size_t>(n_u) * kRank), mt(static_cast<size_t>(n_m) * kRank);
  for (double& v : ut) v = sd * rng.normal();
  for (double& v : mt) v = sd * rng.normal();
  std::vector<int> cnt(n_u, min_per_user);
  const double extra = static_cast<double>(nnz) / n_u - min_per_user;
  if (extra > 0.0) {
    for (int i = 0; i < n_u; ++i) {
      const double c = min_per_user + std::round(extra * std::exp(rng.normal() - 0.5));
      cnt[i] = static_cast<int>(std::min<double>(cap, std::max<double>(min_per_user, c)));
    }
  }
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
  std::vector<int> stamp(n_m, -1);
  int64_t pos = 0;
  for (int i = 0; i < n_u; ++i) {
    const double* u = ut.data() + static_cast<size_t>(i) * kRank;
    for (int drawn = 0; drawn < cnt[i];) {
      const int j = sample_cumulative(cum.data(), n_m, rng.uniform());
      if (stamp[j] == i) continue;
      stamp[j] = i;
      ++drawn;
      const double* m = mt.data() + static_cast<size_t>(j) * kRank;
      double score = 0.0;
      for (int k = 0; k < kRank; ++k) score += u[k] * m[k];
      const double eps = 0.5 * rng.normal();
      const double r = std::round(2.0 * (3.5 + score + eps)) / 2.0;
      users[pos] = i;
      items[pos] = j;
      values[pos] = std::min(5.0, std::max(0.5, r));
      ++pos;
    }
  }
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
