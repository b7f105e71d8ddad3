// host_data.h -- host-side data path (see host_data.cpp).
#pragma once

#include <cstdint>
#include <random>
#include <string>

#include "alsncg_capi.h"

namespace ab2 {

struct HostRng {
  std::mt19937_64 gen;
  bool has_spare = false;
  double spare = 0.0;
  explicit HostRng(uint64_t seed) : gen(seed) {}
  double uniform();
  double normal();
};

int sample_cumulative(const double* cum, int n, double u);

int csr_build(int n_u, int n_m, int64_t nnz, const int* users, const int* items,
              const double* values, bool single, int64_t* uptr, int* uidx, double* uval,
              int64_t* iptr, int* iidx, double* ival, int* dup_user, int* dup_item,
              std::string* err);
void random_init(int n_f, int n_u, int n_m, uint64_t seed, double* user, double* item);
int synth_generate(int n_u, int n_m, int64_t nnz, int min_per_user, uint64_t seed, int* users,
                   int* items, double* values, std::string* err);
int backtracking_search(const double c[5], double slope, double alpha0, double armijo_c,
                        double tau, int max_backtracks, double* alpha, int* backtracks);

}  // namespace ab2
