// alsncg/snapshot.hpp -- drop-in declaration of the "ALSNCG01" model dump
// (/root/reference/proj/include/alsncg/snapshot.hpp:21-44): magic, five
// little-endian int64 {n_f, n_u, n_m, iter, seed}, then user and item data.
#pragma once

#include <cstdint>
#include <string>

#include "alsncg/factors.hpp"

namespace alsncg {

struct SnapshotMeta {
  int n_f = 0;
  int n_u = 0;
  int n_m = 0;
  std::int64_t iter = 0;
  std::uint64_t seed = 0;
};

void save_model(const std::string& path, const FactorModel& model, std::int64_t iter,
                std::uint64_t seed);

struct LoadedModel {
  FactorModel model;
  SnapshotMeta meta;
};

/// DataError on a missing file or malformed header.
LoadedModel load_model(const std::string& path);

}  // namespace alsncg
