// alsncg/ranking.hpp -- drop-in for the reference's ranking evaluation
// (proj/include/alsncg/ranking.hpp:20-41).  rank_items and ranking_accuracy
// are the per-user host utilities; mean_ranking_accuracy -- the all-users
// evaluation the rank-eval harness runs on every snapshot -- executes on the
// B200 (k_ranking.cu) with the reference's exact score arithmetic.
#pragma once

#include <vector>

#include "alsncg/factors.hpp"

namespace alsncg::ranking {

// Item ids by descending u_i.m_j, ties by ascending item id.
using RankingVector = std::vector<int>;

// std::out_of_range on a bad user index (ranking.cpp:40-57).
RankingVector rank_items(const FactorModel& model, int user);

// Normalised top-t Kendall-tau accuracy q = 1 - s/s_max, s the adjacent swaps
// of the top-t walk, s_max = t(2n - t - 1)/2; std::invalid_argument unless p1
// and p2 permute the same [0, n) and 1 <= t <= n (ranking.cpp:59-88).
double ranking_accuracy(const RankingVector& p1, const RankingVector& p2, int t);

// Mean over all users of ranking_accuracy(rank_items(model_final, i),
// rank_items(model_at_k, i), t) (ranking.cpp:90-109).  n_workers is accepted
// for API parity (the device evaluation does not depend on it).
double mean_ranking_accuracy(const FactorModel& model_at_k, const FactorModel& model_final, int t,
                             int n_workers = 1);

}  // namespace alsncg::ranking
