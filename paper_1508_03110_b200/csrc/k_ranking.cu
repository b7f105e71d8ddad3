// k_ranking.cu -- ranking evaluation:
// ranking::mean_ranking_accuracy (ranking.cpp:90-109) on the device.
//
// For every user i the reference ranks all items by the score u_i.m_j
// (sequential dot, separate multiply and add rounding; ties by ascending item
// id, ranking.cpp:40-57) under the converged model (p1) and under the model
// at iteration k (p2), and counts the adjacent swaps of the top-t walk of
// ranking.cpp:59-88.  The walk's count has a closed form: with rank2(x) the
// position of item x in p2,
//     swaps = sum_{r<t} [ rank2(p1[r]) - #{q<r : rank2(p1[q]) < rank2(p1[r])} ],
// so no full sort is needed: per user the top t of p1 are selected and their
// p2 positions counted.
//   K_R1 k_rank_scores: scores of a chunk of users x all items, exactly the
//        reference's arithmetic (__dmul_rn / __dadd_rn in k order) so every
//        comparison, tie included, is the reference's -- GEMM-shaped, FP64
//        pipe bound (2 ops per term, no FMA by construction);
//   K_R2 k_rank_users: one warp per user: a single pass over p1's scores with
//        a per-lane top-t insertion list, a t-round warp merge, one pass over
//        p2's scores counting rank2 of the t picks, the closed form above.
// The per-user accuracies come back to the host, which sums them in user
// order as the reference does (ranking.cpp:104-107).
#include <cfloat>

#include "common.cuh"

namespace ab2 {

namespace {

constexpr int kRankTile = 64;  // users x items per score CTA (16x16 threads, 4x4 each)

__global__ void __launch_bounds__(256) k_rank_scores(const double* __restrict__ U, const double* __restrict__ M,
                                                     int n_f, int u0, int nu, int n_m, double* __restrict__ S) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int ub = blockIdx.y * kRankTile + ty * 4;  // chunk-local user
  const int jb = blockIdx.x * kRankTile + tx * 4;
  const double* ur[4];
  const double* mr[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ur[i] = U + static_cast<int64_t>(u0 + min(ub + i, nu - 1)) * n_f;
    mr[i] = M + static_cast<int64_t>(min(jb + i, n_m - 1)) * n_f;
  }
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k = 0; k < n_f; ++k) {  // ranking.cpp:45-47: s += u[k] * m[k]
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[i] = __ldg(ur[i] + k);
      b[i] = __ldg(mr[i] + k);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ub + i < nu && jb + j < n_m) S[static_cast<int64_t>(ub + i) * n_m + jb + j] = acc[i][j];
}

// item a ranks before item b (score descending, then id ascending)
__device__ __forceinline__ bool before(double sa, int a, double sb, int b) {
  return sa > sb || (sa == sb && a < b);
}

__global__ void __launch_bounds__(256) k_rank_users(const double* __restrict__ S1, const double* __restrict__ S2,
                                                    int nu, int n_m, int t, int cap, double* lane_s, int* lane_id,
                                                    int* picks, double* __restrict__ q) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= nu) return;
  const double* s1 = S1 + static_cast<int64_t>(w) * n_m;
  const double* s2 = S2 + static_cast<int64_t>(w) * n_m;
  // this lane's best-first list of at most cap = min(t, its item count)
  // (score, id) of p1
  double* ls = lane_s + (static_cast<int64_t>(w) * 32 + lane) * cap;
  int* li = lane_id + (static_cast<int64_t>(w) * 32 + lane) * cap;
  int len = 0;
  for (int j = lane; j < n_m; j += 32) {
    const double s = s1[j];
    if (len == cap && !before(s, j, ls[cap - 1], li[cap - 1])) continue;
    int p = len < cap ? len : cap - 1;
    while (p > 0 && before(s, j, ls[p - 1], li[p - 1])) {
      ls[p] = ls[p - 1];
      li[p] = li[p - 1];
      --p;
    }
    ls[p] = s;
    li[p] = j;
    if (len < cap) ++len;
  }
  // t-round merge of the 32 lists: p1[0..t) (t <= 32 * cap always holds)
  int* pk = picks + static_cast<int64_t>(w) * t;
  int head = 0;
  for (int r = 0; r < t; ++r) {
    double bs = head < len ? ls[head] : -DBL_MAX;
    int bi = head < len ? li[head] : 0x7fffffff;
    const bool have = head < len;
    double cs = bs;
    int ci = bi, cl = have ? lane : 32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double os = __shfl_xor_sync(kFull, cs, o);
      const int oi = __shfl_xor_sync(kFull, ci, o);
      const int ol = __shfl_xor_sync(kFull, cl, o);
      if (ol < 32 && (cl == 32 || before(os, oi, cs, ci))) {
        cs = os;
        ci = oi;
        cl = ol;
      }
    }
    if (lane == cl) ++head;
    if (lane == 0) pk[r] = ci;
  }
  __syncwarp();
  // rank2 of every pick: #{j : j ranks before the pick under p2}; lane r
  // counts pick r0 + r with every lane reading the same s2[j] (broadcast).
  // The counts go to a per-warp array in the (already merged) list space.
  int* rk = picks + static_cast<int64_t>(nu) * t + static_cast<int64_t>(w) * t;
  for (int r0 = 0; r0 < t; r0 += 32) {
    const int r = r0 + lane;
    const int x = r < t ? pk[r] : 0;
    const double sx = s2[x];
    int cnt = 0;
    for (int j = 0; j < n_m; ++j) cnt += before(s2[j], j, sx, x) ? 1 : 0;
    if (r < t) rk[r] = cnt;
  }
  __syncwarp();
  int64_t swaps = 0;
  for (int r = lane; r < t; r += 32) {
    int less = 0;
    for (int q2 = 0; q2 < r; ++q2) less += rk[q2] < rk[r] ? 1 : 0;
    swaps += rk[r] - less;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) swaps += __shfl_xor_sync(kFull, swaps, o);
  if (lane == 0) {
    const int64_t smax = static_cast<int64_t>(t) * (2 * static_cast<int64_t>(n_m) - t - 1) / 2;
    q[w] = smax == 0 ? 1.0 : 1.0 - static_cast<double>(swaps) / static_cast<double>(smax);
  }
}

}  // namespace

void launch_mean_ranking(Ctx* ctx, int n_f, int n_u, int n_m, const double* d_uk, const double* d_mk,
                         const double* d_uf, const double* d_mf, int t, double* d_q) {
  // users per chunk: <= 1 GiB of scores per model and <= 1 GiB of lane lists
  const int cap = std::min(t, (n_m + 31) / 32);
  const size_t by_scores = (size_t(1) << 30) / (sizeof(double) * std::max(n_m, 1));
  const size_t by_lists = (size_t(1) << 30) / (12 * 32 * static_cast<size_t>(cap));
  const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(n_u, std::min(by_scores, by_lists))));
  double* S = static_cast<double*>(ctx->scratch(10, sizeof(double) * 2 * static_cast<size_t>(chunk) * n_m));
  double* lane_s = static_cast<double*>(ctx->scratch(11, sizeof(double) * static_cast<size_t>(chunk) * 32 * cap));
  int* lane_id = static_cast<int*>(ctx->scratch(12, sizeof(int) * static_cast<size_t>(chunk) * 32 * cap));
  int* picks = static_cast<int*>(ctx->scratch(13, sizeof(int) * 2 * static_cast<size_t>(chunk) * t));
  for (int u0 = 0; u0 < n_u; u0 += chunk) {
    const int nu = std::min(chunk, n_u - u0);
    const dim3 grid((n_m + kRankTile - 1) / kRankTile, (nu + kRankTile - 1) / kRankTile);
    int tok = ctx->begin_launch("ranking_scores");
    k_rank_scores<<<grid, 256, 0, ctx->stream>>>(d_uf, d_mf, n_f, u0, nu, n_m, S);
    k_rank_scores<<<grid, 256, 0, ctx->stream>>>(d_uk, d_mk, n_f, u0, nu, n_m, S + static_cast<size_t>(chunk) * n_m);
    ctx->end_launch(tok);
    tok = ctx->begin_launch("ranking_users");
    k_rank_users<<<(nu + 7) / 8, 256, 0, ctx->stream>>>(S, S + static_cast<size_t>(chunk) * n_m, nu, n_m, t, cap,
                                                        lane_s, lane_id, picks, d_q + u0);
    ctx->end_launch(tok);
  }
}

}  // namespace ab2
