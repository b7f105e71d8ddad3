// k_residual.cu -- residual passes over the ratings:
//   K5 gradient  (ncg.cpp:70-116): g_i = 2*lambda*n_i*x_i + sum_j 2(x_i.y_j - r_ij) y_j,
//                CSR pass for user rows then CSC pass for item rows;
//   K6 loss      (ncg.cpp:43-68);
//   K7 quartic   (linesearch.cpp:46-111): the exact degree-4 profile of the
//                loss along p, one pass over the ratings.
//
// Layout: a sub-group of TPR lanes owns one rating at a time; each lane holds
// V2 double2 of the row (elements 2*(sl + TPR*k) + {0,1}), so one warp step
// covers 32/TPR ratings with log2(TPR) shuffle rounds.  TPR/V2 are picked
// from n_f (small ranks use many ratings per warp, no wasted lanes).
// Gradient rows are cut into segments (SegPlan) and multi-segment rows are
// reduced in segment order; quartic/loss accumulate double-double partials
// per fixed 64-row tile and reduce the tiles in global tile order, so every
// result is independent of launch geometry and of the GPU count.
// Roofline: HBM/L2-gather bound (K5-K7).
#include "common.cuh"

namespace ab2 {

namespace {

constexpr int kWarpsPerBlock = 8;
// Gradient CTAs are small so they fit beside the half-sweep kernels, which
// they run concurrently with (side stream, Solver::ncg_iteration).
constexpr int kGradWarps = 2;

template <int TPR>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int off = TPR / 2; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  return v;
}

template <int TPR, int V2>
__device__ __forceinline__ void load_row(const double* __restrict__ row, int ld, int sl,
                                         double2 (&v)[V2]) {
#pragma unroll
  for (int k = 0; k < V2; ++k) {
    const int e = 2 * (sl + TPR * k);
    v[k] = e < ld ? ldg2(row + e) : make_double2(0.0, 0.0);
  }
}

template <int V2>
__device__ __forceinline__ double dot2(const double2 (&a)[V2], const double2 (&b)[V2]) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < V2; ++k) s = fma(a[k].x, b[k].x, fma(a[k].y, b[k].y, s));
  return s;
}

// --------------------------------------------------------------- gradient --
struct GradArgs {
  const int64_t* ptr;
  const int* idx;
  const double* val;
  int row0;               // global index of local row 0 (rows of x / g)
  const double* xrows;    // x rows of this side (global row index)
  const double* xother;   // x rows of the other side
  int ld;
  double two_lambda;
  const int* seg_row;
  const int64_t* seg_beg;
  const int* seg_len;
  const int* seg_slot;
  int n_seg;
  double* g;              // g rows of this side (global row index)
  double* partial;        // [slot][ld]
};

template <int TPR, int V2>
__global__ void __launch_bounds__(kGradWarps * 32) k_gradient(GradArgs a) {
  const int lane = threadIdx.x & 31;
  const int seg = blockIdx.x * kGradWarps + (threadIdx.x >> 5);
  if (seg >= a.n_seg) return;
  constexpr int R = 32 / TPR;
  const int sg = lane / TPR, sl = lane % TPR;
  const int lr = a.seg_row[seg];
  const int64_t beg = a.seg_beg[seg];
  const int len = a.seg_len[seg];
  const int ld = a.ld;
  double2 xu[V2];
  load_row<TPR, V2>(a.xrows + static_cast<int64_t>(a.row0 + lr) * ld, ld, sl, xu);
  double2 acc[V2];
#pragma unroll
  for (int k = 0; k < V2; ++k) acc[k] = make_double2(0.0, 0.0);
  // two ratings per sub-group per trip: both gathers are in flight together
  // indices and values of the next trip are loaded one trip ahead
  int jn[2];
  double rn[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = sg + u * R;
    jn[u] = t < len ? a.idx[beg + t] : 0;
    rn[u] = t < len ? a.val[beg + t] : 0.0;
  }
  for (int t0 = 0; t0 < len; t0 += 2 * R) {
    int j[2];
    double r[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = t0 + sg + u * R;
      ok[u] = t < len;
      j[u] = jn[u];
      r[u] = rn[u];
      const int tn = t + 2 * R;
      jn[u] = tn < len ? a.idx[beg + tn] : 0;
      rn[u] = tn < len ? a.val[beg + tn] : 0.0;
    }
    double2 m[2][V2];
#pragma unroll
    for (int u = 0; u < 2; ++u) load_row<TPR, V2>(a.xother + static_cast<int64_t>(j[u]) * ld, ld, sl, m[u]);
    double s[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) s[u] = dot2<V2>(xu, m[u]);
#pragma unroll
    for (int u = 0; u < 2; ++u) s[u] = group_sum<TPR>(s[u]);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double e2 = ok[u] ? 2.0 * (s[u] - r[u]) : 0.0;
#pragma unroll
      for (int k = 0; k < V2; ++k) {
        acc[k].x = fma(e2, m[u][k].x, acc[k].x);
        acc[k].y = fma(e2, m[u][k].y, acc[k].y);
      }
    }
  }
#pragma unroll
  for (int off = 16; off >= TPR; off >>= 1)
#pragma unroll
    for (int k = 0; k < V2; ++k) {
      acc[k].x += __shfl_xor_sync(kFull, acc[k].x, off);
      acc[k].y += __shfl_xor_sync(kFull, acc[k].y, off);
    }
  if (sg != 0) return;
  const int slot = a.seg_slot[seg];
  if (slot < 0) {
    const double w = a.two_lambda * static_cast<double>(a.ptr[lr + 1] - a.ptr[lr]);
    double* out = a.g + static_cast<int64_t>(a.row0 + lr) * ld;
#pragma unroll
    for (int k = 0; k < V2; ++k) {
      const int e = 2 * (sl + TPR * k);
      if (e < ld)
        *reinterpret_cast<double2*>(out + e) =
            make_double2(fma(w, xu[k].x, acc[k].x), fma(w, xu[k].y, acc[k].y));
    }
  } else {
    double* out = a.partial + static_cast<int64_t>(slot) * ld;
#pragma unroll
    for (int k = 0; k < V2; ++k) {
      const int e = 2 * (sl + TPR * k);
      if (e < ld) *reinterpret_cast<double2*>(out + e) = acc[k];
    }
  }
}

// Multi-segment rows: g = 2*lambda*n*x + sum of segment partials in order.
__global__ void k_gradient_reduce(int n_multi, const int* __restrict__ m_row,
                                  const int* __restrict__ m_slot0, const int* __restrict__ m_nslot,
                                  const int64_t* __restrict__ ptr, int row0,
                                  const double* __restrict__ xrows, int ld, double two_lambda,
                                  const double* __restrict__ partial, double* __restrict__ g) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(n_multi) * ld) return;
  const int q = static_cast<int>(i / ld), e = static_cast<int>(i % ld);
  const int lr = m_row[q];
  double s = 0.0;
  for (int k = 0, slot = m_slot0[q]; k < m_nslot[q]; ++k, ++slot)
    s += partial[static_cast<int64_t>(slot) * ld + e];
  const double w = two_lambda * static_cast<double>(ptr[lr + 1] - ptr[lr]);
  const int64_t o = static_cast<int64_t>(row0 + lr) * ld + e;
  g[o] = fma(w, xrows[o], s);
}

// --------------------------------------------------------- quartic / loss --
struct QuartArgs {
  // CSR of this rank's users
  const int64_t* uptr;
  const int* uidx;
  const double* uval;
  int urow0, nurows;
  // CSC pointer of this rank's items (counts for the item regularisation)
  const int64_t* iptr;
  int irow0, nirows;
  const double* x;   // full flat vector (padded rows)
  const double* p;   // direction (quartic only)
  int ld;
  int n_u;           // global user count (item rows start at n_u)
  double lambda;
  int n_utiles;      // local user tiles (blocks [0, n_utiles) )
  int utile0, itile0;  // global tile index of this rank's first user / item tile
  int item_tile_base;  // global tile index where item tiles start
  dd* tiles;         // [global tile][NS]
};

// NS = 5 quartic coefficients, or 3 loss sums (sq, reg_u, reg_m).
template <int TPR, int V2, bool QUART>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_quartic(QuartArgs a) {
  constexpr int NS = QUART ? 5 : 3;
  constexpr int R = 32 / TPR;
  __shared__ dd sh[kWarpsPerBlock * NS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sg = lane / TPR, sl = lane % TPR;
  const int ld = a.ld;
  dd acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = {0.0, 0.0};
  const bool user_tile = static_cast<int>(blockIdx.x) < a.n_utiles;
  const int tile = user_tile ? blockIdx.x : blockIdx.x - a.n_utiles;
  const int lo = tile * kTileRows;
  if (user_tile) {
    const int hi = min(lo + kTileRows, a.nurows);
    // per-row regularisation (linesearch.cpp:68-73; ncg.cpp:57-61)
    for (int lr = lo + warp; lr < hi; lr += kWarpsPerBlock) {
      const int count = static_cast<int>(a.uptr[lr + 1] - a.uptr[lr]);
      const int64_t urow = static_cast<int64_t>(a.urow0 + lr) * ld;
      double2 xu[V2], pu[V2];
      load_row<TPR, V2>(a.x + urow, ld, sl, xu);
      const double xx = group_sum<TPR>(dot2<V2>(xu, xu));
      if constexpr (QUART) {
        load_row<TPR, V2>(a.p + urow, ld, sl, pu);
        const double xp = group_sum<TPR>(dot2<V2>(xu, pu));
        const double pp = group_sum<TPR>(dot2<V2>(pu, pu));
        if (lane == 0 && a.lambda > 0.0 && count > 0) {
          const double w = a.lambda * count;
          dd_add(acc[0], w * xx);
          dd_add(acc[1], 2.0 * w * xp);
          dd_add(acc[2], w * pp);
        }
      } else {
        if (lane == 0) dd_add(acc[1], static_cast<double>(count) * xx);
      }
    }
    // Ratings of the tile split evenly over the CTA's sub-groups (contiguous
    // chunks; a sub-group walks the users its chunk crosses), so a heavy user
    // no longer idles the other warps of its tile.
    constexpr int NG = kWarpsPerBlock * R;
    const int64_t T0 = a.uptr[lo], T1 = a.uptr[hi];
    const int64_t chunk = (T1 - T0 + NG - 1) / NG;
    int64_t t = T0 + static_cast<int64_t>(warp * R + sg) * chunk;
    const int64_t tend = min(T1, t + chunk);
    int u = lo, uhi = hi;
    if (t < tend) {
      while (uhi - u > 1) {
        const int mid = (u + uhi) >> 1;
        if (a.uptr[mid] <= t) u = mid; else uhi = mid;
      }
    }
    int64_t uend = t < tend ? a.uptr[u + 1] : 0;
    double2 xu[V2], pu[V2];
    load_row<TPR, V2>(a.x + static_cast<int64_t>(a.urow0 + u) * ld, ld, sl, xu);
    if constexpr (QUART) load_row<TPR, V2>(a.p + static_cast<int64_t>(a.urow0 + u) * ld, ld, sl, pu);
    // index and value of the next rating are loaded one trip ahead, so a
    // trip's row gathers never wait on their own index load
    int jn = t < tend ? a.uidx[t] : 0;
    double rn = t < tend ? a.uval[t] : 0.0;
    for (int64_t s = 0; s < chunk; ++s, ++t) {
      const bool ok = t < tend;
      if (ok && t >= uend) {
        do {
          ++u;
          uend = a.uptr[u + 1];
        } while (t >= uend);
        load_row<TPR, V2>(a.x + static_cast<int64_t>(a.urow0 + u) * ld, ld, sl, xu);
        if constexpr (QUART) load_row<TPR, V2>(a.p + static_cast<int64_t>(a.urow0 + u) * ld, ld, sl, pu);
      }
      const int j = jn;
      const double r = rn;
      jn = t + 1 < tend ? a.uidx[t + 1] : 0;
      rn = t + 1 < tend ? a.uval[t + 1] : 0.0;
      const int64_t mrow = static_cast<int64_t>(a.n_u + j) * ld;
      double2 xm[V2];
      load_row<TPR, V2>(a.x + mrow, ld, sl, xm);
      if constexpr (QUART) {
        double2 pm[V2];
        load_row<TPR, V2>(a.p + mrow, ld, sl, pm);
        const double sa = group_sum<TPR>(dot2<V2>(xu, xm));
        const double sb = group_sum<TPR>(dot2<V2>(xu, pm) + dot2<V2>(pu, xm));
        const double sd = group_sum<TPR>(dot2<V2>(pu, pm));
        if (ok && sl == 0) {
          // residual along the step: a - b*alpha - d*alpha^2 (linesearch.cpp:76-88)
          const double ra = r - sa;
          dd_add(acc[0], ra * ra);
          dd_add(acc[1], -2.0 * ra * sb);
          dd_add(acc[2], sb * sb - 2.0 * ra * sd);
          dd_add(acc[3], 2.0 * sb * sd);
          dd_add(acc[4], sd * sd);
        }
      } else {
        const double sa = group_sum<TPR>(dot2<V2>(xu, xm));
        if (ok && sl == 0) {
          const double ra = r - sa;
          dd_add(acc[0], ra * ra);
        }
      }
    }

  } else {
    // item regularisation rows (linesearch.cpp:90-103; ncg.cpp:62-66)
    const int hi = min(lo + kTileRows, a.nirows);
    for (int lr = lo + warp; lr < hi; lr += kWarpsPerBlock) {
      const int count = static_cast<int>(a.iptr[lr + 1] - a.iptr[lr]);
      const int64_t mrow = static_cast<int64_t>(a.n_u + a.irow0 + lr) * ld;
      double2 xm[V2];
      load_row<TPR, V2>(a.x + mrow, ld, sl, xm);
      const double xx = group_sum<TPR>(dot2<V2>(xm, xm));
      if constexpr (QUART) {
        double2 pm[V2];
        load_row<TPR, V2>(a.p + mrow, ld, sl, pm);
        const double xp = group_sum<TPR>(dot2<V2>(xm, pm));
        const double pp = group_sum<TPR>(dot2<V2>(pm, pm));
        if (lane == 0 && a.lambda > 0.0 && count > 0) {
          const double w = a.lambda * count;
          dd_add(acc[0], w * xx);
          dd_add(acc[1], 2.0 * w * xp);
          dd_add(acc[2], w * pp);
        }
      } else {
        if (lane == 0) dd_add(acc[2], static_cast<double>(count) * xx);
      }
    }
  }
  block_sum_dd<NS>(acc, sh);
  if (threadIdx.x == 0) {
    const int gt = user_tile ? a.utile0 + tile : a.item_tile_base + a.itile0 + tile;
#pragma unroll
    for (int k = 0; k < NS; ++k) a.tiles[static_cast<int64_t>(gt) * NS + k] = acc[k];
  }
}

// Sums all global tiles (fixed order) -> result.  Quartic: 5 coefficients;
// loss: sq + lambda*(reg_u + reg_m), or sq alone when lambda == 0.
template <int NS>
__global__ void __launch_bounds__(256) k_tiles_final(int n_tiles, const dd* __restrict__ tiles,
                                                     double lambda, double* __restrict__ out) {
  __shared__ dd sh[8 * NS];
  dd acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = {0.0, 0.0};
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
#pragma unroll
    for (int k = 0; k < NS; ++k) acc[k] = dd_plus(acc[k], tiles[static_cast<int64_t>(t) * NS + k]);
  block_sum_dd<NS>(acc, sh);
  if (threadIdx.x != 0) return;
  if constexpr (NS == 5) {
#pragma unroll
    for (int k = 0; k < 5; ++k) out[k] = dd_value(acc[k]);
  } else {
    const double sq = dd_value(acc[0]);
    out[0] = lambda == 0.0 ? sq : sq + lambda * (dd_value(acc[1]) + dd_value(acc[2]));
  }
}

// ------------------------------------------------------------- dispatch --
struct Geometry {
  int tpr, v2;
};

Geometry geometry_for(int n_f) {
  // TPR lanes per rating, V2 <= 4 double2 per lane: few shuffle rounds and
  // 32/TPR ratings in flight per warp step.
  const int pairs = row_stride(n_f) / 2;  // double2 per row
  int tpr = 1;
  while (tpr * 4 < pairs) tpr *= 2;
  if (tpr > 32) throw Error(ALSNCG_EUNSUPPORTED, "n_f too large for the residual kernels");
  const int v2 = (pairs + tpr - 1) / tpr;
  return {tpr, v2};
}

#define AB2_GEOM_V(T, G, MACRO)          \
  do {                                   \
    if (G.v2 == 1) { MACRO(T, 1); }      \
    else if (G.v2 == 2) { MACRO(T, 2); } \
    else if (G.v2 == 3) { MACRO(T, 3); } \
    else { MACRO(T, 4); }                \
  } while (0)

#define AB2_GEOM_DISPATCH(G, MACRO)                      \
  do {                                                   \
    if (G.tpr == 1) { AB2_GEOM_V(1, G, MACRO); }         \
    else if (G.tpr == 2) { AB2_GEOM_V(2, G, MACRO); }    \
    else if (G.tpr == 4) { AB2_GEOM_V(4, G, MACRO); }    \
    else if (G.tpr == 8) { AB2_GEOM_V(8, G, MACRO); }    \
    else if (G.tpr == 16) { AB2_GEOM_V(16, G, MACRO); }  \
    else { AB2_GEOM_V(32, G, MACRO); }                   \
  } while (0)

constexpr int kGradSeg = 2048;

}  // namespace

void launch_gradient(DevRatings& R, int n_f, const double* x, double lambda, double* g) {
  Ctx* ctx = R.ctx;
  const int ld = row_stride(n_f);
  const Geometry geo = geometry_for(n_f);
  for (int kind = 0; kind < 2; ++kind) {
    const View& v = R.view(kind);
    if (v.nrows == 0) continue;
    const SegPlan& P = R.plan(kind, kGradSeg);
    double* partial = P.n_slots > 0
                          ? static_cast<double*>(ctx->scratch(0, sizeof(double) * P.n_slots * ld))
                          : nullptr;
    GradArgs a;
    a.ptr = v.ptr;
    a.idx = v.idx;
    a.val = v.val;
    a.row0 = (kind == 0 ? 0 : R.n_u) + v.row0;
    a.xrows = x;
    a.xother = x + (kind == 0 ? static_cast<int64_t>(R.n_u) * ld : 0);
    a.ld = ld;
    a.two_lambda = 2.0 * lambda;
    a.seg_row = P.seg_row;
    a.seg_beg = P.seg_beg;
    a.seg_len = P.seg_len;
    a.seg_slot = P.seg_slot;
    a.n_seg = P.n_seg;
    a.g = g;
    a.partial = partial;
    const int blocks = (P.n_seg + kGradWarps - 1) / kGradWarps;
    const int tok = ctx->begin_launch(kind == 0 ? "gradient_users" : "gradient_items");
#define AB2_LAUNCH_GRAD(T, V) k_gradient<T, V><<<blocks, kGradWarps * 32, 0, ctx->stream>>>(a)
    AB2_GEOM_DISPATCH(geo, AB2_LAUNCH_GRAD);
#undef AB2_LAUNCH_GRAD
    ctx->end_launch(tok);
    if (P.n_multi > 0) {
      const int64_t n = static_cast<int64_t>(P.n_multi) * ld;
      const int t2 = ctx->begin_launch("gradient_reduce");
      k_gradient_reduce<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
          P.n_multi, P.m_row, P.m_slot0, P.m_nslot, v.ptr, a.row0, x, ld, 2.0 * lambda, partial, g);
      ctx->end_launch(t2);
    }
  }
}

namespace {

template <bool QUART>
void quartic_impl(DevRatings& R, int n_f, const double* x, const double* p, double lambda,
                  int slot) {
  Ctx* ctx = R.ctx;
  constexpr int NS = QUART ? 5 : 3;
  const int ld = row_stride(n_f);
  const Geometry geo = geometry_for(n_f);
  const int utiles_total = (R.n_u + kTileRows - 1) / kTileRows;
  const int itiles_total = (R.n_m + kTileRows - 1) / kTileRows;
  const int n_tiles = utiles_total + itiles_total;
  dd* tiles = static_cast<dd*>(ctx->scratch(1, sizeof(dd) * NS * std::max(n_tiles, 1)));
  QuartArgs a;
  a.uptr = R.users.ptr;
  a.uidx = R.users.idx;
  a.uval = R.users.val;
  a.urow0 = R.users.row0;
  a.nurows = R.users.nrows;
  a.iptr = R.items.ptr;
  a.irow0 = R.items.row0;
  a.nirows = R.items.nrows;
  a.x = x;
  a.p = p;
  a.ld = ld;
  a.n_u = R.n_u;
  a.lambda = lambda;
  a.n_utiles = (R.users.nrows + kTileRows - 1) / kTileRows;
  a.utile0 = R.users.row0 / kTileRows;
  a.itile0 = R.items.row0 / kTileRows;
  a.item_tile_base = utiles_total;
  a.tiles = tiles;
  const int n_itiles_local = (R.items.nrows + kTileRows - 1) / kTileRows;
  const int blocks = a.n_utiles + n_itiles_local;
  if (blocks > 0) {
    const int tok = ctx->begin_launch(QUART ? "quartic_tiles" : "loss_tiles");
#define AB2_LAUNCH_Q(T, V) k_quartic<T, V, QUART><<<blocks, kWarpsPerBlock * 32, 0, ctx->stream>>>(a)
    AB2_GEOM_DISPATCH(geo, AB2_LAUNCH_Q);
#undef AB2_LAUNCH_Q
    ctx->end_launch(tok);
  }
  if (ctx->world > 1) {
    // Replicate every rank's tile partials (tiles are the unit of sharding,
    // so the final reduction sees the same tiles in the same order as on 1 GPU).
    std::vector<int> ub(ctx->world + 1), ib(ctx->world + 1);
    for (int r = 0; r <= ctx->world; ++r) {
      ub[r] = (R.ub[r] + kTileRows - 1) / kTileRows;
      ib[r] = utiles_total + (R.mb[r] + kTileRows - 1) / kTileRows;
    }
    allgather_rows(ctx, reinterpret_cast<double*>(tiles), ub, 2 * NS);
    allgather_rows(ctx, reinterpret_cast<double*>(tiles), ib, 2 * NS);
  }
  const int tok = ctx->begin_launch(QUART ? "quartic_final" : "loss_final");
  k_tiles_final<NS><<<1, 256, 0, ctx->stream>>>(n_tiles, tiles, lambda, ctx->d_scalars + slot);
  ctx->end_launch(tok);
}

}  // namespace

void launch_quartic(DevRatings& R, int n_f, const double* x, const double* p, double lambda,
                    int slot) {
  quartic_impl<true>(R, n_f, x, p, lambda, slot);
}

void launch_loss(DevRatings& R, int n_f, const double* x, double lambda, int slot) {
  quartic_impl<false>(R, n_f, x, nullptr, lambda, slot);
}

}  // namespace ab2
