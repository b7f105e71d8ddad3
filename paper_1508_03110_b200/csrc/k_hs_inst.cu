// k_hs_inst.cu -- the Gram / solve kernels of one half-sweep, instantiated
// for a single block count NB = AB2_HS_NB per translation unit (the Makefile
// compiles this file once per NB in 1..26).  See k_halfsweep.cuh for the
// design notes and k_halfsweep.cu for the dispatcher and fallback.
#include "k_halfsweep.cuh"

#include <cstdlib>
#include <utility>

#ifndef AB2_HS_NB
#error "compile with -DAB2_HS_NB=<block count>"
#endif

namespace ab2 {
namespace hs {

namespace {



// One dynamic shared-memory array for every kernel of this file; all shared
// accesses index it with 32-bit offsets so they compile to LDS/STS.
extern __shared__ __align__(16) double g_smem[];

template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  [&]<int... Is>(std::integer_sequence<int, Is...>) { (f(std::integral_constant<int, Is>{}), ...); }(
      std::make_integer_sequence<int, N>{});
}

// Lower-triangle block pair p -> (row, col), row-major (p = I(I+1)/2 + J).
constexpr int tri_row(int p) {
  int i = 0;
  while ((i + 1) * (i + 2) / 2 <= p) ++i;
  return i;
}
constexpr int tri_col(int p) { return p - tri_row(p) * (tri_row(p) + 1) / 2; }


template <int NB, int GW>
struct HsCfg {
  static constexpr int P = NB * (NB + 1) / 2;     // lower-triangular block pairs
  static constexpr int Q = (P + GW - 1) / GW;     // pairs per warp
  static constexpr int LDS = NB * 8 + 4;          // stage row stride (bank-conflict free)
  static constexpr int CH = GW == 1 ? 16 : 32;    // ratings per stage
  static constexpr bool PACKED = NB > 16;
  static constexpr int MAXF = NB * 8;
  static constexpr int GPC = GW == 1 ? 4 : 1;     // groups per CTA
  static constexpr int THREADS = GW * 32 * GPC;
  static constexpr int GT = GW * 32;              // threads per group
  static constexpr int PART = GW * Q * 64;        // doubles per partial slot
};

template <int GW>
__device__ __forceinline__ void group_sync() {
  if constexpr (GW == 1)
    __syncwarp();
  else
    __syncthreads();
}

template <int NB, int GW>
__host__ __device__ constexpr size_t hs_group_doubles(int ld) {
  using C = HsCfg<NB, GW>;
  const size_t stage = static_cast<size_t>(2) * C::CH * C::LDS;
  const int lda = (ld + 1) | 1;
  const size_t mat = C::PACKED ? static_cast<size_t>(ld + 1) * (ld + 2) / 2
                               : static_cast<size_t>(ld + 1) * lda;
  const size_t body = ((stage > mat ? stage : mat) + 1) & ~static_cast<size_t>(1);
  return body + 2 * static_cast<size_t>(C::MAXF) + 2;  // + dinv[], w[], two stage mbarriers
}

template <bool PACKED>
__device__ __forceinline__ int midx(int i, int j, int lda) {
  if constexpr (PACKED)
    return i * (i + 1) / 2 + j;
  else
    return i * lda + j;
}

// Pair index p -> (I, J) with J <= I, row-major over the lower triangle.
__device__ __forceinline__ void pair_ij(int p, int& I, int& J) {
  int i = static_cast<int>((sqrtf(8.0f * p + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= p) ++i;
  while (i * (i + 1) / 2 > p) --i;
  I = i;
  J = p - i * (i + 1) / 2;
}

// Gram of the augmented rows over one segment, accumulated into acc.
// sb: offset (in doubles) of the group's region in g_smem.
template <int NB, int GW>
__device__ __forceinline__ void gram_segment(const HsArgs& a, int sb, int64_t beg, int len,
                                             int gtid, int warp, int lane,
                                             double (&acc)[HsCfg<NB, GW>::Q][2],
                                             const int (&pI)[HsCfg<NB, GW>::Q],
                                             const int (&pJ)[HsCfg<NB, GW>::Q]) {
  using C = HsCfg<NB, GW>;
  constexpr int BUF = C::CH * C::LDS;
  const int ld = a.ld;
  const int nch = ld >> 1;  // 16-byte chunks per source row
  const int padw = C::LDS - ld;
  // zero the pad columns (ld .. LDS) of both buffers once; column ld carries r
  // divisions by the run-time nch / padw as one multiply-high: x / d ==
  // umulhi(x, ceil(2^32 / d)) for x * d < 2^32 (d = 1 handled apart)
  const unsigned inv_nch = nch > 1 ? 0xffffffffu / static_cast<unsigned>(nch) + 1u : 0u;
  const unsigned inv_padw = padw > 1 ? 0xffffffffu / static_cast<unsigned>(padw) + 1u : 0u;
  for (int e = gtid; e < 2 * C::CH * padw; e += C::GT) {
    const int t = padw > 1 ? static_cast<int>(__umulhi(static_cast<unsigned>(e), inv_padw)) : e;  // row of both buffers
    const int c = e - t * padw;
    g_smem[sb + t * C::LDS + ld + c] = 0.0;
  }
  group_sync<GW>();
  // Each warp loads the stage's CH indices with one coalesced load (lane t
  // holds rating t) and hands them out by shuffle, so every cp.async of the
  // stage issues after a single index-load latency.
  // GW == 1 (the fused path): lane t gathers rating t's source row with one
  // TMA bulk copy completing on the stage's mbarrier -- one instruction per
  // rating instead of ld/2 16-byte cp.async chunks with their index math.
  // Measured (fused ms per iteration, config-1 matrix): f = 25 2.63 -> 2.37,
  // f = 30 2.73 -> 2.39, but f = 16 1.55 -> 1.62 and f = 10 1.37 -> 1.47 (rows
  // under ~150 bytes: the per-copy cost outweighs the chunk loop), hence NB >= 4.
  constexpr bool kTma = GW == 1 && NB >= 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(g_smem + sb + hs_group_doubles<NB, GW>(ld) - 2);
  if constexpr (kTma) {
    if (lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
      mbar_fence_init();
    }
  }
  // indices of stage s: loaded one stage before they are needed, so the
  // gathers of a stage never wait on their own index load
  auto load_idx = [&](int s) {
    const int base = s * C::CH;
    return (lane < C::CH && base + lane < len) ? a.idx[beg + base + lane] : 0;
  };
  auto issue = [&](int s, int bo, int jv) {
    const int base = s * C::CH;
    if constexpr (kTma) {
      const int nv = min(C::CH, len - base);
      if (lane < C::CH) {
        double* row = &g_smem[bo + lane * C::LDS];
        if (lane < nv) {
          cp_async8(row + ld, a.val + beg + base + lane);
        } else {
          for (int c = 0; c < ld; c += 2) *reinterpret_cast<double2*>(row + c) = make_double2(0.0, 0.0);
          row[ld] = 0.0;
        }
      }
      if (lane == 0) mbar_arrive_expect_tx(bars + (s & 1), static_cast<unsigned>(nv) * ld * 8);
      __syncwarp();
      if (lane < nv)
        tma_load_1d(&g_smem[bo + lane * C::LDS], a.src + static_cast<int64_t>(jv) * ld,
                    static_cast<unsigned>(ld) * 8, bars + (s & 1));
      return;
    }
    if (GW == 1 && nch <= 8) {
      // short rows: 4 or 8 lanes per rating, chunk = lane within the rating's
      // lanes -- shifts and masks only (the generic loop below spends ~70
      // instructions per trip on its (rating, chunk) arithmetic)
      const int sh = nch <= 4 ? 2 : 3;
      const int k = lane & ((1 << sh) - 1);
      for (int t = lane >> sh; t < C::CH; t += 32 >> sh) {
        const int j = __shfl_sync(kFull, jv, t);
        if (k < nch) {
          double* dst = &g_smem[bo + t * C::LDS + 2 * k];
          if (base + t < len)
            cp_async16(dst, a.src + static_cast<int64_t>(j) * ld + 2 * k);
          else
            *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
        }
      }
    } else
    for (int c0 = 0; c0 < C::CH * nch; c0 += C::GT) {
      const int c = c0 + gtid;
      const int t = min(nch > 1 ? static_cast<int>(__umulhi(static_cast<unsigned>(c), inv_nch)) : c, C::CH - 1);
      const int k = c - t * nch;
      const int j = __shfl_sync(kFull, jv, t);
      if (c < C::CH * nch) {
        double* dst = &g_smem[bo + t * C::LDS + 2 * k];
        if (base + t < len)
          cp_async16(dst, a.src + static_cast<int64_t>(j) * ld + 2 * k);
        else
          *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
      }
    }
    for (int t = gtid; t < C::CH; t += C::GT) {  // rating values: async too (no stall on the load)
      const int rt = base + t;
      double* dst = &g_smem[bo + t * C::LDS + ld];
      if (rt < len)
        cp_async8(dst, a.val + beg + rt);
      else
        *dst = 0.0;
    }
  };
  int aoff[C::Q], boff[C::Q];
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    aoff[q] = 8 * pI[q];
    boff[q] = 8 * pJ[q];
  }
  const int lofs = (lane & 3) * C::LDS + (lane >> 2);
  const int nst = (len + C::CH - 1) / C::CH;
  int jn = load_idx(0);
  if (nst > 0) issue(0, sb, jn);
  cp_async_commit();
  jn = load_idx(1);
  for (int s = 0; s < nst; ++s) {
    if (s + 1 < nst) {
      issue(s + 1, sb + ((s + 1) & 1) * BUF, jn);
      jn = load_idx(s + 2);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    if constexpr (kTma) mbar_wait(bars + (s & 1), (s >> 1) & 1);
    group_sync<GW>();
    const int bo = sb + (s & 1) * BUF + lofs;
    if constexpr (GW == 1) {
      // one warp owns every block pair: load each 8-row fragment of the
      // k-step once (the A fragment of block I is the B fragment of block I)
      // and issue all NB(NB+1)/2 DMMAs from registers -- NB shared loads per
      // k-step instead of two per DMMA (the fused path was shared-memory bound)
#pragma unroll 2
      for (int kk = 0; kk < C::CH / 4; ++kk) {
        const int base = bo + kk * 4 * C::LDS;
        double fr[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) fr[b] = g_smem[base + 8 * b];
        static_for<C::P>([&](auto pc) {
          constexpr int p = decltype(pc)::value;
          dmma884(acc[p][0], acc[p][1], fr[tri_row(p)], fr[tri_col(p)]);
        });
      }
    } else {
#pragma unroll 2
      for (int kk = 0; kk < C::CH / 4; ++kk) {
        const int base = bo + kk * 4 * C::LDS;
#pragma unroll
        for (int q = 0; q < C::Q; ++q) {
          if (q < C::Q - 1 || warp + q * GW < C::P) {
            const double av = g_smem[base + aoff[q]];
            const double bv = g_smem[base + boff[q]];
            dmma884(acc[q][0], acc[q][1], av, bv);
          }
        }
      }
    }
    group_sync<GW>();
  }
}

// Gram (in registers) -> shared matrix -> shifted elimination -> u.
template <int NB, int GW>
__device__ __forceinline__ void solve_row(const HsArgs& a, double* S, int lr, int count,
                                          int gtid, int warp, int lane,
                                          double (&acc)[HsCfg<NB, GW>::Q][2],
                                          const int (&pI)[HsCfg<NB, GW>::Q],
                                          const int (&pJ)[HsCfg<NB, GW>::Q]) {
  using C = HsCfg<NB, GW>;
  const int n_f = a.n_f, ld = a.ld;
  const int lda = (ld + 1) | 1;
  double* A = S;
  const size_t body = hs_group_doubles<NB, GW>(ld) - 2 * C::MAXF - 2;
  double* dinv = S + body;
  double* w = dinv + C::MAXF;
  double* out = a.out + static_cast<int64_t>(a.row0 + lr) * ld;

  group_sync<GW>();  // stage buffers are dead; A aliases them
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    if (q < C::Q - 1 || warp + q * GW < C::P) {
      const int i = 8 * pI[q] + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * pJ[q] + 2 * (lane & 3) + e;
        if (i <= ld && j <= i) A[midx<C::PACKED>(i, j, lda)] = acc[q][e];
      }
    }
  }
  const double shift = a.lambda * static_cast<double>(count);  // als.cpp:58
  group_sync<GW>();
  bool ok = shift > 0.0;
  if (ok) {
    for (int d = gtid; d < n_f; d += C::GT) A[midx<C::PACKED>(d, d, lda)] += shift;
    group_sync<GW>();
    // Right-looking symmetric elimination on rows {0..n_f-1} U {ld}.
    constexpr int TR = C::GT >= 128 ? 16 : 8;
    constexpr int TC = C::GT / TR;
    const int ti = gtid % TR, tj = gtid / TR;
    for (int k = 0; k < n_f; ++k) {
      const double d = A[midx<C::PACKED>(k, k, lda)];
      if (!(d > 0.0)) {  // Eigen LLT reports NumericalIssue on pivot <= 0
        ok = false;
        break;
      }
      const double invd = 1.0 / d;
      if (gtid == 0) dinv[k] = invd;
      const int nreg = n_f - 1 - k;
      for (int ii = ti; ii <= nreg; ii += TR) {
        const int i = ii < nreg ? k + 1 + ii : ld;
        const int jmax = ii < nreg ? i : n_f - 1;
        const double s = A[midx<C::PACKED>(i, k, lda)] * invd;
        for (int j = k + 1 + tj; j <= jmax; j += TC)
          A[midx<C::PACKED>(i, j, lda)] =
              fma(-s, A[midx<C::PACKED>(j, k, lda)], A[midx<C::PACKED>(i, j, lda)]);
      }
      group_sync<GW>();
    }
  }
  if (!ok) {
    if (gtid == 0) {
      const unsigned slot = atomicAdd(a.fb_count, 1u);
      a.fb_list[slot] = lr;
      atomicAdd(a.fb_total, 1u);
    }
    return;
  }
  // Back substitution (warp 0): u_k = (A[ld][k] - sum_{i>k} A[i][k] u_i) / d_k.
  if (warp == 0) {
    for (int i = lane; i < n_f; i += 32) w[i] = A[midx<C::PACKED>(ld, i, lda)];
    __syncwarp();
    for (int k = n_f - 1; k >= 0; --k) {
      const double u = w[k] * dinv[k];
      for (int i = lane; i < k; i += 32) w[i] = fma(-A[midx<C::PACKED>(k, i, lda)], u, w[i]);
      if (lane == 0) out[k] = u;
      __syncwarp();
    }
    if (lane == 0 && ld > n_f) out[n_f] = 0.0;
  }
}

template <int NB, int GW>
__device__ __forceinline__ void init_pairs(int warp, int (&pI)[HsCfg<NB, GW>::Q],
                                           int (&pJ)[HsCfg<NB, GW>::Q],
                                           double (&acc)[HsCfg<NB, GW>::Q][2]) {
  using C = HsCfg<NB, GW>;
#pragma unroll
  for (int q = 0; q < C::Q; ++q) {
    const int p = warp + q * GW;
    int I = 0, J = 0;
    if (p < C::P) pair_ij(p, I, J);
    pI[q] = I;
    pJ[q] = J;
    acc[q][0] = 0.0;
    acc[q][1] = 0.0;
  }
}

// Blocked elimination of one column's augmented Gram by a single warp
// (small ranks); defined after the k_hs_solve_ws helpers it reuses.
template <int NB>
__device__ void solve_row_blk(const HsArgs& a, double* S, int lr, int count, int lane,
                              double (&acc)[HsCfg<NB, 1>::Q][2]);

template <int NB, int GW>
__global__ void __launch_bounds__(HsCfg<NB, GW>::THREADS) k_hs_main(HsArgs a) {
  using C = HsCfg<NB, GW>;
  const int group = threadIdx.x / C::GT;
  const int gtid = threadIdx.x % C::GT;
  const int warp = gtid >> 5, lane = gtid & 31;
  const int seg = blockIdx.x * C::GPC + group;
  if (seg >= a.n_seg) return;  // uniform per group (GW==1 groups are warps)
  const int sbase = group * static_cast<int>(hs_group_doubles<NB, GW>(a.ld));
  double* S = g_smem + sbase;
  const int lr = a.seg_row[seg];
  const int len = a.seg_len[seg];
  const int slot = a.seg_slot[seg];
  double* out = a.out + static_cast<int64_t>(a.row0 + lr) * a.ld;
  if (len == 0) {  // zero-rating column stays zero (parallel.cpp:175)
    for (int k = gtid; k < a.ld; k += C::GT) out[k] = 0.0;
    return;
  }
  int pI[C::Q], pJ[C::Q];
  double acc[C::Q][2];
  init_pairs<NB, GW>(warp, pI, pJ, acc);
  gram_segment<NB, GW>(a, sbase, a.seg_beg[seg], len, gtid, warp, lane, acc, pI, pJ);
  if (slot >= 0) {
    double* P = a.partial + static_cast<int64_t>(slot) * C::PART;
#pragma unroll
    for (int q = 0; q < C::Q; ++q)
      *reinterpret_cast<double2*>(P + (warp * C::Q + q) * 64 + lane * 2) =
          make_double2(acc[q][0], acc[q][1]);
    return;
  }
  if constexpr (GW == 1)
    solve_row_blk<NB>(a, S, lr, len, lane, acc);
  else
    solve_row<NB, GW>(a, S, lr, len, gtid, warp, lane, acc, pI, pJ);
}

template <int NB, int GW>
__global__ void __launch_bounds__(HsCfg<NB, GW>::THREADS) k_hs_reduce(HsArgs a) {
  using C = HsCfg<NB, GW>;
  const int group = threadIdx.x / C::GT;
  const int gtid = threadIdx.x % C::GT;
  const int warp = gtid >> 5, lane = gtid & 31;
  const int m = blockIdx.x * C::GPC + group;
  if (m >= a.n_multi) return;
  double* S = g_smem + static_cast<size_t>(group) * hs_group_doubles<NB, GW>(a.ld);
  int pI[C::Q], pJ[C::Q];
  double acc[C::Q][2];
  init_pairs<NB, GW>(warp, pI, pJ, acc);
  const int slot0 = a.m_slot0[m], ns = a.m_nslot[m];
  for (int s = 0; s < ns; ++s) {  // segment order -> deterministic
    const double* P = a.partial + static_cast<int64_t>(slot0 + s) * C::PART;
#pragma unroll
    for (int q = 0; q < C::Q; ++q) {
      const double2 v = *reinterpret_cast<const double2*>(P + (warp * C::Q + q) * 64 + lane * 2);
      acc[q][0] += v.x;
      acc[q][1] += v.y;
    }
  }
  const int lr = a.m_row[m];
  const int count = static_cast<int>(a.ptr[lr + 1] - a.ptr[lr]);
  if constexpr (GW == 1)
    solve_row_blk<NB>(a, S, lr, count, lane, acc);
  else
    solve_row<NB, GW>(a, S, lr, count, gtid, warp, lane, acc, pI, pJ);
}

// ------------------------------------------------ split path (n_f >= 31) --
// Warp-specialised persistent Gram kernel (the split path's K1/K2).
//  * warp GR is the producer: for every stage of every segment this CTA owns
//    it waits for the ring slot to be released, writes the rating column and
//    zero tail rows, then gathers the stage's source rows with one TMA bulk
//    copy per rating (cp.async.bulk ... mbarrier::complete_tx);
//  * warps 0..GR-1 are consumers: warp r owns the compile-time contiguous
//    range of canonical block pairs [r*P/GR, (r+1)*P/GR), loads each needed
//    8-row fragment once per k-step and issues its DMMAs from registers; it
//    releases the slot with an mbarrier arrive.  No CTA-wide barrier in the
//    main loop; the producer runs ahead across segment boundaries.
constexpr int kWsCH = 32;

template <int NB>
struct WsShape {
  static constexpr int P = NB * (NB + 1) / 2;
  // ~12 block pairs per consumer warp, 2..8 consumers; 16 consumers (one CTA
  // per SM, a deeper ring) for NB > 20, where 8 warps would need > 255 registers
  static constexpr int GR = NB > 20 ? 16 : (P < 2 ? 1 : ((P + 11) / 12 < 2 ? 2 : ((P + 11) / 12 > 8 ? 8 : (P + 11) / 12)));
  static constexpr int LDS = NB * 8 + 4;
  static constexpr int BUF = kWsCH * LDS;
  // ring depth: 2 stages from NB = 6 up -- more CTAs per SM, more consumer
  // warps on the DMMA pipe (measured 15.6 -> 15.3 ms at n_f = 100, Gram
  // 4.87 -> 4.70 ms at n_f = 50); NB = 5 keeps 3 stages
  static constexpr int STAGES = NB > 20 ? 4 : (NB >= 6 ? 2 : 3);
  // NB > 20: the pairs are split over NPART = 2 CTAs (each gathers every
  // rating of the segment and accumulates half of the pairs): the 351 pair
  // accumulators of NB = 26 alone would fill an SM's register file.  Consumer
  // R of part h is virtual consumer h * GR + R.
  static constexpr int NPART = NB > 20 ? 2 : 1;
  // measured (Gram ms per iteration, config-1 matrix): NB = 16 28.3 -> 24.4 with 4,
  // NB = 26 218 -> 57 with 1; NB <= 13 is fastest fully unrolled
  static constexpr int KUNROLL = NB >= 17 ? 1 : (NB >= 14 ? 4 : kWsCH / 4);  // k-steps unrolled per stage
  static constexpr int p_begin(int r) { return r * P / (GR * NPART); }
  // Order in which block pairs are dealt to the consumers: bands of H block
  // rows, column by column inside a band.  H = 1 is the canonical row-major
  // order; H = 4 (NB > 20) makes a warp's ~22 consecutive pairs a ~4 x 6 tile,
  // so it needs ~10 fragments per k-step instead of ~23.
  static constexpr int H = NB > 20 ? 4 : 1;
  struct Order {
    int i[P], j[P];
  };
  static constexpr Order make_order() {
    Order o{};
    int c = 0;
    for (int b0 = 0; b0 < NB; b0 += H)
      for (int j = 0; j < (b0 + H < NB ? b0 + H : NB); ++j)
        for (int i = (b0 > j ? b0 : j); i < (b0 + H < NB ? b0 + H : NB); ++i) {
          o.i[c] = i;
          o.j[c] = j;
          ++c;
        }
    return o;
  }
  static constexpr Order order = make_order();
  static constexpr int row_of(int p) { return order.i[p]; }
  static constexpr int col_of(int p) { return order.j[p]; }
  static constexpr bool needs(int r, int b) {
    for (int p = p_begin(r); p < p_begin(r + 1); ++p)
      if (row_of(p) == b || col_of(p) == b) return true;
    return false;
  }
  static constexpr int max_pairs() {
    int m = 0;
    for (int r = 0; r < GR * NPART; ++r) m = p_begin(r + 1) - p_begin(r) > m ? p_begin(r + 1) - p_begin(r) : m;
    return m;
  }
  static constexpr int MAXP = max_pairs();
  static constexpr size_t smem_bytes() {
    return sizeof(double) * STAGES * BUF + 2 * STAGES * sizeof(uint64_t) + STAGES * sizeof(int);
  }
};

template <int NB, int R>
__device__ __forceinline__ void ws_kstep(int base, double (&acc)[WsShape<NB>::MAXP][2]) {
  using S = WsShape<NB>;
  constexpr int p0 = S::p_begin(R), p1 = S::p_begin(R + 1);
  double f[NB];
  static_for<NB>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    if constexpr (S::needs(R, b)) f[b] = g_smem[base + 8 * b];
  });
  static_for<p1 - p0>([&](auto pc) {
    constexpr int p = p0 + decltype(pc)::value;
    dmma884(acc[p - p0][0], acc[p - p0][1], f[S::row_of(p)], f[S::col_of(p)]);
  });
}

template <int NB, int R>
__device__ __forceinline__ void ws_consumer(const int* __restrict__ seg_len,
                                            const int* __restrict__ seg_slot, int n_seg,
                                            double* __restrict__ G, uint64_t* full,
                                            uint64_t* empty, const int* hdr, int lane) {
  using S = WsShape<NB>;
  constexpr int p0 = S::p_begin(R), np = S::p_begin(R + 1) - p0;
  const int lofs = (lane & 3) * S::LDS + (lane >> 2);
  int it = 0;
  for (;;) {
    // the first stage of every segment carries the segment id (the producer
    // takes segments from a global counter: dynamic, heavy-first balance)
    int buf = it % S::STAGES;
    mbar_wait(full + buf, (it / S::STAGES) & 1);
    const int seg = hdr[buf];
    if (seg >= n_seg) break;  // stop marker
    double acc[S::MAXP][2];
#pragma unroll
    for (int p = 0; p < S::MAXP; ++p) acc[p][0] = acc[p][1] = 0.0;
    const int nst = (seg_len[seg] + kWsCH - 1) / kWsCH;
    for (int s = 0; s < nst; ++s, ++it) {
      buf = it % S::STAGES;
      if (s > 0) mbar_wait(full + buf, (it / S::STAGES) & 1);
      const int bo = buf * S::BUF + lofs;
      // every consumer warp runs its own code: for large NB the fully
      // unrolled stage loops of an SM's warps overflow the instruction cache
      // (measured at NB = 26: 85 % of stall samples "no instruction")
#pragma unroll(S::KUNROLL)
      for (int kk = 0; kk < kWsCH / 4; ++kk) ws_kstep<NB, R>(bo + kk * 4 * S::LDS, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + buf);
    }
    double* out = G + static_cast<int64_t>(seg_slot[seg]) * S::P * 64 + lane * 2;
    static_for<np>([&](auto pc) {  // stored at the canonical pair index
      constexpr int p = decltype(pc)::value;
      constexpr int pc_idx = S::row_of(p0 + p) * (S::row_of(p0 + p) + 1) / 2 + S::col_of(p0 + p);
      __stcs(reinterpret_cast<double2*>(out + pc_idx * 64), make_double2(acc[p][0], acc[p][1]));
    });
  }
}

template <int NB>
__global__ void __launch_bounds__((WsShape<NB>::GR + 1) * 32)
    k_hs_gram_ws(HsArgs a, const int* __restrict__ seg_len, const int64_t* __restrict__ seg_beg,
                 const int* __restrict__ seg_slot, int n_seg, double* __restrict__ G,
                 int* __restrict__ next_seg) {
  using S = WsShape<NB>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = a.ld;
  const int part = S::NPART == 1 ? 0 : static_cast<int>(blockIdx.x) % S::NPART;
  next_seg += part;  // one segment counter per part
  uint64_t* full = reinterpret_cast<uint64_t*>(g_smem + S::STAGES * S::BUF);
  uint64_t* empty = full + S::STAGES;
  int* hdr = reinterpret_cast<int*>(empty + S::STAGES);  // segment id per stage
  // pad columns ld+1 .. LDS-1 stay zero for the whole kernel
  const int padw = S::LDS - ld - 1;
  for (int e = threadIdx.x; e < S::STAGES * kWsCH * padw; e += blockDim.x) {
    const int t = e / padw, c = e - t * padw;
    g_smem[t * S::LDS + ld + 1 + c] = 0.0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S::STAGES; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, S::GR);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == S::GR) {  // ---------------- producer
    int it = 0;
    for (;;) {
      int seg = 0;
      if (lane == 0) seg = atomicAdd(next_seg, 1);
      seg = __shfl_sync(kFull, seg, 0);
      if (seg >= n_seg) {  // publish a stop marker in the next stage
        const int buf = it % S::STAGES, use = it / S::STAGES;
        if (use > 0) mbar_wait(empty + buf, (use - 1) & 1);
        if (lane == 0) {
          hdr[buf] = n_seg;
          mbar_arrive(full + buf);
        }
        break;
      }
      const int len = seg_len[seg];
      const int64_t beg = seg_beg[seg];
      for (int base = 0; base < len; base += kWsCH, ++it) {
        const int buf = it % S::STAGES, use = it / S::STAGES;
        if (use > 0) mbar_wait(empty + buf, (use - 1) & 1);
        double* B = g_smem + buf * S::BUF;
        if (lane == 0 && base == 0) hdr[buf] = seg;
        const int nv = min(kWsCH, len - base);
        const int t = lane;  // kWsCH == 32: one rating per lane
        B[t * S::LDS + ld] = t < nv ? a.val[beg + base + t] : 0.0;
        if (t >= nv)
          for (int c = 0; c < ld; c += 2) *reinterpret_cast<double2*>(B + t * S::LDS + c) = make_double2(0.0, 0.0);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(full + buf, static_cast<unsigned>(nv) * ld * 8);
        if (t < nv)
          tma_load_1d(B + t * S::LDS, a.src + static_cast<int64_t>(a.idx[beg + base + t]) * ld,
                      static_cast<unsigned>(ld) * 8, full + buf);
      }
    }
    return;
  }
  // ------------------------------------------ consumers (compile-time band)
#define AB2_WS(R)                                                                              \
  if (warp == R && R < S::GR) {                                                                \
    if (part == 0)                                                                             \
      ws_consumer<NB, (R < S::GR ? R : 0)>(seg_len, seg_slot, n_seg, G, full, empty, hdr, lane); \
    else if constexpr (S::NPART > 1)                                                           \
      ws_consumer<NB, (R < S::GR ? S::GR + R : 0)>(seg_len, seg_slot, n_seg, G, full, empty, hdr, \
                                                   lane);                                      \
  }
  AB2_WS(0) AB2_WS(1) AB2_WS(2) AB2_WS(3) AB2_WS(4) AB2_WS(5) AB2_WS(6) AB2_WS(7)
  AB2_WS(8) AB2_WS(9) AB2_WS(10) AB2_WS(11) AB2_WS(12) AB2_WS(13) AB2_WS(14) AB2_WS(15)
#undef AB2_WS
}


__device__ __forceinline__ int pidx(int I, int J) { return I * (I + 1) / 2 + J; }
// Swizzled 8x8 block storage: element (r, c) at 8r + (c ^ 4*((r>>1)&1)); the
// C-fragment (16-byte) and A/B-fragment (8-byte) accesses are conflict-free.
__device__ __forceinline__ int swz(int r, int c) { return 8 * r + (c ^ (4 * ((r >> 1) & 1))); }


// ---------------------------------------------------------------------------
// K3 v2 (k_hs_solve_ws): warp-specialised persistent solve.  One CTA per SM,
// TEAMS teams of 1 + DW warps (DW = 3; 6 or 9 DMMA warps when only one column
// fits per SM), one column in flight per team (the team's
// shared block store holds that column's lower-triangular augmented Gram).
// The measured constraint (profiles/fp64_latency.txt): DFMA and DMMA share the
// FP64 datapath of an SM sub-partition (SMSP), and a dependent scalar FP64
// chain next to a warp streaming DMMAs waits ~87x its idle latency.  So the
// roles are split by SMSP (warp w runs on SMSP w % 4):
//   warp 4t   (SMSP 0, "pivot warp"): only the serial work -- the LDL^T
//             pivots of each 8x8 diagonal block, done as an in-register
//             Gauss-Jordan inverse (lanes hold the C-fragment layout), and
//             the back substitution;
//   warps 4t+1..4t+3 (SMSPs 1-3): only DMMA work -- per panel J
//             Y'_I = -M(I,J) D_J^-1 (the TRSM as two DMMAs per block), then
//             the trailing update M(I,K) += M(I,J) Y'_K^T; the owner of
//             (J+1,J+1) updates it first and signals the pivot warp
//             (lookahead), which inverts D_{J+1} while the rest of panel J's
//             update runs.
// Hand-offs use two mbarriers per team (pivot -> DMMA "inverse ready",
// DMMA -> pivot "next diagonal updated") and a 96-thread named barrier
// among the DMMA warps; no CTA-wide barrier after the prologue.  Blocked
// elimination with explicit diagonal inverses: forward
//   M(I,K) -= M(I,J) D_J^-1 M(K,J)^T  (I >= K > J, the rhs row included);
// back substitution x_J = D_J^-1 (w_J - sum_{I>J} M(I,J)^T x_I), one 8x8
// mat-vec per block instead of an 8-step chain.  A non-positive pivot (Eigen
// LLT's NumericalIssue) sends the column to the least-norm fallback.
template <int NB>
struct WsSolve {
  static constexpr int P = NB * (NB + 1) / 2;
  static constexpr int OFF_S = P * 64;           // Y'_I staging, NB blocks
  static constexpr int OFF_W = OFF_S + NB * 64;  // back-substitution vector, 8*NB
  static constexpr int TEAM_D = OFF_W + NB * 8;  // doubles per team
  static constexpr int TEAM_BYTES = TEAM_D * 8;
  static constexpr int FIT = (227 * 1024) / TEAM_BYTES;
  static constexpr int TEAMS = FIT > 6 ? 6 : (FIT < 1 ? 1 : FIT);
  // Ranks that fit a single column per SM get more DMMA warps per team (WPS
  // per SMSP 1-3); with two columns per SM three DMMA warps per team are still
  // (slightly) faster than six (f = 128: 21.4 vs 22.2 ms).  The CTA has TEAMS * WPS warps on every SMSP; on
  // SMSP 0 only one per team works (the pivot warp), the others exit after
  // the prologue.  Measured (solve ms per iteration, config-1 matrix), DMMA
  // warps per team 3 / 6 / 9 / 12: NB = 20 78 / 50 / 55 / 58, NB = 26
  // 151 / 98 / 82 / 85 -- more warps shorten the update phases but lengthen
  // the two named barriers of every panel.
  static constexpr int WPS = TEAMS == 1 ? (NB >= 24 ? 3 : 2) : 1;
  static constexpr int DW = 3 * WPS;            // DMMA warps per team
  static constexpr int ACT = (1 + DW) * 32;     // working threads per team
  static constexpr int THREADS = TEAMS * WPS * 128;
};

// Compile-time work lists of DMMA warp d for panel J.
template <int NB>
struct WsList {
  int n;
  int I[NB * (NB + 1) / 2];
  int K[NB * (NB + 1) / 2];
  // Y' blocks: I in (J, NB) round-robin, I = J+1 on warp 0 (needed first)
  static constexpr WsList y(int J, int d, int DW) {
    WsList l{};
    for (int i = J + 1; i < NB; ++i)
      if ((i - J - 1) % DW == d) {
        l.I[l.n] = i;
        l.K[l.n] = J;
        ++l.n;
      }
    return l;
  }
  // update blocks (I,K), J < K <= I < NB: (J+1,J+1) is position 0 (warp 0,
  // first); the rest in column-major order, split evenly over the 3 warps
  static constexpr WsList u(int J, int d, int DW) {
    WsList l{};
    const int total = (NB - 1 - J) * (NB - J) / 2;
    int pos = 0;
    for (int k = J + 1; k < NB; ++k)
      for (int i = k; i < NB; ++i) {
        const int p = (i == J + 1 && k == J + 1) ? 0 : ++pos;
        if (p * DW / total == d) {
          l.I[l.n] = i;
          l.K[l.n] = k;
          ++l.n;
        }
      }
    // (J+1,J+1) first within warp 0's list
    for (int e = 1; e < l.n; ++e)
      if (l.I[e] == J + 1 && l.K[e] == J + 1) {
        const int ti = l.I[e], tk = l.K[e];
        for (int f = e; f > 0; --f) {
          l.I[f] = l.I[f - 1];
          l.K[f] = l.K[f - 1];
        }
        l.I[0] = ti;
        l.K[0] = tk;
      }
    return l;
  }
};

template <int NB, int J, int d, int DW>
struct WsY {
  static constexpr WsList<NB> v = WsList<NB>::y(J, d, DW);
};
template <int NB, int J, int d, int DW>
struct WsU {
  static constexpr WsList<NB> v = WsList<NB>::u(J, d, DW);
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// Pivot warp, panel J: Gauss-Jordan inverse of the (Schur-complemented)
// diagonal block restricted to its nv valid pivots; writes -D^-1 (zero
// outside nv x nv) over the block.  When the rhs row lives in this block
// (J == IR) its first nv entries are saved to W first.  Returns false on a
// non-positive (or NaN) pivot; the result is warp-uniform.
template <int NB, int J, bool FULL>
__device__ __forceinline__ bool ws_factor(double* M, int n_f, int IR, int rl, int lane) {
  double* D = M + pidx(J, J) * 64;
  double* W = M + WsSolve<NB>::OFF_W;
  const int r = lane >> 2, q = lane & 3;
  const int c0 = 2 * q, c1 = 2 * q + 1;
  const double2 v = *reinterpret_cast<const double2*>(D + swz(r, c0));
  double a0 = v.x, a1 = v.y;
  const int nv = FULL ? 8 : min(8, n_f - 8 * J);  // FULL: all 8 pivots valid (no per-pivot branch)
  if (J == IR && r == rl) {
    W[8 * J + c0] = c0 < nv ? a0 : 0.0;
    W[8 * J + c1] = c1 < nv ? a1 : 0.0;
  }
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (FULL || k < nv) {
      const double p = __shfl_sync(kFull, (k & 1) ? a1 : a0, 4 * k + (k >> 1));
      ok = ok && (p > 0.0);
      const double ip = fast_rcp(p);
      const double rk0 = __shfl_sync(kFull, a0, 4 * k + q) * ip;  // scaled row k at my columns
      const double rk1 = __shfl_sync(kFull, a1, 4 * k + q) * ip;
      const double ck = __shfl_sync(kFull, (k & 1) ? a1 : a0, 4 * r + (k >> 1));  // my row, column k
      if (r == k) {
        a0 = c0 == k ? ip : rk0;
        a1 = c1 == k ? ip : rk1;
      } else {
        a0 = c0 == k ? -ck * ip : fma(-ck, rk0, a0);
        a1 = c1 == k ? -ck * ip : fma(-ck, rk1, a1);
      }
    }
  }
  if (r >= nv) a0 = a1 = 0.0;
  if (c0 >= nv) a0 = 0.0;
  if (c1 >= nv) a1 = 0.0;
  __syncwarp();
  *reinterpret_cast<double2*>(D + swz(r, c0)) = make_double2(-a0, -a1);
  return ok;
}

// DMMA warp d, panel J, step 1: Y'_I = M(I,J) (-D_J^-1) into the staging area.
template <int NB, int J, int d, int DW = 3>
__device__ __forceinline__ void ws_y(double* M, int r, int q) {
  using L = WsY<NB, J, d, DW>;
  if constexpr (L::v.n > 0) {
    const double* ND = M + pidx(J, J) * 64;
    const double b0 = ND[swz(q, r)], b1 = ND[swz(4 + q, r)];  // B[k][n] = ND[k][n]
    static_for<L::v.n>([&](auto ic) {
      constexpr int I = L::v.I[decltype(ic)::value];
      const double* A = M + pidx(I, J) * 64;
      double y0 = 0.0, y1 = 0.0;
      dmma884(y0, y1, A[swz(r, q)], b0);
      dmma884(y0, y1, A[swz(r, 4 + q)], b1);
      *reinterpret_cast<double2*>(M + WsSolve<NB>::OFF_S + I * 64 + swz(r, 2 * q)) = make_double2(y0, y1);
    });
  }
}

// DMMA warp d, panel J, step 2: M(I,K) += M(I,J) Y'_K^T, four blocks per
// batch (all loads first).  Warp 0 starts with (J+1,J+1) and then signals
// the pivot warp through `upd`.
template <int NB, int J, int d, int DW = 3>
__device__ __forceinline__ void ws_update(double* M, int r, int q, int lane, int KP, uint64_t* upd) {
  using L = WsU<NB, J, d, DW>;
  constexpr int OS = WsSolve<NB>::OFF_S;
  const int oc = swz(r, 2 * q), oa0 = swz(r, q), oa1 = swz(r, 4 + q);
  auto one = [&](auto ic) {
    constexpr int I = L::v.I[decltype(ic)::value], K = L::v.K[decltype(ic)::value];
    double2 c = *reinterpret_cast<const double2*>(M + pidx(I, K) * 64 + oc);
    dmma884(c.x, c.y, M[pidx(I, J) * 64 + oa0], M[OS + K * 64 + oa0]);
    dmma884(c.x, c.y, M[pidx(I, J) * 64 + oa1], M[OS + K * 64 + oa1]);
    *reinterpret_cast<double2*>(M + pidx(I, K) * 64 + oc) = c;
  };
  constexpr int first = (d == 0 && L::v.n > 0) ? 1 : 0;
  if constexpr (first) {
    one(std::integral_constant<int, 0>{});
    __syncwarp();
    if (upd != nullptr && J + 1 < KP && lane == 0) mbar_arrive(upd);
  }
  constexpr int G = 4;
  constexpr int rest = L::v.n - first;
  static_for<(rest + G - 1) / G>([&](auto gc) {
    constexpr int g0 = first + decltype(gc)::value * G;
    double2 c[G];
    double xa[G][2], sb[G][2];
    static_for<G>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if constexpr (g0 + i < L::v.n) {
        constexpr int I = L::v.I[g0 + i], K = L::v.K[g0 + i];
        c[i] = *reinterpret_cast<const double2*>(M + pidx(I, K) * 64 + oc);
        xa[i][0] = M[pidx(I, J) * 64 + oa0];
        xa[i][1] = M[pidx(I, J) * 64 + oa1];
        sb[i][0] = M[OS + K * 64 + oa0];
        sb[i][1] = M[OS + K * 64 + oa1];
      }
    });
    static_for<G>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if constexpr (g0 + i < L::v.n) dmma884(c[i].x, c[i].y, xa[i][0], sb[i][0]);
    });
    static_for<G>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if constexpr (g0 + i < L::v.n) dmma884(c[i].x, c[i].y, xa[i][1], sb[i][1]);
    });
    static_for<G>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if constexpr (g0 + i < L::v.n) {
        constexpr int I = L::v.I[g0 + i], K = L::v.K[g0 + i];
        *reinterpret_cast<double2*>(M + pidx(I, K) * 64 + oc) = c[i];
      }
    });
  });
}

// Back substitution by one warp after the blocked elimination:
// x_J = D_J^-1 (w_J - sum_{I>J} M(I,J)^T x_I), w the final rhs row.
template <int NB>
__device__ __forceinline__ void ws_backsub(double* M, int n_f, int KP, int IR, int rl, int lane, double* out) {
  const double* Wv = M + WsSolve<NB>::OFF_W;
  // w lives in registers: lane l owns entries l + 32u.  Per block J:
  // gather w_J by shuffle, x_J[n] = -(ND_J w_J)[n] in lane n (two 4-term
  // chains), broadcast x_J, fold it into the owned entries of blocks K < J.
  constexpr int NWR = (8 * NB + 31) / 32;
  double wr[NWR];
#pragma unroll
  for (int u = 0; u < NWR; ++u) {
    const int i = lane + 32 * u;
    const int K = i >> 3;
    wr[u] = i < 8 * KP ? (K < IR ? M[pidx(IR, K) * 64 + swz(rl, i & 7)] : Wv[i]) : 0.0;
  }
  // The block loop is unrolled and x is stored after it: a store of x_J to
  // `out` inside the loop (which the compiler must assume may alias the block
  // store) pins the next block's loads behind the dependent chain.
  double xk[NB];  // x_J[lane & 7], kept by every lane
  static_for<NB>([&](auto Jc) {
    constexpr int J = NB - 1 - decltype(Jc)::value;
    xk[J] = 0.0;
    if (J >= KP) return;
    constexpr int u = J >> 2;  // entries 8J..8J+7 sit in register u of lanes (8J & 31)..+7
    const double wsrc = wr[u];
    const double* ND = M + pidx(J, J) * 64;
    const int n = lane & 7;
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      t0 = fma(ND[swz(n, cc)], __shfl_sync(kFull, wsrc, ((8 * J) & 31) + cc), t0);
      t1 = fma(ND[swz(n, 4 + cc)], __shfl_sync(kFull, wsrc, ((8 * J) & 31) + 4 + cc), t1);
    }
    const double x = -(t0 + t1);
    xk[J] = x;
    double xr[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) xr[rr] = __shfl_sync(kFull, x, rr);
#pragma unroll
    for (int v = 0; v < NWR; ++v) {
      const int i = lane + 32 * v;
      if (32 * v < 8 * J && i < 8 * J) {
        const double* blk = M + pidx(J, i >> 3) * 64;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          a0 = fma(blk[swz(rr, i & 7)], xr[rr], a0);
          a1 = fma(blk[swz(4 + rr, i & 7)], xr[4 + rr], a1);
        }
        wr[v] -= a0 + a1;
      }
    }
  });
  if (lane < 8) {
#pragma unroll
    for (int J = 0; J < NB; ++J)
      if (J < KP && 8 * J + lane < n_f) out[8 * J + lane] = xk[J];
  }
}

template <int NB>
__device__ void solve_row_blk(const HsArgs& a, double* S, int lr, int count, int lane,
                              double (&acc)[HsCfg<NB, 1>::Q][2]) {
  // the warp owns every block (GW == 1): acc[p] is block p = I(I+1)/2 + J
  const int n_f = a.n_f, ld = a.ld;
  const int r = lane >> 2, q = lane & 3;
  double* out = a.out + static_cast<int64_t>(a.row0 + lr) * ld;
  __syncwarp();  // the stage buffers are dead; the block store aliases them
#pragma unroll
  for (int p = 0; p < HsCfg<NB, 1>::P; ++p)
    *reinterpret_cast<double2*>(S + p * 64 + swz(r, 2 * q)) = make_double2(acc[p][0], acc[p][1]);
  const double shift = a.lambda * static_cast<double>(count);  // als.cpp:58
  bool ok = shift > 0.0;
  if (ok) {
    __syncwarp();
    for (int k = lane; k < n_f; k += 32) S[pidx(k >> 3, k >> 3) * 64 + swz(k & 7, k & 7)] += shift;
    __syncwarp();
    const int KP = (n_f + 7) >> 3, IR = ld >> 3, rl = ld & 7;
    static_for<NB>([&](auto Jc) {
      constexpr int J = decltype(Jc)::value;
      if (!ok || J >= KP) return;
      ok = 8 * (J + 1) <= n_f ? ws_factor<NB, J, true>(S, n_f, IR, rl, lane)
                              : ws_factor<NB, J, false>(S, n_f, IR, rl, lane);
      __syncwarp();
      if constexpr (J + 1 < NB) {
        if (ok) {
          ws_y<NB, J, 0, 1>(S, r, q);
          __syncwarp();
          ws_update<NB, J, 0, 1>(S, r, q, lane, KP, nullptr);
          __syncwarp();
        }
      }
    });
    if (ok) {
      ws_backsub<NB>(S, n_f, KP, IR, rl, lane, out);
      for (int k = n_f + lane; k < ld; k += 32) out[k] = 0.0;
      return;
    }
  }
  if (lane == 0) {  // lambda*n == 0 or a non-positive pivot: least-norm fallback
    const unsigned slot = atomicAdd(a.fb_count, 1u);
    a.fb_list[slot] = lr;
    atomicAdd(a.fb_total, 1u);
  }
}

template <int NB, int d, int DW>
__device__ __forceinline__ void ws_dmma_role(double* M, int KP, int team, int lane, uint64_t* diag,
                                             uint64_t* upd, unsigned& ph_diag, volatile int* fail,
                                             unsigned long long* probe = nullptr) {
  const int r = lane >> 2, q = lane & 3;
  bool stop = false;
  static_for<NB>([&](auto Jc) {
    constexpr int J = decltype(Jc)::value;
    if (stop || J >= KP) return;
    mbar_wait(diag, ph_diag & 1);
    ++ph_diag;
    if (*fail) {
      stop = true;
      return;
    }
    if constexpr (J + 1 < NB) {
      ws_y<NB, J, d, DW>(M, r, q);
      named_bar(1 + team, 32 * DW);
      ws_update<NB, J, d, DW>(M, r, q, lane, KP, upd);
      named_bar(1 + team, 32 * DW);
      if (probe && lane == 0 && J < 19) probe[4 + 3 * J] = clock64();
    }
  });
}

#ifdef AB2_WS_PROBE
// development probe: phase clocks of the first column of team 0 in CTAs 0..63
__device__ unsigned long long g_ws_probe[64][64];
#define WS_PROBE(slot) \
  do { if (probe_on && lane == 0) g_ws_probe[blockIdx.x][slot] = clock64(); } while (0)
#define WS_PROBE_V(slot, v) \
  do { if (probe_on && lane == 0) g_ws_probe[blockIdx.x][slot] = (v); } while (0)
#else
#define WS_PROBE(slot) do {} while (0)
#define WS_PROBE_V(slot, v) do {} while (0)
#endif

template <int NB>
__global__ void __launch_bounds__(WsSolve<NB>::THREADS, 1)
    k_hs_solve_ws(HsArgs a, SolveArgs s, int* __restrict__ next_col) {
  using W = WsSolve<NB>;
  constexpr int T = W::TEAMS;
  __shared__ uint64_t bars[T][2];  // [0] inverse ready (pivot -> DMMA), [1] next diagonal updated
  __shared__ int team_col[T];
  __shared__ int team_fail[T];
  constexpr int WPS = W::WPS, DW = W::DW, NW = T * WPS * 4;
  __shared__ int slot_of[NW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Roles by SM sub-partition: the warp's hardware slot (%warpid) decides its
  // SMSP (slot % 4), not its index in the CTA (measured: CTA warp 0 lands on
  // slots 1..3).  When the CTA's warps are spread evenly (T per SMSP), the
  // warps on SMSP 0 become the pivot warps and team t takes the t-th warp of
  // every SMSP; otherwise fall back to index order.
  {
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    if (lane == 0) slot_of[warp] = static_cast<int>(wid);
  }
  __syncthreads();
  // role: 0 = pivot warp, 1..DW = DMMA warp role-1, > DW = idle (SMSP 0 spares)
  int team = warp / (WPS * 4), role = warp % (WPS * 4);
  {
    int cnt[4] = {0, 0, 0, 0}, my_s = 0, my_rank = 0;
    for (int w = 0; w < NW; ++w) {
      const int sp = slot_of[w] & 3;
      if (w == warp) {
        my_s = sp;
        my_rank = cnt[sp];
      }
      ++cnt[sp];
    }
    if (cnt[0] == T * WPS && cnt[1] == T * WPS && cnt[2] == T * WPS && cnt[3] == T * WPS) {
      team = my_rank % T;
      const int sub = my_rank / T;
      role = my_s == 0 ? (sub == 0 ? 0 : DW + 1) : 1 + (my_s - 1) * WPS + sub;
    }
  }
  const int ttid = role * 32 + lane;
  double* M = g_smem + static_cast<size_t>(team) * W::TEAM_D;
  double* Wv = M + W::OFF_W;
  const int n_f = a.n_f, ld = a.ld;
  const int KP = (n_f + 7) >> 3;
  const int IR = ld >> 3, rl = ld & 7;
  const int r = lane >> 2, q = lane & 3;
  const int team_bar = 1 + T + team;
  if (ttid == 0) {
    mbar_init(&bars[team][0], 1);
    mbar_init(&bars[team][1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (role > DW) return;  // spare warp on the pivot SMSP: takes no barrier below
  unsigned ph_diag = 0, ph_upd = 0;
#ifdef AB2_WS_PROBE
  bool probe_on = team == 0 && blockIdx.x < 64;
  if (probe_on && lane == 0) {
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    g_ws_probe[blockIdx.x][62 + (role > 0)] = wid;  // SMSP = warpid % 4
  }
#endif
  for (;;) {
    named_bar(team_bar, W::ACT);  // the previous column's smem reads are done
    if (ttid == 0) {
      team_col[team] = atomicAdd(next_col, 1);
      team_fail[team] = 0;
    }
    named_bar(team_bar, W::ACT);
    const int c = team_col[team];
    if (c >= s.nrows) break;
    if (role == 0) WS_PROBE(0);
    const int lr = s.row0 + c;
    double* out = a.out + static_cast<int64_t>(a.row0 + lr) * ld;
    const int count = static_cast<int>(a.ptr[lr + 1] - a.ptr[lr]);
    if (count == 0) {  // parallel.cpp:175 -- empty column stays zero
      for (int k = ttid; k < ld; k += W::ACT) out[k] = 0.0;
      continue;
    }
    const double shift = a.lambda * static_cast<double>(count);  // als.cpp:58
    if (!(shift > 0.0)) {
      if (ttid == 0) {
        a.fb_list[atomicAdd(a.fb_count, 1u)] = lr;
        atomicAdd(a.fb_total, 1u);
      }
      continue;
    }
    {  // heavy rows were folded into their first slot by k_hs_slot_reduce
      const double* base = s.G + static_cast<int64_t>(s.row_slot0[lr]) * W::P * 64 + lane * 2;
      for (int p = role; p < W::P; p += 1 + DW) cp_async16(M + p * 64 + swz(r, 2 * q), base + p * 64);
      cp_async_commit();
      cp_async_wait<0>();
    }
    named_bar(team_bar, W::ACT);
    if (role == 0) WS_PROBE(1);
    if (role == 0) {
      for (int k = lane; k < n_f; k += 32) M[pidx(k >> 3, k >> 3) * 64 + swz(k & 7, k & 7)] += shift;  // als.cpp:58-59
      __syncwarp();
      bool ok = true;
      static_for<NB>([&](auto Jc) {
        constexpr int J = decltype(Jc)::value;
        if (!ok || J >= KP) return;
        if (J > 0) {
          mbar_wait(&bars[team][1], ph_upd & 1);
          ++ph_upd;
        }
        if (J < 19) WS_PROBE(2 + 3 * J);
        ok = 8 * (J + 1) <= n_f ? ws_factor<NB, J, true>(M, n_f, IR, rl, lane)
                                : ws_factor<NB, J, false>(M, n_f, IR, rl, lane);
        if (J < 19) WS_PROBE(3 + 3 * J);
        if (!ok && lane == 0) team_fail[team] = 1;
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[team][0]);
        ++ph_diag;
      });
    } else {
      static_for<DW>([&](auto dc) {
        constexpr int d = decltype(dc)::value;
        if (role != 1 + d) return;
#ifdef AB2_WS_PROBE
        ws_dmma_role<NB, d, DW>(M, KP, team, lane, &bars[team][0], &bars[team][1], ph_diag, &team_fail[team],
                                d == 0 && probe_on ? &g_ws_probe[blockIdx.x][0] : nullptr);
#else
        ws_dmma_role<NB, d, DW>(M, KP, team, lane, &bars[team][0], &bars[team][1], ph_diag, &team_fail[team]);
#endif
      });
    }
    named_bar(team_bar, W::ACT);  // every panel of this column is done
    if (role == 0) WS_PROBE(60);
    if (team_fail[team]) {
      if (ttid == 0) {
        a.fb_list[atomicAdd(a.fb_count, 1u)] = lr;
        atomicAdd(a.fb_total, 1u);
      }
      continue;
    }
#ifdef AB2_WS_PROBE
    if (role != 0) probe_on = false;
#endif
    if (role != 0) continue;
    ws_backsub<NB>(M, n_f, KP, IR, rl, lane, out);
    for (int k = n_f + lane; k < ld; k += 32) out[k] = 0.0;
    WS_PROBE(61);
#ifdef AB2_WS_PROBE
    probe_on = false;
#endif
  }
}

// K3 for small ranks (k_hs_solve_1w): one warp per column, the same blocked
// elimination run by that warp alone (diagonal inverse, DMMA TRSM and update,
// shuffle back substitution) with no inter-warp hand-off.  A column's block
// store is small here (18 KB at n_f = 50), so 10-16 columns are in flight per
// SM instead of the 6 team columns of k_hs_solve_ws, whose per-panel
// hand-offs (~4.5 k cycles per panel whatever NB is) dominate when the panels
// carry only a handful of DMMAs.
template <int NB>
struct OneWarpSolve {
  static constexpr int COL_D = WsSolve<NB>::TEAM_D;
  static constexpr int FIT = (227 * 1024) / (COL_D * 8);
  static constexpr int WARPS = FIT > 16 ? 16 : (FIT < 1 ? 1 : FIT);
  static constexpr int THREADS = WARPS * 32;
  static constexpr size_t smem_bytes() { return size_t(WARPS) * COL_D * 8; }
};

template <int NB>
__global__ void __launch_bounds__(OneWarpSolve<NB>::THREADS, 1)
    k_hs_solve_1w(HsArgs a, SolveArgs s, int* __restrict__ next_col) {
  using W = WsSolve<NB>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* M = g_smem + static_cast<size_t>(warp) * W::TEAM_D;
  const int n_f = a.n_f, ld = a.ld;
  const int KP = (n_f + 7) >> 3;
  const int IR = ld >> 3, rl = ld & 7;
  const int r = lane >> 2, q = lane & 3;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(next_col, 1);
    c = __shfl_sync(kFull, c, 0);
    if (c >= s.nrows) break;
    const int lr = s.row0 + c;
    double* out = a.out + static_cast<int64_t>(a.row0 + lr) * ld;
    const int count = static_cast<int>(a.ptr[lr + 1] - a.ptr[lr]);
    if (count == 0) {  // parallel.cpp:175 -- empty column stays zero
      for (int k = lane; k < ld; k += 32) out[k] = 0.0;
      continue;
    }
    const double shift = a.lambda * static_cast<double>(count);  // als.cpp:58
    bool ok = shift > 0.0;
    if (ok) {
      __syncwarp();  // the previous column's reads of the block store are done
      const double* base = s.G + static_cast<int64_t>(s.row_slot0[lr]) * W::P * 64 + lane * 2;
#pragma unroll 4
      for (int p = 0; p < W::P; ++p) cp_async16(M + p * 64 + swz(r, 2 * q), base + p * 64);
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      for (int k = lane; k < n_f; k += 32) M[pidx(k >> 3, k >> 3) * 64 + swz(k & 7, k & 7)] += shift;  // als.cpp:58-59
      __syncwarp();
      static_for<NB>([&](auto Jc) {
        constexpr int J = decltype(Jc)::value;
        if (!ok || J >= KP) return;
        ok = 8 * (J + 1) <= n_f ? ws_factor<NB, J, true>(M, n_f, IR, rl, lane)
                                : ws_factor<NB, J, false>(M, n_f, IR, rl, lane);
        __syncwarp();
        if constexpr (J + 1 < NB) {
          if (ok) {
            ws_y<NB, J, 0, 1>(M, r, q);
            __syncwarp();
            ws_update<NB, J, 0, 1>(M, r, q, lane, KP, nullptr);
            __syncwarp();
          }
        }
      });
      if (ok) {
        ws_backsub<NB>(M, n_f, KP, IR, rl, lane, out);
        for (int k = n_f + lane; k < ld; k += 32) out[k] = 0.0;
        continue;
      }
    }
    if (lane == 0) {  // lambda*n == 0 or a non-positive pivot: least-norm fallback
      a.fb_list[atomicAdd(a.fb_count, 1u)] = lr;
      atomicAdd(a.fb_total, 1u);
    }
  }
}

// Heavy rows: fold a row's partial Gram slots into its first slot, in slot
// order (deterministic; every load of a thread is independent, so all slots
// of a row are in flight at once).  One thread per double2 of one row.
__global__ void __launch_bounds__(256) k_hs_slot_reduce(const int* __restrict__ rows, int n_rows,
                                                        const int* __restrict__ row_slot0,
                                                        const int* __restrict__ row_nslot, double* G,
                                                        int slot_d2) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(n_rows) * slot_d2) return;
  const int m = static_cast<int>(e / slot_d2), i = static_cast<int>(e % slot_d2);
  const int row = rows[m];
  double2* base = reinterpret_cast<double2*>(G) + static_cast<int64_t>(row_slot0[row]) * slot_d2 + i;
  const int ns = row_nslot[row];
  double2 v = base[0];
  int t = 1;
  for (; t + 4 <= ns; t += 4) {
    const double2 a = base[static_cast<int64_t>(t) * slot_d2], b = base[static_cast<int64_t>(t + 1) * slot_d2];
    const double2 c = base[static_cast<int64_t>(t + 2) * slot_d2], d = base[static_cast<int64_t>(t + 3) * slot_d2];
    v.x += a.x; v.y += a.y;
    v.x += b.x; v.y += b.y;
    v.x += c.x; v.y += c.y;
    v.x += d.x; v.y += d.y;
  }
  for (; t < ns; ++t) {
    const double2 a = base[static_cast<int64_t>(t) * slot_d2];
    v.x += a.x; v.y += a.y;
  }
  base[0] = v;
}

template <int NB>
struct Mode {
  static constexpr int GW = NB <= 4 ? 1 : (NB <= 16 ? 4 : (NB <= 20 ? 8 : 16));
};

constexpr size_t kGramBudget = size_t(8) << 30;  // bytes of partial Grams per batch

// Largest block count solved by k_hs_solve_1w (one warp per column); above it
// the warp-specialised team kernel.  ALSNCG_SOLVE_1W_MAX overrides (development A/B).
#ifndef AB2_SOLVE_1W_MAX_NB
#define AB2_SOLVE_1W_MAX_NB 11
#endif
inline int solve_1w_max_nb() {
  static const int v = [] {
    const char* e = std::getenv("ALSNCG_SOLVE_1W_MAX");
    return e ? std::atoi(e) : AB2_SOLVE_1W_MAX_NB;
  }();
  return v;
}
template <int NB>
void run_hs_impl(Ctx* ctx, DevRatings& R, int kind, HsArgs& a, int S) {
  constexpr int GW = Mode<NB>::GW;
  using C = HsCfg<NB, GW>;
#ifndef AB2_FUSED_MAX_NB
#define AB2_FUSED_MAX_NB 4
#endif
  if constexpr (NB <= AB2_FUSED_MAX_NB) {
    // fused warp-per-segment kernel (Gram + solve in one pass)
    const SegPlan& P = R.plan(kind, S);
    a.seg_row = P.seg_row;
    a.seg_beg = P.seg_beg;
    a.seg_len = P.seg_len;
    a.seg_slot = P.seg_slot;
    a.n_seg = P.n_seg;
    a.m_row = P.m_row;
    a.m_slot0 = P.m_slot0;
    a.m_nslot = P.m_nslot;
    a.n_multi = P.n_multi;
    const size_t smem = sizeof(double) * hs_group_doubles<NB, GW>(a.ld) * C::GPC;
    ctx->prepare_kernel(reinterpret_cast<const void*>(k_hs_main<NB, GW>), 227 * 1024, 0, 0);
    ctx->prepare_kernel(reinterpret_cast<const void*>(k_hs_reduce<NB, GW>), 227 * 1024, 0, 0);
    if (P.n_slots > 0)
      a.partial = static_cast<double*>(ctx->scratch(2, sizeof(double) * C::PART * P.n_slots));
    {
      const int blocks = (P.n_seg + C::GPC - 1) / C::GPC;
      const int tok = ctx->begin_launch("halfsweep_fused");
      k_hs_main<NB, GW><<<blocks, C::THREADS, smem, ctx->stream>>>(a);
      ctx->end_launch(tok);
    }
    if (P.n_multi > 0) {
      const int blocks = (P.n_multi + C::GPC - 1) / C::GPC;
      const int tok = ctx->begin_launch("halfsweep_fused_reduce");
      k_hs_reduce<NB, GW><<<blocks, C::THREADS, smem, ctx->stream>>>(a);
      ctx->end_launch(tok);
    }
  } else {
    const size_t slot_bytes = sizeof(double) * C::P * 64;
    const HsPlan& P = R.hs_plan(kind, S, std::max<int64_t>(1, kGramBudget / slot_bytes));
    // per-device attribute / occupancy cache (Ctx::prepare_kernel)
    const int gram_per_sm =
        ctx->prepare_kernel(reinterpret_cast<const void*>(k_hs_gram_ws<NB>), 227 * 1024,
                            (WsShape<NB>::GR + 1) * 32, WsShape<NB>::smem_bytes());
    ctx->prepare_kernel(reinterpret_cast<const void*>(k_hs_solve_ws<NB>),
                        WsSolve<NB>::TEAMS * WsSolve<NB>::TEAM_BYTES, 0, 0);
    double* G = static_cast<double*>(ctx->scratch(2, slot_bytes * std::max(P.max_batch_slots, 1)));
    // Keep the gathered source factor rows resident in L2 while the Gram
    // stream (written with evict-first stores) passes through.
    const int n_src = kind == 0 ? R.n_m : R.n_u;
    L2Window l2(ctx, a.src, sizeof(double) * static_cast<size_t>(n_src) * a.ld);
    for (const HsBatch& b : P.batches) {
      if (ctx->side_join) {  // side work runs beside the previous batch's solve only
        AB2_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
        ctx->side_join = false;
      }
      if (b.seg1 > b.seg0) {
        using WS = WsShape<NB>;
        const int nseg = b.seg1 - b.seg0;
        // persistent CTAs, the same number for every part
        const int grid = WS::NPART * std::min(nseg, std::max(gram_per_sm * ctx->sm_count / WS::NPART, 1));
        int* next_seg = static_cast<int*>(ctx->scratch(8, WS::NPART * sizeof(int)));
        AB2_CUDA(cudaMemsetAsync(next_seg, 0, WS::NPART * sizeof(int), ctx->stream));
        const int tok = ctx->begin_launch("halfsweep_gram");
        k_hs_gram_ws<NB><<<grid, (WS::GR + 1) * 32, WS::smem_bytes(), ctx->stream>>>(
            a, P.seg_len + b.seg0, P.seg_beg + b.seg0, P.seg_slot + b.seg0, nseg, G, next_seg);
        ctx->end_launch(tok);
      }
      if (ctx->side_work) {  // independent side work overlaps this batch's solve
        AB2_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
        auto w = std::move(ctx->side_work);
        ctx->side_work = nullptr;
        w();
        ctx->side_join = true;
      }
      SolveArgs s;
      s.row0 = b.row0;
      s.nrows = b.row1 - b.row0;
      s.row_slot0 = P.row_slot0;
      s.row_nslot = P.row_nslot;
      s.G = G;
      if (b.multi1 > b.multi0) {  // the solve reads one (folded) slot per row
        const int slot_d2 = C::P * 32;
        const int64_t n = static_cast<int64_t>(b.multi1 - b.multi0) * slot_d2;
        const int tok = ctx->begin_launch("halfsweep_slot_reduce");
        k_hs_slot_reduce<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
            P.multi_rows + b.multi0, b.multi1 - b.multi0, P.row_slot0, P.row_nslot, G, slot_d2);
        ctx->end_launch(tok);
      }
      int* next_col = static_cast<int*>(ctx->scratch(9, sizeof(int)));
      AB2_CUDA(cudaMemsetAsync(next_col, 0, sizeof(int), ctx->stream));
      using WSV = WsSolve<NB>;
      const int grid = std::min(s.nrows, ctx->sm_count);  // persistent: one CTA per SM
      const int tok = ctx->begin_launch("halfsweep_solve");
      if (NB <= solve_1w_max_nb()) {
        using OW = OneWarpSolve<NB>;
        ctx->prepare_kernel(reinterpret_cast<const void*>(k_hs_solve_1w<NB>), static_cast<int>(OW::smem_bytes()), 0, 0);
        k_hs_solve_1w<NB><<<grid, OW::THREADS, OW::smem_bytes(), ctx->stream>>>(a, s, next_col);
      } else {
        k_hs_solve_ws<NB><<<grid, WSV::THREADS, WSV::TEAMS * WSV::TEAM_BYTES, ctx->stream>>>(a, s, next_col);
      }
      ctx->end_launch(tok);
    }
  }
}

}  // namespace

template <>
void run_hs<AB2_HS_NB>(Ctx* ctx, DevRatings& R, int kind, HsArgs& a, int S) {
  run_hs_impl<AB2_HS_NB>(ctx, R, kind, a, S);
}

}  // namespace hs
}  // namespace ab2

#ifdef AB2_WS_PROBE
#define AB2_CAT2(a, b) a##b
#define AB2_CAT(a, b) AB2_CAT2(a, b)
extern "C" int AB2_CAT(alsncg_debug_ws_probe_, AB2_HS_NB)(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, ab2::hs::g_ws_probe, sizeof(ab2::hs::g_ws_probe)));
}
#endif
