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
  const size_t body = stage > mat ? stage : mat;
  return body + 2 * static_cast<size_t>(C::MAXF);  // + dinv[], w[]
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
  for (int e = gtid; e < 2 * C::CH * padw; e += C::GT) {
    const int t = e / padw, c = e - t * padw;  // t indexes rows of both buffers
    g_smem[sb + t * C::LDS + ld + c] = 0.0;
  }
  group_sync<GW>();
  // Each warp loads the stage's CH indices with one coalesced load (lane t
  // holds rating t) and hands them out by shuffle, so every cp.async of the
  // stage issues after a single index-load latency.
  auto issue = [&](int s, int bo) {
    const int base = s * C::CH;
    const int jv = (lane < C::CH && base + lane < len) ? a.idx[beg + base + lane] : 0;
    for (int c0 = 0; c0 < C::CH * nch; c0 += C::GT) {
      const int c = c0 + gtid;
      const int t = min(c / nch, C::CH - 1), k = c - t * nch;
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
  if (nst > 0) issue(0, sb);
  cp_async_commit();
  for (int s = 0; s < nst; ++s) {
    if (s + 1 < nst) {
      issue(s + 1, sb + ((s + 1) & 1) * BUF);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    group_sync<GW>();
    const int bo = sb + (s & 1) * BUF + lofs;
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
  const size_t body = hs_group_doubles<NB, GW>(ld) - 2 * C::MAXF;
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
  solve_row<NB, GW>(a, S, lr, count, gtid, warp, lane, acc, pI, pJ);
}

// ------------------------------------------------ split path (n_f >= 31) --
// K1/K2: Gram-only kernel.  The NB(NB+1)/2 lower-triangular 8x8 blocks are
// split into GR bands of block rows (compile-time, balanced pair counts);
// warp w owns band w / GK and every GK-th k-step (k-group w % GK).  Per
// k-step a warp loads each needed 8-row fragment ONCE into registers (the
// A fragment of block I equals the B fragment of block I) and issues all of
// its band's DMMAs from registers: ~0.3 shared loads per DMMA instead of 2,
// which is what lets the FP64 tensor pipe run near its peak.
constexpr int kGramStage = 32;  // ratings per TMA stage in the Gram kernel

template <int NB>
struct GramShape {
  static constexpr int P = NB * (NB + 1) / 2;
  // ~24 block pairs per warp (48 accumulator doubles): enough register reuse
  // per fragment load, and light enough for 3-4 CTAs per SM.
  // <= ~48 block pairs (96 accumulator doubles) per warp; the k-steps of a
  // stage are split over GK warps per band when there are few bands.
  static constexpr int GR = (P + 47) / 48 < 2 ? 2 : ((P + 47) / 48 > 8 ? 8 : (P + 47) / 48);
  static constexpr int GK = GR >= 4 ? 1 : 4 / GR;
  static constexpr int W = GR * GK;
  // first block row of band r (balanced by pair count)
  static constexpr int band_start(int r) {
    if (r <= 0) return 0;
    if (r >= GR) return NB;
    int acc = 0;
    for (int I = 0; I < NB; ++I) {
      if (acc * GR >= r * P) return I;
      acc += I + 1;
    }
    return NB;
  }
  static constexpr int band_pairs(int r) {
    const int a = band_start(r), b = band_start(r + 1);
    return b * (b + 1) / 2 - a * (a + 1) / 2;
  }
  static constexpr int max_pairs() {
    int m = 0;
    for (int r = 0; r < GR; ++r) m = band_pairs(r) > m ? band_pairs(r) : m;
    return m;
  }
  static constexpr int MAXP = max_pairs();
};

template <int NB, int R>
__device__ __forceinline__ void gram_band_kstep(int base, double (&acc)[GramShape<NB>::MAXP][2]) {
  using G = GramShape<NB>;
  constexpr int I0 = G::band_start(R), I1 = G::band_start(R + 1);
  double f[I1 > 0 ? I1 : 1];
#pragma unroll
  for (int b = 0; b < I1; ++b) f[b] = g_smem[base + 8 * b];
  int p = 0;
#pragma unroll
  for (int I = I0; I < I1; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J) {
      dmma884(acc[p][0], acc[p][1], f[I], f[J]);
      ++p;
    }
}

template <int NB, int R>
__device__ __forceinline__ void gram_band(const HsArgs& a, int64_t beg, int len, int kgroup,
                                          int lane, double (&acc)[GramShape<NB>::MAXP][2]) {
  using G = GramShape<NB>;
  using C = HsCfg<NB, G::W>;
  constexpr int CH = kGramStage;
  constexpr int BUF = CH * C::LDS;
  const int gtid = threadIdx.x, warp = gtid >> 5;
  const int ld = a.ld;
  const int padw = C::LDS - ld;
  uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem + 2 * BUF);  // 2 mbarriers after the buffers
  for (int e = gtid; e < 2 * CH * padw; e += C::GT) {
    const int t = e / padw, c = e - t * padw;
    g_smem[t * C::LDS + ld + c] = 0.0;
  }
  if (gtid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  __syncthreads();
  // Stage s -> buffer s&1: warp 0 gathers the stage's rows with one TMA bulk
  // copy per rating (lane t copies source row idx[t], ld*8 bytes) completing
  // on the buffer's mbarrier; missing tail rows are zero-filled and the
  // rating values go to column ld with ordinary stores.
  auto issue = [&](int s) {
    const int base = s * CH;
    const int bo = (s & 1) * BUF;
    const int nv = min(CH, len - base);
    if (warp == 0) {
      fence_proxy_async_smem();  // prior generic reads of this buffer happen-before the async writes
      if (lane == 0) mbar_arrive_expect_tx(bar + (s & 1), static_cast<unsigned>(nv) * ld * 8);
      __syncwarp();
      for (int t = lane; t < nv; t += 32) {
        const int j = a.idx[beg + base + t];
        tma_load_1d(&g_smem[bo + t * C::LDS], a.src + static_cast<int64_t>(j) * ld,
                    static_cast<unsigned>(ld) * 8, bar + (s & 1));
      }
    }
    for (int e = gtid; e < (CH - nv) * ld; e += C::GT) {
      const int t = nv + e / ld, c = e % ld;
      g_smem[bo + t * C::LDS + c] = 0.0;
    }
    for (int t = gtid; t < CH; t += C::GT)
      g_smem[bo + t * C::LDS + ld] = t < nv ? a.val[beg + base + t] : 0.0;
  };
  const int lofs = (lane & 3) * C::LDS + (lane >> 2);
  const int nst = (len + CH - 1) / CH;
  if (nst > 0) issue(0);
  for (int s = 0; s < nst; ++s) {
    if (s + 1 < nst) issue(s + 1);
    mbar_wait(bar + (s & 1), (s >> 1) & 1);
    __syncthreads();  // zero rows / rating column of stage s visible
    const int bo = (s & 1) * BUF + lofs;
#pragma unroll
    for (int kk = kgroup; kk < CH / 4; kk += G::GK) gram_band_kstep<NB, R>(bo + kk * 4 * C::LDS, acc);
    __syncthreads();
  }
}

template <int NB, int R>
__device__ __forceinline__ void gram_band_out(int kgroup, int lane, double* out,
                                              double (&acc)[GramShape<NB>::MAXP][2]) {
  using G = GramShape<NB>;
  constexpr int I0 = G::band_start(R);
  constexpr int NP = G::band_pairs(R);
  constexpr int p0 = I0 * (I0 + 1) / 2;
  // k-groups > 0 park their partials in shared memory; k-group 0 adds them in
  // k-group order (deterministic) and writes the band's canonical blocks.
  double* park = g_smem + R * (G::GK - 1) * G::MAXP * 64;
  if (kgroup > 0) {
#pragma unroll
    for (int p = 0; p < NP; ++p)
      *reinterpret_cast<double2*>(park + ((kgroup - 1) * G::MAXP + p) * 64 + lane * 2) =
          make_double2(acc[p][0], acc[p][1]);
  }
  __syncthreads();
  if (kgroup == 0) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double2 v = make_double2(acc[p][0], acc[p][1]);
      for (int g = 1; g < G::GK; ++g) {
        const double2 u = *reinterpret_cast<const double2*>(park + ((g - 1) * G::MAXP + p) * 64 + lane * 2);
        v.x += u.x;
        v.y += u.y;
      }
      __stcs(reinterpret_cast<double2*>(out + (p0 + p) * 64 + lane * 2), v);  // streaming: keep L2 for factor rows
    }
  }
}

template <int NB>
__global__ void __launch_bounds__(GramShape<NB>::W * 32)
    k_hs_gram(HsArgs a, const int* __restrict__ seg_len, const int64_t* __restrict__ seg_beg,
              const int* __restrict__ seg_slot, double* __restrict__ G) {
  using GS = GramShape<NB>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int band = warp / GS::GK, kgroup = warp % GS::GK;
  const int seg = blockIdx.x;
  const int64_t beg = seg_beg[seg];
  const int len = seg_len[seg];
  double* out = G + static_cast<int64_t>(seg_slot[seg]) * GS::P * 64;
  double acc[GS::MAXP][2];
#pragma unroll
  for (int p = 0; p < GS::MAXP; ++p) acc[p][0] = acc[p][1] = 0.0;
  // one fully specialised body per band (compile-time fragment indices)
#define AB2_BAND(R)                                              \
  if (band == R && R < GS::GR) {                                 \
    gram_band<NB, (R < GS::GR ? R : 0)>(a, beg, len, kgroup, lane, acc); \
    gram_band_out<NB, (R < GS::GR ? R : 0)>(kgroup, lane, out, acc);     \
  }
  AB2_BAND(0) AB2_BAND(1) AB2_BAND(2) AB2_BAND(3) AB2_BAND(4) AB2_BAND(5) AB2_BAND(6) AB2_BAND(7)
  AB2_BAND(8) AB2_BAND(9) AB2_BAND(10) AB2_BAND(11) AB2_BAND(12) AB2_BAND(13) AB2_BAND(14) AB2_BAND(15)
#undef AB2_BAND
}

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
  // ~12 block pairs per consumer warp, 2..8 consumers
  static constexpr int GR = P < 2 ? 1 : ((P + 11) / 12 < 2 ? 2 : ((P + 11) / 12 > 8 ? 8 : (P + 11) / 12));
  static constexpr int LDS = NB * 8 + 4;
  static constexpr int BUF = kWsCH * LDS;
  // ring depth: 2 stages from NB = 6 up -- more CTAs per SM, more consumer
  // warps on the DMMA pipe (measured 15.6 -> 15.3 ms at n_f = 100, Gram
  // 4.87 -> 4.70 ms at n_f = 50); NB = 5 keeps 3 stages
  static constexpr int STAGES = NB >= 6 ? 2 : 3;
  static constexpr int p_begin(int r) { return r * P / GR; }
  static constexpr int row_of(int p) {
    int i = 0;
    while ((i + 1) * (i + 2) / 2 <= p) ++i;
    return i;
  }
  static constexpr int col_of(int p) { return p - row_of(p) * (row_of(p) + 1) / 2; }
  static constexpr bool needs(int r, int b) {
    for (int p = p_begin(r); p < p_begin(r + 1); ++p)
      if (row_of(p) == b || col_of(p) == b) return true;
    return false;
  }
  static constexpr int max_pairs() {
    int m = 0;
    for (int r = 0; r < GR; ++r) m = p_begin(r + 1) - p_begin(r) > m ? p_begin(r + 1) - p_begin(r) : m;
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
#pragma unroll
  for (int b = 0; b < NB; ++b)
    if (S::needs(R, b)) f[b] = g_smem[base + 8 * b];
#pragma unroll
  for (int p = p0; p < p1; ++p)
    dmma884(acc[p - p0][0], acc[p - p0][1], f[S::row_of(p)], f[S::col_of(p)]);
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
#pragma unroll
      for (int kk = 0; kk < kWsCH / 4; ++kk) ws_kstep<NB, R>(bo + kk * 4 * S::LDS, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + buf);
    }
    double* out = G + static_cast<int64_t>(seg_slot[seg]) * S::P * 64 + p0 * 64 + lane * 2;
#pragma unroll
    for (int p = 0; p < np; ++p)
      __stcs(reinterpret_cast<double2*>(out + p * 64), make_double2(acc[p][0], acc[p][1]));
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
#define AB2_WS(R)                                                                           \
  if (warp == R && R < S::GR)                                                               \
    ws_consumer<NB, (R < S::GR ? R : 0)>(seg_len, seg_slot, n_seg, G, full, empty, hdr, lane);
  AB2_WS(0) AB2_WS(1) AB2_WS(2) AB2_WS(3) AB2_WS(4) AB2_WS(5) AB2_WS(6) AB2_WS(7)
#undef AB2_WS
}


template <int NB>
struct SolveCfg {
  static constexpr int P = NB * (NB + 1) / 2;  // lower-triangular 8x8 blocks of the augmented Gram
};

__device__ __forceinline__ int pidx(int I, int J) { return I * (I + 1) / 2 + J; }
// Swizzled 8x8 block storage: element (r, c) at 8r + (c ^ 4*((r>>1)&1)); the
// C-fragment (16-byte) and A/B-fragment (8-byte) accesses are conflict-free.
__device__ __forceinline__ int swz(int r, int c) { return 8 * r + (c ^ (4 * ((r >> 1) & 1))); }

// K3 (static-schedule form): one 4-warp CTA per column, right-looking blocked
// LDL^T on the swizzled shared-memory block store, with the whole schedule
// resolved at compile time (panel J, block coordinates and owning warp are
// template constants, so the instruction stream is the arithmetic plus
// immediate-offset shared loads/stores):
//   F(J)  warp 0 factors the 8x8 diagonal block (lanes = rows, pivots by
//         shuffle) and publishes 1/d and the 28 in-block coefficients;
//   T(J)  one thread per row below the diagonal eliminates it against the
//         block (TRSM form) and writes X = L~(I,J) and S = -X D^-1;
//   U(J)  warps 1..3 apply C(I,K) += X_I S_K^T (two DMMAs per block,
//         column-major chunks so S_K fragments are reused) while warp 0
//         updates the next diagonal block and immediately factors it
//         (F(J+1) overlaps the rest of U(J)).
// Two CTA barriers per panel.  Back substitution by warp 0 as in k_hs_solve.
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  [&]<int... Is>(std::integer_sequence<int, Is...>) { (f(std::integral_constant<int, Is>{}), ...); }(
      std::make_integer_sequence<int, N>{});
}

constexpr int kSwWarps = 4;

template <int NB, int W>
struct SwSched {
  static constexpr int P = NB * (NB + 1) / 2;
  // U(J) blocks (I,K), J < K <= I < NB, column-major, without (J+1,J+1)
  static constexpr int count(int J) { return (NB - 1 - J) * (NB - J) / 2 - 1; }
  static constexpr int order(int J, int I, int K) {
    return (K - 1 - J) * NB - ((K - 1) * K / 2 - J * (J + 1) / 2) + (I - K) - 1;
  }
  static constexpr int owner(int J, int I, int K) {
    return (I == J + 1 && K == J + 1) ? 0 : 1 + order(J, I, K) * (W - 1) / count(J);
  }
  static constexpr int cidx(int c) { return c * 7 - c * (c - 1) / 2; }  // first coefficient of column c
  // shared layout (doubles)
  static constexpr int OFF_S = P * 64;             // NB blocks: -X D^-1 of the current panel
  static constexpr int OFF_C = OFF_S + NB * 64;    // 28 TRSM coefficients (+4)
  static constexpr int OFF_DINV = OFF_C + 32;      // NB*8
  static constexpr int OFF_W = OFF_DINV + NB * 8;  // NB*8 back-substitution vector
  static constexpr int SMEM = OFF_W + NB * 8;
};

// F(J): factor the diagonal block (warp 0): lane rr holds row rr (four
// replicas per warp), pivots by shuffle.  Publishes the factored rows, 1/d
// and the 28 in-block coefficients L(c2, c).  Returns false on a
// non-positive pivot (uniform across the warp).
template <int NB, int W, int J>
__device__ __forceinline__ bool sw_factor(double* M, int n_f, int lane) {
  using SS = SwSched<NB, W>;
  double* D = M + pidx(J, J) * 64;
  double* coef = M + SS::OFF_C;
  double* dinv = M + SS::OFF_DINV;
  const int rr = lane & 7;
  __syncwarp();  // the block was just updated by this warp's lanes
  double row[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) row[c] = D[swz(rr, c)];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int k = 8 * J + c;
    double inv = 0.0;
    if (k < n_f) {
      const double d = __shfl_sync(kFull, row[c], c);
      if (!(d > 0.0)) {  // Eigen LLT: NumericalIssue on a non-positive pivot
        ok = false;
        break;
      }
      inv = fast_rcp(d);
      const double l = row[c] * inv;
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) {
        const double av = __shfl_sync(kFull, row[c], c2);  // A(c2, c)
        if (rr > c && c2 <= rr) row[c2] = fma(-l, av, row[c2]);
      }
    }
    if (lane == 0) dinv[k] = inv;
    if (c < 7 && lane < 8 && rr > c) coef[SS::cidx(c) + rr - c - 1] = row[c] * inv;  // L(rr, c)
  }
  if (ok && lane < 8)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c <= rr) D[swz(rr, c)] = row[c];
  return ok;
}

// T(J): eliminate every row of the blocks below the diagonal (one per thread).

template <int NB, int W, int J>
__device__ __forceinline__ void sw_trsm_row(double* M, int row) {
  using SS = SwSched<NB, W>;
  const int I = J + 1 + (row >> 3), rr = row & 7;
  const bool sw = (rr >> 1) & 1;  // swizzle: columns 0-3 and 4-7 swap halves
  double2* xr = reinterpret_cast<double2*>(M + (I * (I + 1) / 2 + J) * 64 + 8 * rr);
  double2* sr = reinterpret_cast<double2*>(M + SS::OFF_S + I * 64 + 8 * rr);
  const double2* cf = reinterpret_cast<const double2*>(M + SS::OFF_C);
  const double2* dv = reinterpret_cast<const double2*>(M + SS::OFF_DINV + 8 * J);
  double x[8];
  {
    const double2 v0 = xr[0], v1 = xr[1], v2 = xr[2], v3 = xr[3];
    x[0] = sw ? v2.x : v0.x; x[1] = sw ? v2.y : v0.y; x[2] = sw ? v3.x : v1.x; x[3] = sw ? v3.y : v1.y;
    x[4] = sw ? v0.x : v2.x; x[5] = sw ? v0.y : v2.y; x[6] = sw ? v1.x : v3.x; x[7] = sw ? v1.y : v3.y;
  }
  double cc[28];
#pragma unroll
  for (int u = 0; u < 14; ++u) {
    const double2 v = cf[u];
    cc[2 * u] = v.x;
    cc[2 * u + 1] = v.y;
  }
  {
    int u = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) x[c2] = fma(-x[c], cc[u++], x[c2]);
  }
  double iv[8];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const double2 v = dv[h];
    iv[2 * h] = v.x;
    iv[2 * h + 1] = v.y;
  }
  double s[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) s[c] = -x[c] * iv[c];
  const int a = sw ? 2 : 0, b = sw ? 0 : 2;
  xr[a] = make_double2(x[0], x[1]);
  xr[a + 1] = make_double2(x[2], x[3]);
  xr[b] = make_double2(x[4], x[5]);
  xr[b + 1] = make_double2(x[6], x[7]);
  sr[a] = make_double2(s[0], s[1]);
  sr[a + 1] = make_double2(s[2], s[3]);
  sr[b] = make_double2(s[4], s[5]);
  sr[b + 1] = make_double2(s[6], s[7]);
}

template <int NB, int W, int J>
__device__ __forceinline__ void sw_trsm(double* M, int tid) {
  constexpr int ROWS = 8 * (NB - 1 - J);
  for (int row = tid; row < ROWS; row += W * 32) sw_trsm_row<NB, W, J>(M, row);
}

// Compile-time list of the U(J) blocks warp w owns (column-major order).
template <int NB, int W>
struct SwList {
  int n;
  int I[NB * (NB + 1) / 2];
  int K[NB * (NB + 1) / 2];
  static constexpr SwList make(int J, int w) {
    SwList l{};
    for (int k = J + 1; k < NB; ++k)
      for (int i = k; i < NB; ++i)
        if (SwSched<NB, W>::owner(J, i, k) == w) {
          l.I[l.n] = i;
          l.K[l.n] = k;
          ++l.n;
        }
    return l;
  }
};

template <int NB, int W, int J, int w>
struct SwL {
  static constexpr SwList<NB, W> v = SwList<NB, W>::make(J, w);
};

// U(J) for warp w: C(I,K) += X_I S_K^T (S holds -X D^-1), G blocks at a time
// with every load of a group issued before its DMMAs and stores (the
// blocks are independent; the compiler cannot prove it through the lane
// offsets, so the batching is explicit).
template <int NB, int W, int J, int w>
__device__ __forceinline__ void sw_update(double* M, int oc, int oa0, int oa1) {
  using SS = SwSched<NB, W>;
  using L = SwL<NB, W, J, w>;
  constexpr int G = 4;
  static_for<(L::v.n + G - 1) / G>([&](auto gc) {
    constexpr int g0 = decltype(gc)::value * G;
    double2 c[G];
    double xa[G][2], sb[G][2];
    static_for<G>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if constexpr (g0 + i < L::v.n) {
        constexpr int I = L::v.I[g0 + i], K = L::v.K[g0 + i];
        c[i] = *reinterpret_cast<const double2*>(M + (I * (I + 1) / 2 + K) * 64 + oc);
        xa[i][0] = M[(I * (I + 1) / 2 + J) * 64 + oa0];
        xa[i][1] = M[(I * (I + 1) / 2 + J) * 64 + oa1];
        sb[i][0] = M[SS::OFF_S + K * 64 + oa0];
        sb[i][1] = M[SS::OFF_S + K * 64 + oa1];
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
        *reinterpret_cast<double2*>(M + (I * (I + 1) / 2 + K) * 64 + oc) = c[i];
      }
    });
  });
}

#ifdef AB2_SW_PROBE
// development probe: per-phase clocks of the first 64 columns (warp 0, lane 0)
__device__ unsigned long long g_sw_probe[64][64];
#define SW_PROBE(slot) \
  do { if ((blockIdx.x & 1023) == 0 && blockIdx.x < 65536 && (threadIdx.x & 127) == 0) g_sw_probe[blockIdx.x >> 10][slot] = clock64(); } while (0)
#define SW_PROBE_W(slot) \
  do { if ((blockIdx.x & 1023) == 0 && blockIdx.x < 65536 && (threadIdx.x & 31) == 0) g_sw_probe[blockIdx.x >> 10][slot] = clock64(); } while (0)
#else
#define SW_PROBE(slot) do {} while (0)
#define SW_PROBE_W(slot) do {} while (0)
#endif

// The factorization proper for warp w; false if a pivot was non-positive.
template <int NB, int W, int w>
__device__ __forceinline__ bool sw_run(double* M, int n_f, int tid, int lane, volatile int* fail) {
  using SS = SwSched<NB, W>;
  const int KP = (n_f + 7) >> 3;
  const int r = lane >> 2, q = lane & 3;
  const int oc = swz(r, 2 * q), oa0 = swz(r, q), oa1 = swz(r, 4 + q);
  if constexpr (w == 0)
    if (!sw_factor<NB, W, 0>(M, n_f, lane) && lane == 0) *fail = 1;
  __syncthreads();
  if (*fail) return false;
  bool ok = true;
  static_for<NB>([&](auto Jc) {
    constexpr int J = decltype(Jc)::value;
    if (!ok || J >= KP) return;
    SW_PROBE(2 + 4 * J);
    sw_trsm<NB, W, J>(M, tid);
    SW_PROBE(3 + 4 * J);
    __syncthreads();
    if constexpr (J + 1 < NB) {
      // (blocks of column NB-1 are updated even when it is not a pivot
      // column: harmless, they are never read again)
      SW_PROBE(4 + 4 * J);
      sw_update<NB, W, J, w>(M, oc, oa0, oa1);
      if constexpr (w == 0) {
        SW_PROBE_W(5 + 4 * J);
        if (J + 1 < KP && !sw_factor<NB, W, J + 1>(M, n_f, lane) && lane == 0) *fail = 1;
      }
    }
    __syncthreads();
    if (*fail) ok = false;
  });
  return ok;
}

template <int NB>
__global__ void __launch_bounds__(kSwWarps * 32) k_hs_solve_sw(HsArgs a, SolveArgs s) {
  using C = SolveCfg<NB>;
  using SS = SwSched<NB, kSwWarps>;
  constexpr int NT = kSwWarps * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  SW_PROBE(0);
  const int lr = s.row0 + blockIdx.x;
  const int n_f = a.n_f, ld = a.ld;
  double* M = g_smem;
  double* dinv = M + SS::OFF_DINV;
  double* w = M + SS::OFF_W;
  __shared__ int fail;
  double* out = a.out + static_cast<int64_t>(a.row0 + lr) * ld;
  const int count = static_cast<int>(a.ptr[lr + 1] - a.ptr[lr]);
  if (count == 0) {  // parallel.cpp:175 -- empty column stays zero
    for (int k = tid; k < ld; k += NT) out[k] = 0.0;
    return;
  }
  const double shift = a.lambda * static_cast<double>(count);  // als.cpp:58
  if (!(shift > 0.0)) {
    if (tid == 0) {
      a.fb_list[atomicAdd(a.fb_count, 1u)] = lr;
      atomicAdd(a.fb_total, 1u);
    }
    return;
  }
  const int r = lane >> 2, q = lane & 3;
  {
    // heavy rows were folded into their first slot by k_hs_slot_reduce
    const double* base = s.G + static_cast<int64_t>(s.row_slot0[lr]) * C::P * 64 + lane * 2;
    for (int p = warp; p < C::P; p += kSwWarps) cp_async16(M + p * 64 + swz(r, 2 * q), base + p * 64);
    cp_async_commit();
    cp_async_wait<0>();
    if (tid == 0) fail = 0;
    __syncthreads();
    for (int k = tid; k < n_f; k += NT) M[pidx(k >> 3, k >> 3) * 64 + swz(k & 7, k & 7)] += shift;  // als.cpp:58-59
    __syncthreads();
  }
  SW_PROBE(1);
  bool ok;
  switch (warp) {
    case 0: ok = sw_run<NB, kSwWarps, 0>(M, n_f, tid, lane, &fail); break;
    case 1: ok = sw_run<NB, kSwWarps, 1>(M, n_f, tid, lane, &fail); break;
    case 2: ok = sw_run<NB, kSwWarps, 2>(M, n_f, tid, lane, &fail); break;
    default: ok = sw_run<NB, kSwWarps, 3>(M, n_f, tid, lane, &fail); break;
  }
  if (!ok) {
    if (tid == 0) {
      a.fb_list[atomicAdd(a.fb_count, 1u)] = lr;
      atomicAdd(a.fb_total, 1u);
    }
    return;
  }
  SW_PROBE(60);
  // Back substitution, all warps: u_k = (w_k - sum_{i>k} A~(i,k) u_i) / d_k,
  // one 8-row block at a time: every thread solves the block's 8 unknowns
  // from registers (same arithmetic in every thread), then thread i < 8K
  // folds them into w_i.
  const int KP = (n_f + 7) >> 3;
  {
    const int IR = ld >> 3, rl = ld & 7;
    for (int k = tid; k < n_f; k += NT) w[k] = M[pidx(IR, k >> 3) * 64 + swz(rl, k & 7)];
  }
  __syncthreads();
  for (int K = KP - 1; K >= 0; --K) {
    const double* D = M + pidx(K, K) * 64;
    double u[8];
#pragma unroll
    for (int c = 7; c >= 0; --c) {
      double v = 0.0;
      if (8 * K + c < n_f) {
        v = w[8 * K + c];
#pragma unroll
        for (int i = 7; i > c; --i) v = fma(-D[swz(i, c)], u[i], v);  // u[c+1] (latest) last
        v *= dinv[8 * K + c];
      }
      u[c] = v;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (tid == c && 8 * K + c < n_f) out[8 * K + c] = u[c];
    for (int i = tid; i < 8 * K; i += NT) {
      const double* blk = M + pidx(K, i >> 3) * 64;
      double acc = w[i];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc = fma(-blk[swz(c, i & 7)], u[c], acc);
      w[i] = acc;
    }
    __syncthreads();
  }
  for (int k = n_f + tid; k < ld; k += NT) out[k] = 0.0;
  SW_PROBE(61);
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

constexpr size_t kGramBudget = size_t(3) << 30;  // bytes of partial Grams per batch
// compile-time kernel choice: only the kernels a rank uses are instantiated
template <int NB>
constexpr bool kGramWs = NB <= 20;                // warp-specialised persistent Gram

template <int NB>
void run_hs_impl(Ctx* ctx, DevRatings& R, int kind, HsArgs& a, int S) {
  constexpr int GW = Mode<NB>::GW;
  using C = HsCfg<NB, GW>;
  if constexpr (NB <= 4) {
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
    static bool attr_set = false;
    if (!attr_set) {
      AB2_CUDA(cudaFuncSetAttribute(k_hs_main<NB, GW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      AB2_CUDA(cudaFuncSetAttribute(k_hs_reduce<NB, GW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr_set = true;
    }
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
    using GS = GramShape<NB>;
    using GC = HsCfg<NB, GS::W>;
    const size_t gsmem = sizeof(double) * std::max<size_t>(2 * kGramStage * GC::LDS + 2,
                                                           size_t(GS::GR) * (GS::GK - 1) * GS::MAXP * 64);
    static bool attr_set = false;
    if (!attr_set) {
      if constexpr (kGramWs<NB>)
        AB2_CUDA(cudaFuncSetAttribute(k_hs_gram_ws<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      else
        AB2_CUDA(cudaFuncSetAttribute(k_hs_gram<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      AB2_CUDA(cudaFuncSetAttribute(k_hs_solve_sw<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sizeof(double) * SwSched<NB, kSwWarps>::SMEM)));
      attr_set = true;
    }
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
      if constexpr (kGramWs<NB>) {
        if (b.seg1 > b.seg0) {
          using WS = WsShape<NB>;
          const int nseg = b.seg1 - b.seg0;
          static int per_sm = 0;
          if (per_sm == 0) {
            AB2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hs_gram_ws<NB>, (WS::GR + 1) * 32,
                                                                   WS::smem_bytes()));
            per_sm = std::max(per_sm, 1);
          }
          const int grid = std::min(nseg, per_sm * ctx->sm_count);  // persistent CTAs
          int* next_seg = static_cast<int*>(ctx->scratch(8, sizeof(int)));
          AB2_CUDA(cudaMemsetAsync(next_seg, 0, sizeof(int), ctx->stream));
          const int tok = ctx->begin_launch("halfsweep_gram");
          k_hs_gram_ws<NB><<<grid, (WS::GR + 1) * 32, WS::smem_bytes(), ctx->stream>>>(
              a, P.seg_len + b.seg0, P.seg_beg + b.seg0, P.seg_slot + b.seg0, nseg, G, next_seg);
          ctx->end_launch(tok);
        }
      } else if (b.seg1 > b.seg0) {
        const int tok = ctx->begin_launch("halfsweep_gram");
        k_hs_gram<NB><<<b.seg1 - b.seg0, GS::W * 32, gsmem, ctx->stream>>>(
            a, P.seg_len + b.seg0, P.seg_beg + b.seg0, P.seg_slot + b.seg0, G);
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
      const int tok = ctx->begin_launch("halfsweep_solve");
      k_hs_solve_sw<NB><<<s.nrows, kSwWarps * 32, sizeof(double) * SwSched<NB, kSwWarps>::SMEM, ctx->stream>>>(a, s);
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

#ifdef AB2_SW_PROBE
#define AB2_CAT2(a, b) a##b
#define AB2_CAT(a, b) AB2_CAT2(a, b)
extern "C" int AB2_CAT(alsncg_debug_sw_probe_, AB2_HS_NB)(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, ab2::hs::g_sw_probe, sizeof(ab2::hs::g_sw_probe)));
}
#endif
