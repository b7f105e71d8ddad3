// common.cuh -- device helpers shared by the k_*.cu kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace ab2 {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Double-double accumulation (Knuth TwoSum).  Every reduction that feeds a
// discrete decision of the NCG driver (Armijo test, descent tests, beta
// restart, stopping test) is accumulated this way, so the device result is
// the correctly rounded sum to within a couple of ulps -- at least as
// accurate as the reference's sequential sums and Kahan chunks
// (linesearch.cpp:26-35), and independent of the launch geometry.
struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}

__device__ __forceinline__ void dd_add(dd& acc, double x) {
  const dd t = two_sum(acc.hi, x);
  acc.hi = t.hi;
  acc.lo = __dadd_rn(acc.lo, t.lo);
}

__device__ __forceinline__ dd dd_plus(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  s.lo = __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo));
  const double hi = __dadd_rn(s.hi, s.lo);  // renormalise (fast two-sum)
  const double lo = __dsub_rn(s.lo, __dsub_rn(hi, s.hi));
  return {hi, lo};
}

__device__ __forceinline__ double dd_value(dd a) { return __dadd_rn(a.hi, a.lo); }

__device__ __forceinline__ dd shfl_xor_dd(dd v, int off) {
  return {__shfl_xor_sync(kFull, v.hi, off), __shfl_xor_sync(kFull, v.lo, off)};
}

__device__ __forceinline__ dd warp_sum_dd(dd v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = dd_plus(v, shfl_xor_dd(v, off));
  return v;
}

// Block-wide sum of NS double-doubles; result valid in thread 0.  `sh` must
// hold (blockDim.x/32)*NS dd.  Fixed combination order -> deterministic.
template <int NS>
__device__ __forceinline__ void block_sum_dd(dd (&v)[NS], dd* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NS; ++k) v[k] = warp_sum_dd(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NS; ++k) sh[warp * NS + k] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      dd x = lane < nw ? sh[lane * NS + k] : dd{0.0, 0.0};
      v[k] = warp_sum_dd(x);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// --- TMA bulk copies (cp.async.bulk) completing on an mbarrier ------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// Global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned).
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, unsigned bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1/d for a positive normal d: hardware reciprocal seed (MUFU.RCP64H) and two
// Newton steps -- a short dependency chain instead of the IEEE division
// subroutine; error <= 1 ulp, used only on Cholesky pivots.
__device__ __forceinline__ double fast_rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

// FP64 tensor-core MMA (lowers to SASS DMMA.8x8x4 on sm_100a):
// D(8x8) += A(8x4) * B(4x8); lane l holds A[l>>2][l&3], B[l&3][l>>2],
// D[l>>2][2*(l&3) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace ab2
