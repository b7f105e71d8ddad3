// k_halfsweep.cu -- K1-K4 dispatcher: picks the per-NB Gram/solve unit
// (k_hs_inst.cu) for the rank and runs the least-norm fallback pass
// (als.cpp:71-81) for the rows those kernels listed.
#include "k_halfsweep.cuh"

namespace ab2 {

using hs::HsArgs;

namespace {

// ------------------------------------------------------------ fallback --
// Least-norm solve for listed rows.  Workspace per CTA: W (n x n), Q (n x n).
constexpr int kFbThreads = 256;
constexpr int kFbBlocks = 296;  // 2 per SM: rank-deficient columns (lambda*n = 0) are solved in parallel

__device__ void fb_block_sum2(double& a, double& b, double* sh) {
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(kFull, a, off);
    b += __shfl_xor_sync(kFull, b, off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh[2 * warp] = a;
    sh[2 * warp + 1] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0, y = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) {
      x += sh[2 * w2];
      y += sh[2 * w2 + 1];
    }
    sh[64] = x;
    sh[65] = y;
  }
  __syncthreads();
  a = sh[64];
  b = sh[65];
  __syncthreads();
}

// out = pinv(W-eigen) * rhs, using eigenvalues on W's diagonal and vectors in Q.
__device__ void fb_pinv_apply(int n, const double* W, const double* Q, const double* rhs,
                              double* out, double* tmp, double* sh) {
  double emax = 0.0, dummy = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) emax = fmax(emax, fabs(W[i * n + i]));
  // block max via sum trick: reuse fb_block_sum2 with max semantics
  for (int off = 16; off > 0; off >>= 1) emax = fmax(emax, __shfl_xor_sync(kFull, emax, off));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) m = fmax(m, sh[w2]);
    sh[64] = m;
  }
  __syncthreads();
  emax = sh[64];
  __syncthreads();
  (void)dummy;
  const double thresh = emax * n * 2.220446049250313e-16;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const double lam = W[e * n + e];
    double proj = 0.0;
    if (fabs(lam) > thresh) {
      for (int k = 0; k < n; ++k) proj += Q[k * n + e] * rhs[k];
      proj /= lam;
    }
    tmp[e] = proj;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double s = 0.0;
    for (int e = 0; e < n; ++e) s += tmp[e] * Q[k * n + e];
    out[k] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kFbThreads) k_hs_fallback(HsArgs a, double* work) {
  const int n = a.n_f, ld = a.ld;
  const size_t nn = static_cast<size_t>(n) * n;
  double* A = work + blockIdx.x * (3 * nn + 6 * static_cast<size_t>(n));
  double* W = A + nn;
  double* Q = W + nn;
  double* v = Q + nn;
  double* u = v + n;
  double* res = u + n;
  double* du = res + n;
  double* tmp = du + n;
  __shared__ double sh[80];
  __shared__ double rot[2];
  const unsigned total = *a.fb_count;
  for (unsigned f = blockIdx.x; f < total; f += gridDim.x) {
    const int lr = a.fb_list[f];
    const int64_t b = a.ptr[lr];
    const int count = static_cast<int>(a.ptr[lr + 1] - b);
    // Gram + rhs in the reference's summation order (als.cpp:49-57), no FMA.
    for (size_t e = threadIdx.x; e < nn + n; e += blockDim.x) {
      double s = 0.0;
      if (e < nn) {
        const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
        const int lo = j <= i ? j : i, hi = j <= i ? i : j;
        for (int t = 0; t < count; ++t) {
          const double* m = a.src + static_cast<int64_t>(a.idx[b + t]) * ld;
          s = __dadd_rn(s, __dmul_rn(m[hi], m[lo]));
        }
        if (i == j) s = __dadd_rn(s, a.lambda * count);
        A[e] = s;
        W[e] = s;
        Q[e] = i == j ? 1.0 : 0.0;
      } else {
        const int i = static_cast<int>(e - nn);
        for (int t = 0; t < count; ++t) {
          const double* m = a.src + static_cast<int64_t>(a.idx[b + t]) * ld;
          s = __dadd_rn(s, __dmul_rn(a.val[b + t], m[i]));
        }
        v[i] = s;
      }
    }
    __syncthreads();
    // cyclic Jacobi (same sweep structure as the oracle restatement)
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (size_t e = threadIdx.x; e < nn; e += blockDim.x) {
        const double x = W[e] * W[e];
        tot += x;
        if (e / n != e % n) off += x;
      }
      fb_block_sum2(off, tot, sh);
      if (off <= 1e-30 * tot || off == 0.0) break;
      for (int p = 0; p < n; ++p)
        for (int r = p + 1; r < n; ++r) {
          if (threadIdx.x == 0) {
            const double apr = W[p * n + r];
            if (apr == 0.0) {
              rot[0] = 1.0;
              rot[1] = 0.0;
            } else {
              const double app = W[p * n + p], arr = W[r * n + r];
              const double theta = (arr - app) / (2.0 * apr);
              const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
              const double c = 1.0 / sqrt(t * t + 1.0);
              rot[0] = c;
              rot[1] = t * c;
            }
          }
          __syncthreads();
          const double c = rot[0], s = rot[1];
          if (s != 0.0) {
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
              const double wkp = W[k * n + p], wkr = W[k * n + r];
              W[k * n + p] = c * wkp - s * wkr;
              W[k * n + r] = s * wkp + c * wkr;
            }
            __syncthreads();
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
              const double wpk = W[p * n + k], wrk = W[r * n + k];
              W[p * n + k] = c * wpk - s * wrk;
              W[r * n + k] = s * wpk + c * wrk;
              const double qkp = Q[k * n + p], qkr = Q[k * n + r];
              Q[k * n + p] = c * qkp - s * qkr;
              Q[k * n + r] = s * qkp + c * qkr;
            }
          }
          __syncthreads();
        }
    }
    fb_pinv_apply(n, W, Q, v, u, tmp, sh);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // one refinement step (als.cpp:79)
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += A[i * n + k] * u[k];
      res[i] = v[i] - s;
    }
    __syncthreads();
    fb_pinv_apply(n, W, Q, res, du, tmp, sh);
    double* out = a.out + static_cast<int64_t>(a.row0 + lr) * ld;
    for (int i = threadIdx.x; i < ld; i += blockDim.x) out[i] = i < n ? u[i] + du[i] : 0.0;
    __syncthreads();
  }
}

int hs_segment_size(int n_f) {
  if (n_f <= 32) return 8192;
  if (n_f <= 64) return 4096;
  return 2048;
}

}  // namespace

void launch_half_sweep(DevRatings& R, int kind, int n_f, const double* src_rows, double lambda,
                       double* out_rows, int counter) {
  Ctx* ctx = R.ctx;
  if (n_f > kMaxRank) throw Error(ALSNCG_EUNSUPPORTED, "n_f exceeds the half-sweep kernel range");
  const View& v = R.view(kind);
  if (v.nrows == 0) return;
  const int ld = row_stride(n_f);
  HsArgs a;
  a.ptr = v.ptr;
  a.idx = v.idx;
  a.val = v.val;
  a.row0 = (kind == 0 ? 0 : R.n_u) + v.row0;
  a.src = src_rows;
  a.out = out_rows;
  a.n_f = n_f;
  a.ld = ld;
  a.lambda = lambda;
  a.partial = nullptr;
  // fallback bookkeeping: counters[2+...] region
  unsigned* fb_count = ctx->d_counters + 8;
  a.fb_list = static_cast<int*>(ctx->scratch(3, sizeof(int) * std::max(v.nrows, 1)));
  a.fb_count = fb_count;
  a.fb_total = ctx->d_counters + counter;
  AB2_CUDA(cudaMemsetAsync(fb_count, 0, sizeof(unsigned), ctx->stream));
  switch (gram_blocks(n_f)) {
#define AB2_HS_CASE(NB) \
  case NB:              \
    hs::run_hs<NB>(ctx, R, kind, a, hs_segment_size(n_f)); \
    break;
    AB2_HS_CASE(1) AB2_HS_CASE(2) AB2_HS_CASE(3) AB2_HS_CASE(4) AB2_HS_CASE(5) AB2_HS_CASE(6)
    AB2_HS_CASE(7) AB2_HS_CASE(8) AB2_HS_CASE(9) AB2_HS_CASE(10) AB2_HS_CASE(11) AB2_HS_CASE(12)
    AB2_HS_CASE(13) AB2_HS_CASE(14) AB2_HS_CASE(15) AB2_HS_CASE(16) AB2_HS_CASE(17)
    AB2_HS_CASE(18) AB2_HS_CASE(19) AB2_HS_CASE(20) AB2_HS_CASE(21) AB2_HS_CASE(22)
    AB2_HS_CASE(23) AB2_HS_CASE(24) AB2_HS_CASE(25) AB2_HS_CASE(26)
#undef AB2_HS_CASE
    default:
      throw Error(ALSNCG_EUNSUPPORTED, "n_f exceeds the half-sweep kernel range");
  }
  // Fallback pass (no host sync: the kernel reads the device-side count).
  const size_t per = 3 * static_cast<size_t>(n_f) * n_f + 6 * static_cast<size_t>(n_f);
  double* work = static_cast<double*>(ctx->scratch(4, sizeof(double) * per * kFbBlocks));
  const int tok = ctx->begin_launch("halfsweep_fallback");
  k_hs_fallback<<<kFbBlocks, kFbThreads, 0, ctx->stream>>>(a, work);
  ctx->end_launch(tok);
}

}  // namespace ab2
