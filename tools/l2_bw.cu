// Development probe: L2 -> SM bandwidth on this B200 (the roofline of the
// gather-bound residual kernels).  (1) streaming reads of an L2-resident
// buffer (16-byte loads, .cg = L2 only); (2) row gathers like the quartic /
// gradient: random 800-byte rows (f = 100) of a 21 MB matrix, 16 lanes x
// 16 B per row per step, default caching (L1 + L2) and .cg (L2 only).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void stream_cg(const double2* __restrict__ p, int64_t n, int reps, double* out) {
  double s = 0.0;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      s += v.x + v.y;
    }
  if (s == 1.2345) out[0] = s;
}

template <bool CG>
__global__ void gather_rows(const double* __restrict__ M, int n_rows, int ld, const int* __restrict__ idx,
                            int64_t n_idx, double* out) {
  const int lane = threadIdx.x & 31, sg = lane >> 4, sl = lane & 15;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double s = 0.0;
  for (int64_t t = warp * 2 + sg; t < n_idx; t += nw * 2) {
    const double2* row = reinterpret_cast<const double2*>(M + (int64_t)idx[t] * ld);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = sl + 16 * k;
      if (2 * e < ld) {
        double2 v = CG ? __ldcg(row + e) : __ldg(row + e);
        s += v.x + v.y;
      }
    }
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t mb : {32, 64, 96}) {
    const int64_t n = (int64_t)mb * (1 << 20) / 16;
    double2* p;
    cudaMalloc(&p, n * 16);
    cudaMemset(p, 0, n * 16);
    const int reps = 20;
    stream_cg<<<148 * 4, 512>>>(p, n, 2, out);
    cudaEventRecord(a);
    stream_cg<<<148 * 4, 512>>>(p, n, reps, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("stream .cg  %3zu MB resident: %.2f TB/s\n", mb, (double)n * 16 * reps / (ms * 1e-3) / 1e12);
    cudaFree(p);
  }
  // gathers: 26,744 rows x 100 doubles (21 MB), Zipf-ish and uniform random indices
  const int rows = 26744, ld = 100;
  const int64_t n_idx = 20000000;
  double* M;
  int* idx;
  cudaMalloc(&M, (size_t)rows * ld * 8);
  cudaMemset(M, 0, (size_t)rows * ld * 8);
  cudaMalloc(&idx, n_idx * 4);
  int* h = new int[n_idx];
  uint64_t x = 88172645463325252ull;
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t i = 0; i < n_idx; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      if (pass == 0) h[i] = (int)(x % rows);
      else {  // Zipf(1) by inversion of the harmonic CDF (approximate)
        const double u = (double)(x >> 11) * 0x1.0p-53;
        int j = (int)(exp(u * log((double)rows + 1.0)) - 1.0);
        h[i] = j < 0 ? 0 : (j >= rows ? rows - 1 : j);
      }
    }
    cudaMemcpy(idx, h, n_idx * 4, cudaMemcpyHostToDevice);
    for (int cg = 0; cg < 2; ++cg) {
      if (cg) gather_rows<true><<<148 * 8, 256>>>(M, rows, ld, idx, n_idx, out);
      else gather_rows<false><<<148 * 8, 256>>>(M, rows, ld, idx, n_idx, out);
      cudaEventRecord(a);
      if (cg) gather_rows<true><<<148 * 8, 256>>>(M, rows, ld, idx, n_idx, out);
      else gather_rows<false><<<148 * 8, 256>>>(M, rows, ld, idx, n_idx, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("gather %s rows 800 B, %s indices: %.3f ms for 20M rows = %.2f TB/s of row bytes\n",
             cg ? ".cg (L2)  " : "default   ", pass ? "Zipf   " : "uniform", ms,
             (double)n_idx * 800 / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
