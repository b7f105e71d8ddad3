// Microbenchmark: dependent-chain latencies on the B200 (one warp per SM,
// optionally with DMMA load from other warps).  nvcc -arch=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void lat(double* out, long long* cyc, int n, int mode) {
  const int warp = threadIdx.x >> 5;
  double x = out[threadIdx.x], y = 1.0000001, z = 0.5;
  if (warp > 0) {  // background DMMA load (mode 1) or idle
    if (mode == 1) {
      double a0 = 0, a1 = 0, b0 = 0, b1 = 0, c0 = 0, c1 = 0, e0 = 0, e1 = 0;
      for (int i = 0; i < n * 4; ++i) { dmma(a0, a1, x, y); dmma(b0, b1, x, z); dmma(c0, c1, y, z); dmma(e0, e1, z, x); }
      out[threadIdx.x + 4096] = a0 + b1 + c0 + e1 + a1 + b0 + c1 + e0;
    }
    return;
  }
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, z);                 // DFMA chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;                        // DMUL chain
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + z; }  // MUFU + DADD
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31) + z;   // SHFL(2x) + DADD
  long long t4 = clock64();
  double c0 = x, c1 = z;
  for (int i = 0; i < n; ++i) dmma(c0, c1, y, z);               // DMMA chain
  long long t5 = clock64();
  volatile double* sp; __shared__ double sm[64]; sm[threadIdx.x & 63] = x; __syncwarp();
  double v = x; int idx = threadIdx.x & 31;
  for (int i = 0; i < n; ++i) { v = sm[idx]; idx = (int)(v) & 31; }  // LDS chain
  long long t6 = clock64();
  out[threadIdx.x] = x + c0 + c1 + v;
  if (threadIdx.x == 0) { cyc[blockIdx.x * 8 + 0] = t1 - t0; cyc[blockIdx.x * 8 + 1] = t2 - t1; cyc[blockIdx.x * 8 + 2] = t3 - t2;
    cyc[blockIdx.x * 8 + 3] = t4 - t3; cyc[blockIdx.x * 8 + 4] = t5 - t4; cyc[blockIdx.x * 8 + 5] = t6 - t5; }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1 << 16);
  cudaMemset(out, 0, 1 << 20);
  const int n = 1000;
  const char* names[] = {"DFMA", "DMUL", "MUFU.RCP64H+DADD", "SHFL.f64+DADD", "DMMA", "LDS"};
  for (int mode = 0; mode < 2; ++mode) for (int warps : {1, 4, 16}) {
    lat<<<148, 32 * warps>>>(out, cyc, n, mode);
    lat<<<148, 32 * warps>>>(out, cyc, n, mode);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %s warps %2d:", mode ? "dmma-load" : "idle     ", warps);
    for (int k = 0; k < 6; ++k) printf("  %s %.1f", names[k], (double)h[k] / n);
    printf("\n");
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
