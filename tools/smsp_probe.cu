// Development probe: which warps share an SM sub-partition's FP64 pipe?
// One CTA of 16 warps per SM.  "Chain" warps time a dependent DFMA chain
// while the other warps stream independent DMMAs.  Mode 0: chain warps are
// those with %warpid % 4 == 0; mode 1: CTA warp index % 4 == 0; mode 2: no
// DMMA streams (idle reference).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int mode, double* out, long long* cyc) {
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 32 warps per CTA (8 per SMSP).  mode 3: warps on SMSP 0 only, half
  // chain / half DMMA; mode 4: chain on SMSP 0, DMMA on SMSP 1.
  bool chain = mode == 0 ? (wid % 4 == 0) : (warp % 4 == 0);
  bool dmma = !chain;
  if (mode == 3) { chain = wid % 4 == 0 && (wid / 4) % 2 == 0; dmma = wid % 4 == 0 && !chain; }
  if (mode == 4) { chain = wid % 4 == 0; dmma = wid % 4 == 1; }
  double x = lane * 1e-3 + 1.0, y = 0.999999;
  if (chain) {
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) x = fma(x, y, 1e-9);
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = (t1 - t0);
  } else if (mode != 2 && dmma) {
    double d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4096; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d0[k]), "+d"(d1[k]) : "d"(x), "d"(y));
    x = d0[0] + d0[1] + d0[2] + d0[3] + d1[0] + d1[1] + d1[2] + d1[3];
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = -1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 32 * 8);
  long long h[148 * 32];
  for (int mode = 0; mode < 5; ++mode) {
    cudaMemset(cyc, 0, sizeof h);
    probe<<<148, 1024>>>(mode, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0; int n = 0;
    for (int i = 0; i < 148 * 32; ++i) if (h[i] > 0) { s += h[i] / 4096.0; ++n; }
    printf("mode %d (%s): %d chain warps, %.1f cycles per dependent DFMA\n", mode,
           mode == 0 ? "chain = %warpid%4==0" : mode == 1 ? "chain = warp index%4==0" : mode == 2 ? "idle" : mode == 3 ? "chain+dmma both on SMSP0" : "chain SMSP0, dmma SMSP1", n, s / n);
  }
  return 0;
}
