// fp64_peak.cu -- measures the B200 FP64 ceilings the roofline uses:
// DFMA (CUDA cores) and DMMA.8x8x4 (mma.sync f64) throughput, full chip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double s) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], s, 1e-7);
  double t = 0;
  for (int k = 0; k < 8; ++k) t += a[k];
  if (t == 12345.0) out[threadIdx.x] = t;
}

__global__ void dmma_kernel(double* out, int iters) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double t = 0;
  for (int k = 0; k < 8; ++k) t += c[k][0] + c[k][1];
  if (t == 12345.0) out[threadIdx.x] = t;
}

template <int NACC>
__global__ void dmma_occ(double* out, int iters) {
  double c[NACC][2];
  for (int k = 0; k < NACC; ++k) c[k][0] = c[k][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
          : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double t = 0;
  for (int k = 0; k < NACC; ++k) t += c[k][0] + c[k][1];
  if (t == 12345.0) out[threadIdx.x] = t;
}

template <int NACC>
void occ_sweep(double* out, int sms, cudaEvent_t a, cudaEvent_t b) {
  for (int bps : {1, 2, 4, 8}) {
    const int blocks = sms * bps, iters = 4000;
    dmma_occ<NACC><<<blocks, 128>>>(out, 10);
    cudaEventRecord(a);
    dmma_occ<NACC><<<blocks, 128>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 256 * NACC * double(iters) * blocks * 4;
    printf("DMMA occupancy: %2d warps/SM, %2d independent acc/warp: %.2f TFLOP/s\n", 4 * bps, NACC,
           flops / ms / 1e9);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    const int blocks = sms * (2048 / threads);
    dfma_kernel<<<blocks, threads>>>(out, 100, 0.999);
    cudaEventRecord(a);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 8 * iters * double(blocks) * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    const int blocks = sms * (1024 / threads);
    dmma_kernel<<<blocks, threads>>>(out, 100);
    cudaEventRecord(a);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 256 * 8 * iters * double(blocks) * (threads / 32);
    printf("DMMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  occ_sweep<4>(out, sms, a, b);
  occ_sweep<8>(out, sms, a, b);
  occ_sweep<16>(out, sms, a, b);
  occ_sweep<24>(out, sms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d max_clock=%d MHz err=%s\n", sms, clk / 1000, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
