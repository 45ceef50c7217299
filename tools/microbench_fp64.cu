// Microbenchmark: FP64 throughput on this GPU -- DFMA (CUDA cores) and DMMA
// (mma.sync m8n8k4 f64). Prints TFLOP/s. Used to size the router's roofline.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

// half the warps on DMMA, half on DFMA: do the two FP64 pipes add up?
__global__ void mixed_kernel(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 1.0000001, 1e-9);
    }
    for (int i = 0; i < 8; ++i) s += a[i];
  } else {
    double d[8][2];
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    dfma_kernel<<<sms * 2, 32 * warps / 2>>>(out, 16);
    cudaEventRecord(e0);
    dfma_kernel<<<sms * 2, 32 * warps / 2>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)sms * 2 * 32 * warps / 2;
    printf("DFMA warps/SM=%2d : %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    dmma_kernel<<<sms * 2, 32 * warps / 2>>>(out, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<sms * 2, 32 * warps / 2>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 8 * iters * (double)sms * 2 * warps / 2;
    printf("DMMA warps/SM=%2d : %.1f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  {
    const int iters = 4096, warps = 16;
    mixed_kernel<<<sms * 2, 32 * warps / 2>>>(out, 16);
    cudaEventRecord(e0);
    mixed_kernel<<<sms * 2, 32 * warps / 2>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per SM: 8 DMMA warps x iters x 8 x 256 FMA + 8 DFMA warps x 4*iters x 8 x 32 FMA
    double fl = 2.0 * (double)sms * 2 * (4.0 * iters * 8 * 256 + 4.0 * 4 * iters * 8 * 32);
    printf("MIXED DMMA+DFMA : %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  }
  return 0;
}
