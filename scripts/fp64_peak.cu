// FP64 peak microbenchmark on B200: vector DFMA and tensor-core DMMA
// (mma.sync.m8n8k4.f64) throughput with independent accumulator chains.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

// both pipes at once: 8 DFMA chains and 4 DMMA chains per thread
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  double x[8], d[4][2];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    const int blocks = sms * 8, threads = 256;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s\n", flop / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters / 4, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop2 = 2.0 * 256 * 8 * (iters / 4) * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", flop2 / (ms * 1e-3) / 1e12);
    const int mit = iters / 8;
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(out, mit, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f_dfma = 2.0 * 32 * mit * (double)blocks * threads;
    const double f_dmma = 2.0 * 256 * 4 * mit * (double)blocks * (threads / 32);
    printf("mixed: %.2f TFLOP/s total (DFMA part %.2f, DMMA part %.2f)\n", (f_dfma + f_dmma) / (ms * 1e-3) / 1e12,
           f_dfma / (ms * 1e-3) / 1e12, f_dmma / (ms * 1e-3) / 1e12);
  }
  return 0;
}
