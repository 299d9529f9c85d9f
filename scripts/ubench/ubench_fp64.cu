// DFMA and DMMA (mma.sync m8n8k4 f64) throughput on one B200 (dev micro-benchmark).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 42.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2];
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
  if (s == 42.0) out[0] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  double acc[4][4];
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0, b1 = 2.0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  double s = 0;
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  if (s == 42.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    const int blocks = sms * 2;
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * iters * double(blocks) * threads;
    printf("DFMA  threads %4d: %.2f TFLOP/s  (%.1f DFMA/clk/SM at %d MHz)\n", threads, flops / ms / 1e9,
           flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mflops = 2.0 * 8 * 8 * 4 * 4 * iters * double(blocks) * (threads / 32);
    printf("DMMA m8n8k4  threads %4d: %.2f TFLOP/s\n", threads, mflops / ms / 1e9);
    dmma16_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    dmma16_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double m16 = 2.0 * 16 * 8 * 8 * 4 * iters * double(blocks) * (threads / 32);
    printf("DMMA m16n8k8 threads %4d: %.2f TFLOP/s  err=%s\n", threads, m16 / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
