// FMA-pipe throughput on sm_100a: scalar FFMA vs packed FFMA2 vs a 1:1 mix
// (does scalar FFMA run on the fma-lite half while FFMA2 occupies fma-heavy?).
// 8 independent chains per thread, 16 warps per SM, clock64 per CTA.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* clk, int iters, float s) {
  float a[8];
  float2 b[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i, b[i] = make_float2(a[i], a[i] + 1.f);
  const float2 s2 = make_float2(s, s);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { a[i] = fmaf(a[i], s, 0.5f); a[i] = fmaf(a[i], s, 0.25f); }
      if (MODE == 1) { b[i] = __ffma2_rn(b[i], s2, s2); }
      if (MODE == 2) { b[i] = __ffma2_rn(b[i], s2, s2); a[i] = fmaf(a[i], s, 0.5f); }
      if (MODE == 3) { b[i] = __ffma2_rn(b[i], s2, s2); a[i] = __fmul_rn(a[i], s); }
      if (MODE == 4) { b[i] = __ffma2_rn(b[i], s2, s2); a[i] = __fadd_rn(a[i], s); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float r = 0.f;
  for (int i = 0; i < 8; ++i) r += a[i] + b[i].x + b[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, double ops_per_iter_thread) {
  const int blocks = 148, threads = 512, iters = 4096;
  float* out; long long* clk;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&clk, blocks * 8);
  k<MODE><<<blocks, threads>>>(out, clk, 16, 0.999f);
  k<MODE><<<blocks, threads>>>(out, clk, iters, 0.999f);
  long long h[148]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < blocks; ++i) m += h[i]; m /= blocks;
  const double ops = ops_per_iter_thread * iters * threads;  // fp32 FMA-ops per SM
  printf("%-28s %8.1f fp32 ops/clk/SM  (%.2f warp-instr/clk/SM)\n", name, ops / m,
         (MODE == 0 ? 16.0 : MODE == 1 ? 8.0 : 16.0) * iters * (threads / 32) / m);
  cudaFree(out); cudaFree(clk);
}

int main() {
  run<0>("FFMA only", 16);
  run<1>("FFMA2 only", 16);
  run<2>("FFMA2 + FFMA 1:1", 24);
  run<3>("FFMA2 + FMUL 1:1", 24);
  run<4>("FFMA2 + FADD 1:1", 24);
  return 0;
}
