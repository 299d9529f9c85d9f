// Microbenchmark 7: does a warp issuing back-to-back tcgen05.mma slow the
// other warps of its SMSP?  (16 warps: 1..3 idle, 4..15 three per SMSP.)  Warp 0 issues MMAs (tf32 TS M=128 N=64 K=8, or
// f16 N=80 K=16) for the whole run; warps 1..7 run an epilogue-like MUFU/FMA
// loop and time themselves.  Warp 4 shares SMSP 0 with warp 0.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p) {
  const uint32_t a = su32(p);
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma8(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id));
}
__global__ void __launch_bounds__(512, 1) bench(int mma_on, int N, int iters, int work, long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  const long long t0 = clock64();
  if (warp == 0) {
    if (mma_on) {
      const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int it = 0; it < iters; ++it) mma8(tm, tm + 384, desc(sm), id);
    }
  } else if (warp >= 4) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = 1.0f + 0.01f * (threadIdx.x + i);
    for (int it = 0; it < work; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float u;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(u) : "f"(x[i]));
        float e;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-u));
        x[i] = fmaf(fmaf(0.69f, u, 1.0f), e, x[i]);
      }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.f) sink[threadIdx.x] = s;
  }
  const long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}
int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 64 * 16);
  cudaMalloc(&sink, 1024 * 4);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const int Ns[] = {0, 32, 64, 128, 256};
  for (int mode = 0; mode < 5; ++mode) {
    const int N = Ns[mode];
    bench<<<1, 512, 40000>>>(mode > 0, N > 0 ? N : 64, N > 0 ? 4000 * 64 / N : 0, 400, d, sink);
    long long h[16];
    cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("mma N=%3d: MMA warp %lld clk | epilogue-like warps:", N, h[0]);
    for (int w = 4; w < 16; ++w) printf(" w%d(smsp%d)=%lld", w, w & 3, h[w]);
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
