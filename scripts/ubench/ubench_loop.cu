// Microbenchmark 8: per-iteration cost of the MMA warp's control ops, one warp
// alone: try_wait on an already-completed phase, tcgen05.fence, tcgen05.commit
// (nothing outstanding), a trace store.  mode bits: 1 waits (3), 2 fences (3),
// 4 commits (2), 8 stores (7).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void test_(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void relaxed_(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void commit_(uint64_t* b) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(su32(b)) : "memory");
}
__global__ void bench(int mode, int iters, long long* out, long long* tr) {
  __shared__ __align__(8) uint64_t bar[4], cb[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[i])));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&cb[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // complete phase 0 of bar[0..3]
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&bar[i])) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode & 1) { wait_(&bar[0], 0); wait_(&bar[1], 0); wait_(&bar[2], 0); }
      if (mode & 2) { for (int k = 0; k < 3; ++k) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
      if (mode & 4) { commit_(&cb[it & 7]); commit_(&cb[(it + 4) & 7]); }
      if (mode & 16) { test_(&bar[0], 0); test_(&bar[1], 0); test_(&bar[2], 0); }
      if (mode & 32) { relaxed_(&bar[0], 0); relaxed_(&bar[1], 0); relaxed_(&bar[2], 0); }
      if (mode & 64) { wait_(&bar[0], 0); wait_(&bar[1], 0); wait_(&bar[2], 0); asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
      if (mode & 8) { if ((threadIdx.x & 31) == 0) for (int k = 0; k < 7; ++k) tr[(it & 63) * 8 + k] = clock64(); }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(slot));
}
int main() {
  long long *d, *tr;
  cudaMalloc(&d, 64);
  cudaMalloc(&tr, 64 * 8 * 8);
  for (int mode : {1, 2, 4, 8, 15, 16, 32, 64}) {
    bench<<<1, 128>>>(mode, 1000, d, tr);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %2d: %.1f clk per iteration\n", mode, h / 1000.0);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
