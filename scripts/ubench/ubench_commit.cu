// Microbenchmark 3: tcgen05.commit cost and latency (one CTA).
//   mode 0: commit (nothing outstanding) -> wait, round trip
//   mode 1: 8 back-to-back commits to 8 barriers: issue clk per commit, then wait all
//   mode 2: one bf16 M=128 N=80 K=16 TS MMA x3 + commit -> wait, round trip
//   mode 3: plain mbarrier.arrive -> wait round trip (same warp)
//   mode 4: as 0 while a second warp streams MMAs (tensor pipe busy)
//   mode 5: as 1 while a second warp streams MMAs
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p) {
  const uint32_t a = su32(p);
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t id_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void ts3_f16(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void commit_e(uint64_t* b) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void arrive_e(uint64_t* b) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(128, 1) bench(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[8], bar_bg;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bars[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar_bg)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    stop = 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  const uint64_t db = desc(sm);
  const uint32_t id = id_bf16(128, 80);
  if (warp == 1 && (mode == 4 || mode == 5)) {
    // background MMA stream into columns [256, 336)
    while (!stop) {
      ts3_f16(tm + 256, tm + 384, db, id);
    }
  }
  if (warp == 0) {
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tot = 0, tot2 = 0;
    for (int it = 0; it < iters; ++it) {
      __syncwarp();
      const long long t0 = clock64();
      if (mode == 0 || mode == 4) {
        commit_e(&bars[0]);
        wait(&bars[0], ph[0]);
        ph[0] ^= 1;
      } else if (mode == 1 || mode == 5) {
        for (int k = 0; k < 8; ++k) commit_e(&bars[k]);
        const long long t1 = clock64();
        tot2 += t1 - t0;
        for (int k = 0; k < 8; ++k) {
          wait(&bars[k], ph[k]);
          ph[k] ^= 1;
        }
      } else if (mode == 2) {
        ts3_f16(tm, tm + 128, db, id);
        commit_e(&bars[0]);
        wait(&bars[0], ph[0]);
        ph[0] ^= 1;
      } else if (mode == 3) {
        arrive_e(&bars[0]);
        wait(&bars[0], ph[0]);
        ph[0] ^= 1;
      }
      tot += clock64() - t0;
    }
    if (threadIdx.x == 0) {
      out[0] = tot / iters;
      out[1] = tot2 / iters;
      stop = 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  const char* names[] = {"commit->wait round trip (idle pipe)", "8 commits: total issue clk / round trip",
                         "3 MMA + commit -> wait", "plain arrive -> wait", "commit->wait, pipe busy",
                         "8 commits issue / round trip, pipe busy"};
  for (int mode = 0; mode < 6; ++mode) {
    bench<<<1, 128, 40960>>>(mode, 200, d);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    printf("mode %d %-45s %lld clk (issue part %lld)  %s\n", mode, names[mode], h[0], h[1],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
