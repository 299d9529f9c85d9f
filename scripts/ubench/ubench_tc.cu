// Microbenchmark: cost of tcgen05.mma issue vs execution, commits and
// mbarrier waits on one SM (kind::tf32, M=128).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tc ubench_tc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p) {
  const uint32_t a = su32(p);
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void ts3_e(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p, t, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n setp.eq.u32 t, 0, 0;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, t;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, t;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_e(uint64_t* b) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(128, 1) bench(int mode, int n, int N, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar, dummy;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&dummy)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (mode >= 4 && threadIdx.x < 32) {
    const uint32_t id = idesc(128, N);
    const uint64_t bd = desc(sm);
    long long t0 = clock64();
    if (mode == 4) {
      for (int i = 0; i < n; ++i) ts_e(tm, tm + 256 + 8 * (i & 7), bd + 2 * (i & 3), id, i > 0);
    } else {
      for (int i = 0; i < n; i += 3) {
        ts3_e(tm, tm + 256 + 8 * (i & 7), bd + 2 * (i & 3), id, i > 0);
        if (mode == 6) commit_e(&dummy);
      }
    }
    long long t1 = clock64();
    commit_e(&bar);
    wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (mode < 4 && threadIdx.x == 0) {
    const uint32_t id = idesc(128, N);
    const uint64_t bd = desc(sm), ad = desc(sm + 32768);
    // pre-arm dummy so try_wait(0) on it is already complete after one arrive
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&dummy)) : "memory");
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      if (mode == 0 || mode == 2 || mode == 3) ts(tm, tm + 256 + 8 * (i & 7), bd + 2 * (i & 3), id, i > 0);
      else ss(tm, ad + 2 * (i & 3), bd + 2 * (i & 3), id, i > 0);
      if (mode == 2 && (i % 3) == 2) commit(&dummy);
      if (mode == 3 && (i % 3) == 2) { wait(&dummy, 0); asm volatile("tcgen05.fence::after_thread_sync;"); }
    }
    long long t1 = clock64();
    commit(&bar);
    wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const char* names[] = {"TS (A tmem)", "SS (A smem)", "TS + commit/3", "TS + trywait/3", "warp TS elect", "warp TS x3", "warp TS x3+cmt"};
  for (int mode = 0; mode < 7; ++mode)
    for (int N : {16, 64, 80, 128, 256}) {
      const int n = 240;
      bench<<<1, 128, 70 * 1024>>>(mode, n, N, d);
      bench<<<1, 128, 70 * 1024>>>(mode, n, N, d);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      cudaError_t e = cudaGetLastError();
      printf("%-16s N=%3d  issue %6.1f clk/mma  complete %6.1f clk/mma  floor %5.1f  %s\n", names[mode], N,
             (double)h[0] / n, (double)h[1] / n, 128.0 * N / 256.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
