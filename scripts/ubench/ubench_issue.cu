// Microbenchmark 4: tcgen05.mma issue throughput per instruction for the
// hv_tc shapes, back to back (no waits), from one warp or two warps at once.
//   shapes: tf32 TS M=128 K=8 with N = 32, 64, 80, 128, 256; bf16 TS N=80 K=16
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p) {
  const uint32_t a = su32(p);
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t id_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t id_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int KIND>
__device__ __forceinline__ void mma8(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  if (KIND == 0)
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                 " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
                 " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
                 " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
                 " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(id));
  else
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                 " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
                 " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
                 " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
                 " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void commit_wait(uint64_t* b, uint32_t& ph) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(su32(b)) : "memory");
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  ph ^= 1;
}

// warps 0 and (if two) 1 each issue `iters` x 4 MMAs of (kind, N) into their own D columns
__global__ void __launch_bounds__(128, 1) bench(int kind, int N, int two, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  const uint64_t db = desc(sm + (warp ? 32768 : 0));
  const uint32_t id = kind == 0 ? id_tf32(128, N) : id_bf16(128, N);
  if (warp < 1 + two) {
    uint32_t ph = 0;
    const uint32_t d = tm + (warp ? 256 : 0);
    const uint32_t a = tm + 384 + (warp ? 64 : 0);
    commit_wait(&bar[warp], ph);
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (kind == 0) mma8<0>(d, a, db, id); else mma8<1>(d, a, db, id);
    }
    const long long t1 = clock64();
    commit_wait(&bar[warp], ph);
    const long long t2 = clock64();
    if (threadIdx.x % 32 == 0) {
      out[warp * 2 + 0] = t1 - t0;  // issue
      out[warp * 2 + 1] = t2 - t0;  // complete
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int iters = 256;  // x4 MMAs
  struct S { int kind, N; } shapes[] = {{0, 32}, {0, 64}, {0, 80}, {0, 128}, {0, 256}, {1, 80}, {1, 128}};
  for (auto sh : shapes) {
    for (int two = 0; two < 2; ++two) {
      cudaMemset(d, 0, 64);
      bench<<<1, 128, 70000>>>(sh.kind, sh.N, two, iters, d);
      long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      const double n = 4.0 * iters;
      const double macs = 128.0 * sh.N * (sh.kind == 0 ? 8 : 16);
      printf("%s N=%3d %s: issue %.1f clk/instr, complete %.1f clk/instr (%.0f MAC/clk)%s", sh.kind ? "bf16" : "tf32",
             sh.N, two ? "2 warps" : "1 warp ", h[0] / n, h[1] / n, macs / (h[1] / n),
             two ? "" : "\n");
      if (two) printf("  | warp1 complete %.1f clk/instr\n", h[3] / n);
    }
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
