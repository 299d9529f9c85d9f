// Microbenchmark 2: the MMA shapes of hv_tc, alone and concurrently.
//   M1: SS kind::tf32 M=128 N=64 (A and B in smem)     floor 32 clk
//   M2: TS kind::f16 (bf16) M=128 N=80 (A in TMEM)     floor 40 clk
//   M2t: TS kind::tf32 M=128 N=80                      floor 40 clk
// modes: 0 M1 alone, 1 M2 alone, 2 M2t alone, 3 M1 || M2 (two warps),
//        4 M1 || M2 + 8 warps streaming tcgen05.ld/st, 5 M2 + 8 warps ld/st
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
__device__ __forceinline__ void ss3(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void ts3_f16(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void ts3_tf32(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n"
               " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n"
               :: "r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void commit_e(uint64_t* b) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(384, 1) bench(int mode, int iters, long long* out, int* flag) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar1, bar2;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar1)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const bool m1 = (mode == 0 || mode == 3 || mode == 4);
  const bool m2 = (mode == 1 || mode == 3 || mode == 4 || mode == 5);
  if (warp == 0 && m1) {
    const uint64_t ad = desc(sm), bd = desc(sm + 32768);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      for (int k = 0; k < 4; ++k) ss3(tm + 128, ad + 2 * k, bd + 2 * k, id_tf32(128, 64));
    commit_e(&bar1);
    wait(&bar1, 0);
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  } else if (warp == 1 && (m2 || mode == 2)) {
    const uint64_t vd = desc(sm + 65536);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      for (int k = 0; k < 4; ++k) {
        if (mode == 2) ts3_tf32(tm, tm + 256 + 8 * k, vd + 2 * k, id_tf32(128, 80));
        else ts3_f16(tm, tm + 256 + 8 * k, vd + 2 * k, id_bf16(128, 80));
      }
    commit_e(&bar2);
    wait(&bar2, 0);
    if (threadIdx.x == 32) out[1] = clock64() - t0;
  } else if (warp >= 4 && (mode == 4 || mode == 5)) {
    // 8 warps streaming TMEM ld/st like the epilogue (their own columns 384..447)
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col = 384 + 32 * ((warp - 4) >> 2);
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    for (int i = 0; i < iters * 2; ++i) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(tm + lanes + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   :: "r"(tm + lanes + col), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

int main() {
  long long* d;
  int* f;
  cudaMalloc(&d, 32);
  cudaMalloc(&f, 4);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[] = {"M1 SS tf32 N64", "M2 TS bf16 N80", "M2 TS tf32 N80", "M1 || M2", "M1||M2 + ld/st", "M2 + ld/st"};
  const int iters = 200;
  for (int mode = 0; mode < 6; ++mode) {
    cudaMemset(d, 0, 32);
    bench<<<1, 384, 100 * 1024>>>(mode, iters, d, f);
    bench<<<1, 384, 100 * 1024>>>(mode, iters, d, f);
    long long h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    // per "tile": M1 = 12 MMAs, M2 = 12 MMAs
    printf("%-16s  M1 warp %7.1f clk/tile  M2 warp %7.1f clk/tile   (floors: M1 384, M2 480) %s\n", names[mode],
           (double)h[0] / iters, (double)h[1] / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
