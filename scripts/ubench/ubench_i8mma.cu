// tcgen05.mma kind::i8 throughput with both operands in shared memory (the
// hv_i8 MMA shape: M = 128, K = 32 bytes per instruction) for 64- and
// 128-byte-swizzled K-major layouts and N = 64 .. 256: one CTA per SM, one
// thread issuing 16 MMAs per commit, 4096 MMAs timed with clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_i8mma ubench_i8mma.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(const void* p, int sw) {  // sw: 64 or 128
  const uint32_t a = smem_u32(p);
  const uint64_t sbo = sw == 128 ? 1024 : 512, lt = sw == 128 ? 2 : 4;
  return static_cast<uint64_t>((a >> 4) & 0x3FFF) | (1ull << 16) | ((sbo >> 4) << 32) | (1ull << 46) | (lt << 61);
}

template <int N, int SWA, int SWB>
__global__ void __launch_bounds__(128, 1) k(long long* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* A = s;            // 128 rows
  uint8_t* B = s + 32768;    // N rows
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = i * 2654435761u;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
    const uint64_t da = desc(A, SWA), db = desc(B, SWB);
    long long t0 = 0;
    uint32_t ph = 0;
    for (int it = 0; it < 257; ++it) {
      if (it == 1) t0 = clock64();
#pragma unroll
      for (int m = 0; m < 16; ++m)
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da + 2 * (m & 1)),
                     "l"(db + 2 * (m & 1)), "r"(idesc));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(&bar)), "r"(ph) : "memory");
      ph ^= 1u;
    }
    clk[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int SWA, int SWB>
void run() {
  long long* clk;
  cudaMalloc(&clk, 148 * 8);
  cudaFuncSetAttribute(k<N, SWA, SWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  k<N, SWA, SWB><<<148, 128, 80 * 1024>>>(clk);
  k<N, SWA, SWB><<<148, 128, 80 * 1024>>>(clk);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148;
  const double mac = 256.0 * 16 * 128 * N * 32;
  printf("N=%3d A sw%3d B sw%3d: %6.0f int8 MAC/clk/SM  (%5.1f clk per MMA)  %s\n", N, SWA, SWB, mac / m,
         m / (256.0 * 16), cudaGetErrorString(e));
  cudaFree(clk);
}

int main() {
  run<64, 64, 64>();
  run<128, 64, 64>();
  run<256, 64, 64>();
  run<64, 128, 128>();
  run<128, 128, 128>();
  run<256, 128, 128>();
  run<256, 128, 64>();
  return 0;
}
