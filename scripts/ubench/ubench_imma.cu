// Warp-level MMA throughput on B200 (sm_100a): int8 m16n8k32 (s32 accumulate)
// vs fp64 m16n8k8 -- sizing an exact integer-slice fp64 operator.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_imma ubench_imma.cu
#include <cstdio>
#include <cstdint>
constexpr int IT = 2048, CH = 8;
__global__ void __launch_bounds__(256, 2) imma(int* out, long long* clk) {
  int acc[CH][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x1234, b1 = a0 ^ 0x4321;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                   : "r"(a0 + c), "r"(a1), "r"(a2), "r"(a3), "r"(b0 ^ c), "r"(b1));
  }
  long long t1 = clock64();
  int s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void __launch_bounds__(256, 2) dmma(double* out, long long* clk) {
  double acc[CH][4] = {};
  double a[4] = {1.0 + threadIdx.x, 2.0, 3.0, 4.0}, b0 = 0.5, b1 = 0.25;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < IT / 4; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                   : "d"(a[0] + c), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0 + c), "d"(b1));
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  int* oi; double* od; long long* clk;
  const int G = 148 * 8;  // 8 CTAs of 256 per SM worth of work, 2 resident
  cudaMalloc(&oi, G * 256 * 4); cudaMalloc(&od, G * 256 * 8); cudaMalloc(&clk, G * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    imma<<<G, 256>>>(oi, clk);
    cudaEventRecord(e0); imma<<<G, 256>>>(oi, clk); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mi = double(G) * 8 * IT * CH * 16 * 8 * 32;
    printf("IMMA m16n8k32 u8*s8: %.1f TOPS (%.0f MAC/clk/SM at 1965 MHz) %s\n", 2 * mi / ms / 1e9,
           mi / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    dmma<<<G, 256>>>(od, clk);
    cudaEventRecord(e0); dmma<<<G, 256>>>(od, clk); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double md = double(G) * 8 * (IT / 4) * CH * 16 * 8 * 8;
    printf("DMMA m16n8k8 f64:    %.1f TFLOP/s (%.0f MAC/clk/SM)\n", 2 * md / ms / 1e9, md / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
