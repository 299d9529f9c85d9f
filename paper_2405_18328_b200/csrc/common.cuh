// common.cuh — shared device helpers for the warmgp B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace wgp {

// Errors carry the reference's exception classes (proj/include/warmgp/common.hpp:13-22).
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

#define WGP_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t err__ = (call);                                                          \
    if (err__ != cudaSuccess)                                                            \
      throw ::wgp::DeviceError(std::string("CUDA error ") + cudaGetErrorString(err__) + \
                               " at " + __FILE__ + ":" + std::to_string(__LINE__));      \
  } while (0)

// Every kernel launch of the library is followed by WGP_LAUNCH_CHECK, which
// also counts it (wgp_launch_count: bench.py's gpu_launches).
std::atomic<uint64_t>& launch_counter();
// Bumped whenever a device workspace is (re)allocated: captured CUDA graphs
// bake buffer addresses in and are re-captured when this changes.
std::atomic<uint64_t>& alloc_generation();
#define WGP_LAUNCH_CHECK()                                                   \
  do {                                                                       \
    ::wgp::launch_counter().fetch_add(1, std::memory_order_relaxed);         \
    WGP_CUDA(cudaGetLastError());                                            \
  } while (0)

// Opt a kernel into `bytes` of dynamic shared memory once per device (the
// attribute belongs to the device's copy of the kernel: a process driving two
// GPUs through two contexts must set it on each).
#define WGP_SMEM_ATTR(kernel, bytes)                                                            \
  do {                                                                                          \
    static std::atomic<unsigned long long> mask__{0};                                           \
    int dev__ = 0;                                                                              \
    WGP_CUDA(cudaGetDevice(&dev__));                                                            \
    const unsigned long long bit__ = 1ull << (dev__ & 63);                                      \
    if (!(mask__.load(std::memory_order_acquire) & bit__)) {                                    \
      WGP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)); \
      mask__.fetch_or(bit__, std::memory_order_acq_rel);                                        \
    }                                                                                           \
  } while (0)

constexpr double kSqrt3 = 1.7320508075688772;
constexpr double kLog2e = 1.4426950408889634;
constexpr double kLn2 = 0.6931471805599453;

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// 2^x for x <= 0 on the FMA/ALU pipes (no MUFU): round-to-nearest split
// x = n + f via the 1.5*2^23 magic constant (no F2I), degree-5 minimax
// polynomial for 2^f on [-1/2, 1/2] (max rel. error 2.4e-7 in fp32 Horner,
// the same order as ex2.approx), exponent add for 2^n.  Used for half the
// entries of the tensor-core epilogue so the MUFU pipe stops binding (FA4).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const int n = __float_as_int(t) - 0x4B400000;
  float p = 1.3276466634e-3f;
  p = fmaf(p, f, 9.6755409613e-3f);
  p = fmaf(p, f, 5.5507134646e-2f);
  p = fmaf(p, f, 2.4022120237e-1f);
  p = fmaf(p, f, 6.9314694405e-1f);
  p = fmaf(p, f, 1.0000001192f);
  return __int_as_float(__float_as_int(p) + (n << 23));
}

// Matern-3/2 value from u = sqrt(3) * log2(e) * r (the scaled distance the
// kernels carry): k = sf^2 (1 + sqrt3 r) exp(-sqrt3 r) = (a u + sf^2) 2^-u,
// a = sf^2 ln 2.  (proj/src/kernel.cpp:79-93, 130-134)
__device__ __forceinline__ float matern_from_u(float u, float sf2, float a) {
  return fmaf(a, u, sf2) * ex2_approx(-u);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace wgp
