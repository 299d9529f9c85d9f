// common.cuh — shared device helpers for the warmgp B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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

#define WGP_LAUNCH_CHECK() WGP_CUDA(cudaGetLastError())

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
