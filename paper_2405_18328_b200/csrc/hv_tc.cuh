// hv_tc.cuh — tcgen05 / TMEM / TMA fused H.V, see hv_tc.cu.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

#include "kernels.cuh"

namespace wgp {

// Tensor-core operand set derived from the prepared points: per point the
// augmented rows a_i = [x_i, |x_i|^2, 1, 0...] and b_j = [-2 x_j, 1, |x_j|^2, 0...]
// (so a_i . b_j = u_ij^2 comes out of one MMA), each split into tf32 hi + lo.
struct TcWorkspaces;
struct TcOperands {
  bool valid = false;
  int64_t n = 0, n_pad = 0;
  int d = 0;
  void* a_hi = nullptr;  // [n_pad][32] fp32 (tf32-rounded)
  void* a_lo = nullptr;
  void* b_hi = nullptr;
  void* b_lo = nullptr;
  void* sq = nullptr;    // [n_pad] fp32 |x|^2 (diagonal fix)
  // Packed Gram (d + 2 <= 21): the 64 floats [a_hi | a_hi | a_lo] (A) and
  // [b_hi | b_lo | b_hi] (B), each segment d + 2 wide, split over the two
  // planes (K 0..31 in *_hi, 32..63 in *_lo); MMA-1 then takes nk1 =
  // ceil(3 (d + 2) / 8) K steps instead of 12 MMAs.  0: the hi / lo planes.
  int nk1 = 0;
  size_t bytes = 0;
  TcWorkspaces* ws = nullptr;  // per-launch scratch (V planes, gathered rows, split partials)
  // Kernel timing (wgp_profile): CUDA events around every hv_tc_kernel launch.
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  double profile_ms(int* launches);  // sums and releases the recorded events
  void invalidate() { valid = false; }
  void build(const float* xs, int64_t n, int dp, int d, cudaStream_t st);
  ~TcOperands();
};

bool hv_tc_supported(int d, int s);
// Gram (MMA-1) in 3xTF32; K.V (MMA-2) in 3xTF32 (bf16 = false, ~2^-21 per
// product) or bf16x3 (bf16 = true, ~2^-17, half the tensor work); fp32
// accumulation in chunks of 1024 points summed at higher precision.
void hv_tc(TcOperands& ops, const HvParams& p, cudaStream_t st, bool bf16);

// Shared host helpers of the tcgen05 kernels (hv_tc.cu, grad_tc.cu): a 2D
// fp32 TMA map with 128-byte swizzle (box_in x box_out elements) and the SM count.
CUtensorMap tc_tensor_map(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                          uint32_t box_out);
int tc_sm_count();

}  // namespace wgp
