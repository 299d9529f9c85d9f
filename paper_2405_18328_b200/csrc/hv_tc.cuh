// hv_tc.cuh — tcgen05 / TMEM / TMA fused H.V (3xTF32), see hv_tc.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
  size_t bytes = 0;
  TcWorkspaces* ws = nullptr;  // per-launch scratch (V planes, gathered rows, split partials)
  void invalidate() { valid = false; }
  void build(const float* xs, int64_t n, int dp, int d, cudaStream_t st);
  ~TcOperands();
};

bool hv_tc_supported(int d, int s);
// bf16 = false: 3xTF32 K.V (~2^-21 per product); true: bf16x3 K.V (kind::f16,
// half the tensor work, ~2^-17 per product).  The Gram (MMA-1) is 3xTF32 in both.
void hv_tc(TcOperands& ops, const HvParams& p, cudaStream_t st, bool bf16);

}  // namespace wgp
