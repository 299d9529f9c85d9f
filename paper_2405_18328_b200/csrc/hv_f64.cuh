// hv_f64.cuh — fp64-accumulating fused H.V (the fp64 CG operator; hv_f64.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wgp {

enum : int { kHv64Store = 0, kHv64Residual = 1 };

struct Hv64Params {
  const float* xs;    // [n_pad][dp] prepared points (kernels.cuh)
  int64_t n;          // points (contracted over all of them)
  int dp;             // padded dimension (row stride of xs, multiple of 4)
  int d;              // dimension
  int64_t r0, m;      // output rows [r0, r0 + m) (global)
  const double* V;    // V[j + c ldv], global j
  int64_t ldv;
  int s;
  double* out;        // out[r + c ldo], r local
  int64_t ldo;
  const double* B;    // residual mode: B[global row + c ldb]
  int64_t ldb;
  int mode;
  const float* hyp;   // device [sf2, a, diag]
  const int* done;    // optional: skip when *done != 0
  double* part;       // workspace, hv64_workspace_bytes(n, m, s)
};

int hv64_splits(int64_t n);
size_t hv64_workspace_bytes(int64_t n, int64_t m, int s);  // per launch of <= 80 columns
void hv64(const Hv64Params& p, cudaStream_t st);
// Exact integer-slice engine (hv_i8.cu): d <= 16, s <= 80; writes the fp64
// split partials into p.part (hv_i8_workspace_bytes: partials + V byte images).
bool hv_i8_supported(int d, int s);
size_t hv_i8_workspace_bytes(int64_t n, int64_t m, int s);
bool hv_i8_partials(const Hv64Params& p, cudaStream_t st, int* splits, int64_t* m_pad);
// The kernel only (s <= 80 columns): p.part holds the fp64 split partials
// part[(k s + c) m_pad + r], k < *splits, for the caller to sum in split
// order (cg_fused_cl); false (nothing launched) for wider V.
bool hv64_partials(const Hv64Params& p, cudaStream_t st, int* splits, int64_t* m_pad);

}  // namespace wgp
