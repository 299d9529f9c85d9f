// exact.cuh — dense fp64 exact path (proj/src/exact.cpp:25-50), see exact.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wgp {

constexpr int kExactMaxD = 30;
constexpr int64_t kDenseGuard = 20000;  // proj/include/warmgp/exact.hpp:23

// Lower triangle (and diagonal) of H = K + sigma^2 I in fp64, column-major
// n x n, from the raw inputs X (column-major fp32 n x d) with the reference's
// Gram-trick distances (kernel.cpp:101-139).
void exact_build(const float* X, int64_t n, int d, const double* inv_ls_dev, double sf2, double noise2, double* H,
                 cudaStream_t st);
// Constrained-space contractions <dH/dtheta_k, W> over the lower triangle with
// W = 1/2 alpha alpha^T - 1/2 Hinv (Hinv: lower triangle), k = lengthscales,
// signal, noise; fixed-order fp64 reductions.  out (device): d + 2 doubles as
// [sum decay*W*(dx_k/l_k)^2 ... (d), sum k*W, sum_i W_ii].
void exact_grad_sums(const float* X, int64_t n, int d, const double* inv_ls_dev, double sf2, const double* alpha,
                     const double* Hinv, double* part, int parts, double* out, cudaStream_t st);
int exact_grad_parts();
// sum_i log(L_ii) of the Cholesky factor (lower, column-major) -> out (device)
void exact_logdiag(const double* L, int64_t n, double* out, cudaStream_t st);

}  // namespace wgp
