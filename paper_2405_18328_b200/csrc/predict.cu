// predict.cu — kernels of the iterative predictive path (proj/src/exact.cpp:52-92
// restated over iterative solves): the train x test cross
// kernel matrix K* and the column dots K*^T alpha.
#include "common.cuh"
#include "kernels.cuh"

namespace wgp {
namespace {

// K*[j + i * ld] = k(x_train_j, x_test_i) from prepared points (u^2 = |xs_j - xt_i|^2),
// k = (a u + sf^2) 2^-u (kernel.cpp:79-93 in the kernels' scaled form).
__global__ void cross_kernel(const float* __restrict__ xs, int64_t n, const float* __restrict__ xt, int64_t m,
                             int dp, float sf2, float a, float* __restrict__ out, int64_t ld) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (i >= m) return;
  float* col = out + i * ld;
  if (j >= ld) return;
  if (j >= n) {
    col[j] = 0.f;
    return;
  }
  double u2 = 0.0;
  for (int k = 0; k < dp; ++k) {
    const double df = static_cast<double>(xs[j * dp + k]) - static_cast<double>(xt[i * dp + k]);
    u2 += df * df;
  }
  const double u = sqrt(u2);
  col[j] = static_cast<float>((static_cast<double>(a) * u + sf2) * exp2(-u));
}

// out[i] = sum_j K*[j, i] alpha[j] in fp64 (one block per test point, fixed order)
__global__ void colvec_dots_kernel(const float* __restrict__ K, int64_t ld, int64_t n,
                                   const float* __restrict__ alpha, double* __restrict__ out) {
  __shared__ double red[32];
  const float* col = K + static_cast<int64_t>(blockIdx.x) * ld;
  double v = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) v += static_cast<double>(col[j]) * alpha[j];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned w = 0; w < blockDim.x / 32; ++w) t += red[w];
    out[blockIdx.x] = t;
  }
}

}  // namespace

void cross_matrix(const float* xs, int64_t n, const float* xt, int64_t m, int dp, float sf2, float a, float* out,
                  int64_t ld, cudaStream_t st) {
  if (m <= 0) return;
  cross_kernel<<<dim3(static_cast<unsigned>(ceil_div(ld, 256)), static_cast<unsigned>(m)), 256, 0, st>>>(
      xs, n, xt, m, dp, sf2, a, out, ld);
  WGP_LAUNCH_CHECK();
}

void colvec_dots(const float* K, int64_t ld, int64_t n, int64_t m, const float* alpha, double* out,
                 cudaStream_t st) {
  if (m <= 0) return;
  colvec_dots_kernel<<<static_cast<unsigned>(m), 256, 0, st>>>(K, ld, n, alpha, out);
  WGP_LAUNCH_CHECK();
}

}  // namespace wgp
