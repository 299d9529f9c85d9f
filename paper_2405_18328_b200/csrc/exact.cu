// exact.cu — the reference's exact (dense Cholesky) path on the GPU in fp64:
// exact_mll / exact_gradient (proj/src/exact.cpp:25-50), the trajectory oracle
// of train_exact (proj/src/optimizer.cpp:117-118, 179-181).  H is built once
// per call (lower triangle), factored with cuSOLVER potrf, alpha = H^-1 y by
// potrs, H^-1 by potri; the gradient contractions
//   g_k = <dH_k, 1/2 alpha alpha^T> - <dH_k, 1/2 H^-1>   (exact.cpp:45-48)
// are one pass over the lower triangle evaluating the derivative entries on
// the fly (kernel.cpp:216-252) with fixed-order fp64 reductions.
#include "common.cuh"
#include "exact.cuh"

namespace wgp {
namespace {

constexpr int kTile = 32;
constexpr int kBuildThreads = 256;  // 32 x 8, 4 entries per thread
constexpr int kGradThreads = 256;
constexpr int kGradBlocks = 148 * 4;
constexpr double kSqrt3d = 1.7320508075688772;

// Reference distance: D = (sq_i + sq_j) - 2 G_ij clamped at 0 (kernel.cpp:101-116).
__device__ __forceinline__ double scaled_sqdist(const float* X, int64_t n, int d, const double* inv_ls, int64_t i,
                                                int64_t j) {
  double sqi = 0.0, sqj = 0.0, g = 0.0;
  for (int k = 0; k < d; ++k) {
    const double a = static_cast<double>(X[i + k * n]) * inv_ls[k];
    const double b = static_cast<double>(X[j + k * n]) * inv_ls[k];
    sqi += a * a;
    sqj += b * b;
    g += a * b;
  }
  const double D = (sqi + sqj) - 2.0 * g;
  return D > 0.0 ? D : 0.0;
}

__global__ void build_kernel(const float* __restrict__ X, int64_t n, int d, const double* __restrict__ inv_ls,
                             double sf2, double noise2, double* __restrict__ H) {
  __shared__ double ls_s[kExactMaxD];
  if (threadIdx.x < d) ls_s[threadIdx.x] = inv_ls[threadIdx.x];
  __syncthreads();
  const int64_t bi = blockIdx.x, bj = blockIdx.y;
  if (bi < bj) return;  // lower triangle of tiles
  const int tx = threadIdx.x % kTile, ty = threadIdx.x / kTile;
  const int64_t i = bi * kTile + tx;
  if (i >= n) return;
  for (int r = ty; r < kTile; r += kBuildThreads / kTile) {
    const int64_t j = bj * kTile + r;
    if (j >= n || j > i) continue;
    const double u = kSqrt3d * sqrt(scaled_sqdist(X, n, d, ls_s, i, j));
    double h = sf2 * (1.0 + u) * exp(-u);
    if (i == j) h += noise2;
    H[i + j * n] = h;
  }
}

// One block per strided set of lower-triangle tiles (fixed assignment), one
// fp64 partial per block and quantity.
__global__ void __launch_bounds__(kGradThreads) grad_kernel(const float* __restrict__ X, int64_t n, int d,
                                                            const double* __restrict__ inv_ls, double sf2,
                                                            const double* __restrict__ alpha,
                                                            const double* __restrict__ Hinv, double* __restrict__ part) {
  __shared__ double ls_s[kExactMaxD];
  __shared__ double red[kGradThreads / 32][kExactMaxD + 2];
  if (threadIdx.x < d) ls_s[threadIdx.x] = inv_ls[threadIdx.x];
  __syncthreads();
  const int64_t nt = (n + kTile - 1) / kTile;
  const int64_t ntri = nt * (nt + 1) / 2;
  double acc[kExactMaxD + 2];
  for (int k = 0; k < d + 2; ++k) acc[k] = 0.0;
  const int tx = threadIdx.x % kTile, ty = threadIdx.x / kTile;
  for (int64_t tile = blockIdx.x; tile < ntri; tile += gridDim.x) {
    // tile -> (bi >= bj): bi = floor((sqrt(8 tile + 1) - 1) / 2)
    int64_t bi = static_cast<int64_t>((sqrt(8.0 * static_cast<double>(tile) + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > tile) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= tile) ++bi;
    const int64_t bj = tile - bi * (bi + 1) / 2;
    const int64_t i = bi * kTile + tx;
    if (i >= n) continue;
    for (int r = ty; r < kTile; r += kGradThreads / kTile) {
      const int64_t j = bj * kTile + r;
      if (j >= n || j > i) continue;
      // W_ij counts twice off the diagonal (symmetry)
      const double w = (0.5 * alpha[i] * alpha[j] - 0.5 * Hinv[i + j * n]) * (i == j ? 1.0 : 2.0);
      const double D = scaled_sqdist(X, n, d, ls_s, i, j);
      const double u = kSqrt3d * sqrt(D);
      const double decay = exp(-u);
      acc[d] += w * sf2 * (1.0 + u) * decay;  // kernel value (signal term)
      if (i == j) {
        acc[d + 1] += w;  // noise term: tr(W)
        continue;
      }
      const double wd = w * decay;
      for (int k = 0; k < d; ++k) {  // direct differences
        const double dx = (static_cast<double>(X[i + k * n]) - static_cast<double>(X[j + k * n])) * ls_s[k];
        acc[k] += wd * dx * dx;
      }
    }
  }
  // block reduction: warp shuffles, then the warps in order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < d + 2; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < d + 2) {
    double v = 0.0;
    for (int w = 0; w < kGradThreads / 32; ++w) v += red[w][threadIdx.x];
    part[static_cast<int64_t>(blockIdx.x) * (d + 2) + threadIdx.x] = v;
  }
}

__global__ void sum_parts_kernel(const double* part, int parts, int w, double* out) {
  const int k = threadIdx.x;
  if (k >= w) return;
  double v = 0.0;
  for (int b = 0; b < parts; ++b) v += part[static_cast<int64_t>(b) * w + k];
  out[k] = v;
}

__global__ void logdiag_kernel(const double* L, int64_t n, double* out) {
  __shared__ double red[32];
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v += log(L[i + i * n]);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
    *out = t;
  }
}

}  // namespace

int exact_grad_parts() { return kGradBlocks; }

void exact_build(const float* X, int64_t n, int d, const double* inv_ls, double sf2, double noise2, double* H,
                 cudaStream_t st) {
  if (d > kExactMaxD) throw std::invalid_argument("exact path: input dimension above 30");
  const unsigned nt = static_cast<unsigned>(ceil_div(n, kTile));
  build_kernel<<<dim3(nt, nt), kBuildThreads, 0, st>>>(X, n, d, inv_ls, sf2, noise2, H);
  WGP_LAUNCH_CHECK();
}

void exact_grad_sums(const float* X, int64_t n, int d, const double* inv_ls, double sf2, const double* alpha,
                     const double* Hinv, double* part, int parts, double* out, cudaStream_t st) {
  grad_kernel<<<parts, kGradThreads, 0, st>>>(X, n, d, inv_ls, sf2, alpha, Hinv, part);
  WGP_LAUNCH_CHECK();
  sum_parts_kernel<<<1, 32, 0, st>>>(part, parts, d + 2, out);
  WGP_LAUNCH_CHECK();
}

void exact_logdiag(const double* L, int64_t n, double* out, cudaStream_t st) {
  logdiag_kernel<<<1, 1024, 0, st>>>(L, n, out);
  WGP_LAUNCH_CHECK();
}

}  // namespace wgp
