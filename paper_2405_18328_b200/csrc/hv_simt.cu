// hv_simt.cu — SIMT fp32 fused H.V (v0) and point preparation.
//
// Replaces the dense products H * V of the reference solvers
// (proj/src/solvers.cpp:71,92,110,120,169,186,188,211,242) without ever
// forming H: each 64 x 64 tile of K is evaluated in registers from the
// prepared points (direct per-dimension differences, exact zero on the
// diagonal), staged through shared memory and contracted with the 64 x s
// tile of V.  It handles every variant the solvers need: all rows, a row
// range (sharding), gathered rows (SGD minibatch), a contracted column range
// (AP block update), and store / residual / subtract epilogues.  It is the
// general-shape path and the accuracy baseline for the tcgen05 kernel.
#include "common.cuh"
#include "kernels.cuh"

namespace wgp {
namespace {

constexpr int TM = 64;   // output rows per CTA
constexpr int TJ = 64;   // contracted points per tile
constexpr int NT = 256;  // threads

template <int CPT>  // columns per thread; the CTA covers 16 * CPT columns
__global__ void __launch_bounds__(NT) hv_simt_kernel(HvParams p) {
  if (p.done && *p.done) return;
  extern __shared__ float smem[];
  const int dps = p.dp + 1;  // odd stride against bank conflicts
  constexpr int SP = 16 * CPT;
  float* xi = smem;                    // [TM][dps]
  float* xj = xi + TM * dps;           // [TJ][dps]
  float* ks = xj + TJ * dps;           // [TJ][TM + 4]
  float* vs = ks + TJ * (TM + 4);      // [TJ][SP]
  __shared__ int64_t grow_s[TM];

  const int tid = threadIdx.x;
  const float hsf2 = p.hyp ? p.hyp[0] : p.sf2, ha = p.hyp ? p.hyp[1] : p.a, hdiag = p.hyp ? p.hyp[2] : p.diag;
  const int64_t rbase = static_cast<int64_t>(blockIdx.x) * TM;
  for (int r = tid; r < TM; r += NT) {
    const int64_t lr = rbase + r;
    int64_t g = -1;
    if (lr < p.m) g = p.row_idx ? static_cast<int64_t>(p.row_idx[lr]) : p.r0 + lr;
    grow_s[r] = g;
  }
  __syncthreads();
  for (int e = tid; e < TM * p.dp; e += NT) {
    const int r = e / p.dp, k = e % p.dp;
    const int64_t g = grow_s[r];
    xi[r * dps + k] = g >= 0 ? p.xs[g * p.dp + k] : 0.f;
  }

  const int ty = tid / 16, tx = tid % 16;
  const int ii = ty * 4;   // rows of this thread (K phase and GEMM phase)
  const int jj = tx * 4;   // points of this thread (K phase)
  // Each 64-point tile is accumulated in fp32 (tacc) and added to an fp64
  // running sum, so the rounding error does not grow with n (one fp32 sum
  // over all n points drifts like sqrt(n) 2^-24 |out|: 2.7e-6 relative at
  // n = 20000 on dense data, measured).
  double acc[4][CPT];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < CPT; ++q) acc[r][q] = 0.0;

  for (int64_t jt = p.j0; jt < p.j1; jt += TJ) {
    __syncthreads();
    for (int e = tid; e < TJ * p.dp; e += NT) {
      const int j = e / p.dp, k = e % p.dp;
      const int64_t g = jt + j;
      xj[j * dps + k] = g < p.j1 ? p.xs[g * p.dp + k] : 0.f;
    }
    for (int e = tid; e < TJ * SP; e += NT) {
      const int c = e / TJ, j = e % TJ;
      const int64_t g = jt + j;
      vs[j * SP + c] = (g < p.j1 && c < p.s) ? p.V[g + c * p.ldv] : 0.f;
    }
    __syncthreads();
    // K tile: 4 x 4 entries per thread.
    float r2[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) r2[a][b] = 0.f;
    for (int k = 0; k < p.dp; ++k) {
      float xa[4], xb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xa[a] = xi[(ii + a) * dps + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) xb[b] = xj[(jj + b) * dps + k];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const float df = xa[a] - xb[b];
          r2[a][b] = fmaf(df, df, r2[a][b]);
        }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t gj = jt + jj + b;
      const bool valid = gj < p.j1;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float kv = matern_from_u(sqrt_approx(r2[a][b]), hsf2, ha);
        ks[(jj + b) * (TM + 4) + ii + a] = (valid && gj != grow_s[ii + a]) ? kv : 0.f;
      }
    }
    __syncthreads();
    // acc[4 rows][CPT cols] += K[rows, j] * V[j, cols]
    float tacc[4][CPT];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < CPT; ++q) tacc[r][q] = 0.f;
#pragma unroll 4
    for (int j = 0; j < TJ; ++j) {
      const float4 kk = *reinterpret_cast<const float4*>(&ks[j * (TM + 4) + ii]);
      float vb[CPT];
#pragma unroll
      for (int q = 0; q < CPT; ++q) vb[q] = vs[j * SP + tx + 16 * q];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        tacc[0][q] = fmaf(kk.x, vb[q], tacc[0][q]);
        tacc[1][q] = fmaf(kk.y, vb[q], tacc[1][q]);
        tacc[2][q] = fmaf(kk.z, vb[q], tacc[2][q]);
        tacc[3][q] = fmaf(kk.w, vb[q], tacc[3][q]);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < CPT; ++q) acc[r][q] += static_cast<double>(tacc[r][q]);
  }
  // Epilogue: + sigma^2 V on the diagonal, then store / residual / subtract.
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t lr = rbase + ii + a;
    if (lr >= p.m) continue;
    const int64_t g = grow_s[ii + a];
    const bool diag = g >= p.j0 && g < p.j1;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tx + 16 * q;
      if (c >= p.s) continue;
      float v = static_cast<float>(acc[a][q]);
      if (diag) v = fmaf(hdiag, p.V[g + c * p.ldv], v);
      float* o = p.out + lr + c * p.ldo;
      if (p.mode == kHvStore)
        *o = v;
      else if (p.mode == kHvResidual)
        *o = p.B[g + c * p.ldb] - v;
      else
        *o -= v;
    }
  }
}

template <int CPT>
void launch(const HvParams& p, cudaStream_t st) {
  const int dps = p.dp + 1;
  const size_t smem = sizeof(float) * (TM * dps + TJ * dps + TJ * (TM + 4) + TJ * 16 * CPT);
  WGP_SMEM_ATTR(hv_simt_kernel<CPT>, 96 * 1024);
  const unsigned grid = static_cast<unsigned>(ceil_div(p.m, TM));
  if (grid == 0) return;
  hv_simt_kernel<CPT><<<grid, NT, smem, st>>>(p);
  WGP_LAUNCH_CHECK();
}

__global__ void prepare_kernel(const float* X, int64_t n, int d, const double* mu,
                               const double* scale, float* xs, int64_t n_pad, int dp) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n_pad * dp) return;
  const int64_t i = e / dp;
  const int k = static_cast<int>(e % dp);
  float v = 0.f;
  if (i < n && k < d) v = static_cast<float>((static_cast<double>(X[i + k * n]) - mu[k]) * scale[k]);
  xs[e] = v;
}

}  // namespace

void hv_simt(const HvParams& p, cudaStream_t st) {
  if (p.s <= 0 || p.m <= 0) return;
  if (p.s <= 16) return launch<1>(p, st);
  if (p.s <= 32) return launch<2>(p, st);
  if (p.s <= 48) return launch<3>(p, st);
  if (p.s <= 64) return launch<4>(p, st);
  if (p.s <= 80) return launch<5>(p, st);
  if (p.s <= 96) return launch<6>(p, st);
  if (p.s <= 128) return launch<8>(p, st);
  // wider right-hand sides: process in column chunks of 128
  for (int c0 = 0; c0 < p.s; c0 += 128) {
    HvParams q = p;
    q.s = p.s - c0 < 128 ? p.s - c0 : 128;
    q.V = p.V + c0 * p.ldv;
    q.out = p.out + c0 * p.ldo;
    if (p.B) q.B = p.B + c0 * p.ldb;
    hv_simt(q, st);
  }
}

void prepare_points(const float* X, int64_t n, int d, const double* mu, const double* scale,
                    float* xs, int64_t n_pad, int dp, cudaStream_t st) {
  const int64_t total = n_pad * dp;
  const unsigned grid = static_cast<unsigned>(ceil_div(total, 256));
  prepare_kernel<<<grid, 256, 0, st>>>(X, n, d, mu, scale, xs, n_pad, dp);
  WGP_LAUNCH_CHECK();
}

}  // namespace wgp
