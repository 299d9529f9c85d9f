// grad_rff.cu — fused gradient-contraction kernel and the pathwise
// random-Fourier-feature probe kernel.
//
// Gradient: one pass over all (i, j) entries computes, per entry,
//   u_ij (scaled distance), decay = 2^-u, k_ij, W^A_ij = vy_i vy_j / 2,
//   W^B_ij = coef_b sum_c L_ic R_jc,
// and accumulates sum decay W (x_ik - x_jk)^2 per lengthscale (direct
// differences -- the fp32-safe form of the reference's expansion trick,
// proj/src/kernel.cpp:227-243) and sum k W for the signal.
// The noise contraction (the trace of W) is an O(n s) diagonal sum done by
// the host-side driver.  Reductions: fp32 within a 4x4 register tile, fp64
// per warp in shared memory, one fp64 partial per CTA, then a fixed-order
// sum over CTAs (bitwise deterministic).
#include "common.cuh"
#include "kernels.cuh"

namespace wgp {
namespace {

constexpr int TM = 64, TJ = 64, NT = 256;

template <int DMAX>
__global__ void __launch_bounds__(NT) grad_kernel(GradParams p) {
  extern __shared__ float smem[];
  const int dps = p.dp + 1;
  const int sp = p.s + 1;
  float* xi = smem;                 // [TM][dps]
  float* xj = xi + TM * dps;        // [TJ][dps]
  float* li = xj + TJ * dps;        // [TM][sp]
  float* rj = li + TM * sp;         // [TJ][sp]
  float* vyi = rj + TJ * sp;        // [TM]
  float* vyj = vyi + TM;            // [TJ]
  __shared__ double wacc[NT / 32][2 * (DMAX + 1)];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = 2 * (p.d + 1);
  for (int e = tid; e < (NT / 32) * 2 * (DMAX + 1); e += NT) (&wacc[0][0])[e] = 0.0;
  const int64_t ib = p.r0 + static_cast<int64_t>(blockIdx.x) * TM;
  const int64_t iend = p.r0 + (p.m < 0 ? p.n : p.m);  // rows [r0, iend)
  for (int e = tid; e < TM * p.dp; e += NT) {
    const int r = e / p.dp, k = e % p.dp;
    xi[r * dps + k] = ib + r < iend ? p.xs[(ib + r) * p.dp + k] : 0.f;
  }
  for (int e = tid; e < TM * p.s; e += NT) {
    const int c = e / TM, r = e % TM;
    li[r * sp + c] = ib + r < iend ? p.L[ib + r + c * p.ld] : 0.f;
  }
  for (int r = tid; r < TM; r += NT) vyi[r] = ib + r < iend ? p.vy[ib + r] : 0.f;

  const int ii = (tid / 16) * 4, jj = (tid % 16) * 4;
  float accA[DMAX + 1], accB[DMAX + 1];
#pragma unroll
  for (int k = 0; k <= DMAX; ++k) accA[k] = accB[k] = 0.f;
  int tiles_since_flush = 0;

  for (int64_t jt = 0; jt < p.n; jt += TJ) {
    __syncthreads();
    for (int e = tid; e < TJ * p.dp; e += NT) {
      const int r = e / p.dp, k = e % p.dp;
      xj[r * dps + k] = jt + r < p.n ? p.xs[(jt + r) * p.dp + k] : 0.f;
    }
    for (int e = tid; e < TJ * p.s; e += NT) {
      const int c = e / TJ, r = e % TJ;
      rj[r * sp + c] = jt + r < p.n ? p.R[jt + r + c * p.ld] : 0.f;
    }
    for (int r = tid; r < TJ; r += NT) vyj[r] = jt + r < p.n ? p.vy[jt + r] : 0.f;
    __syncthreads();

    float wb[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) wb[a][b] = 0.f;
    for (int c = 0; c < p.s; ++c) {
      float la[4], rb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) la[a] = li[(ii + a) * sp + c];
#pragma unroll
      for (int b = 0; b < 4; ++b) rb[b] = rj[(jj + b) * sp + c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) wb[a][b] = fmaf(la[a], rb[b], wb[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        // entries outside [0, n) have zero L/R/vy and contribute nothing
        float r2 = 0.f;
#pragma unroll
        for (int k = 0; k < DMAX; ++k) {
          if (k < p.d) {
            const float df = xi[(ii + a) * dps + k] - xj[(jj + b) * dps + k];
            r2 = fmaf(df, df, r2);
          }
        }
        const float u = sqrt_approx(r2);
        const float dec = ex2_approx(-u);
        const float kv = fmaf(p.a, u, p.sf2) * dec;
        const float wA = 0.5f * vyi[ii + a] * vyj[jj + b];
        const float wB = p.coef_b * wb[a][b];
        const float dA = dec * wA, dB = dec * wB;
#pragma unroll
        for (int k = 0; k < DMAX; ++k) {
          if (k < p.d) {
            const float df = xi[(ii + a) * dps + k] - xj[(jj + b) * dps + k];
            const float q = df * df;
            accA[k] = fmaf(q, dA, accA[k]);
            accB[k] = fmaf(q, dB, accB[k]);
          }
        }
        accA[DMAX] = fmaf(kv, wA, accA[DMAX]);
        accB[DMAX] = fmaf(kv, wB, accB[DMAX]);
      }
    }
    // flush fp32 register sums into fp64 per-warp slots every 8 tiles
    if (++tiles_since_flush == 8 || jt + TJ >= p.n) {
      tiles_since_flush = 0;
#pragma unroll
      for (int k = 0; k <= DMAX; ++k) {
        if (k < p.d || k == DMAX) {
          const int slot = k == DMAX ? p.d : k;
          const float sa = warp_sum(accA[k]);
          const float sb = warp_sum(accB[k]);
          if (lane == 0) {
            wacc[warp][slot] += static_cast<double>(sa);
            wacc[warp][p.d + 1 + slot] += static_cast<double>(sb);
          }
          accA[k] = accB[k] = 0.f;
        }
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < W; q += NT) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += wacc[w][q];
    p.part[static_cast<int64_t>(blockIdx.x) * W + q] = t;
  }
}

__global__ void grad_finalize_kernel(const double* part, int nblk, int width, double* out) {
  for (int q = threadIdx.x; q < width; q += blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < nblk; ++b) t += part[static_cast<int64_t>(b) * width + q];
    out[q] = t;
  }
}

template <int DMAX>
void launch_grad(const GradParams& p, cudaStream_t st) {
  const int dps = p.dp + 1, sp = p.s + 1;
  const size_t smem = sizeof(float) * (2 * 64 * dps + 2 * 64 * sp + 2 * 64);
  WGP_SMEM_ATTR(grad_kernel<DMAX>, 200 * 1024);
  grad_kernel<DMAX><<<grad_blocks(p.m < 0 ? p.n : p.m), NT, smem, st>>>(p);
  WGP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// RFF probes.  CTA = 64 rows; loop over features in chunks of 64: the phase
// b_f + om_f . x_i is formed in fp64 and range-reduced before the fp32
// cosine, the 64 x 64 feature tile goes through shared memory and is
// contracted with w on the CUDA cores.
constexpr int RT = 64, RF = 64;

__global__ void __launch_bounds__(NT) rff_kernel(RffParams p) {
  extern __shared__ float smem[];
  const int SP = ((p.s + 15) / 16) * 16;
  float* ph = smem;              // [RF][RT + 4]
  float* ws = ph + RF * (RT + 4);  // [RF][SP]
  const int tid = threadIdx.x;
  const int64_t ib = static_cast<int64_t>(blockIdx.x) * RT;
  const int ty = tid / 16, tx = tid % 16;
  const int CPT = SP / 16;
  float acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[a][q] = 0.f;
  for (int f0 = 0; f0 < p.F; f0 += RF) {
    __syncthreads();
    for (int e = tid; e < RF * RT; e += NT) {
      const int f = e / RT, r = e % RT;
      float v = 0.f;
      if (f0 + f < p.F && ib + r < p.n) {
        double phase = p.b[f0 + f];
        for (int k = 0; k < p.d; ++k)
          phase = fma(p.om[(f0 + f) * static_cast<int64_t>(p.d) + k],
                      static_cast<double>(p.x[ib + r + k * p.n]), phase);
        const double twopi = 6.283185307179586;
        phase -= twopi * rint(phase / twopi);
        v = cosf(static_cast<float>(phase));
      }
      ph[f * (RT + 4) + r] = v;
    }
    for (int e = tid; e < RF * SP; e += NT) {
      const int c = e / RF, f = e % RF;
      ws[f * SP + c] = (f0 + f < p.F && c < p.s) ? p.w[(f0 + f) + static_cast<int64_t>(c) * p.F] : 0.f;
    }
    __syncthreads();
    for (int f = 0; f < RF; ++f) {
      const float4 pv = *reinterpret_cast<const float4*>(&ph[f * (RT + 4) + ty * 4]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < CPT) {
          const float wv = ws[f * SP + tx + 16 * q];
          acc[0][q] = fmaf(pv.x, wv, acc[0][q]);
          acc[1][q] = fmaf(pv.y, wv, acc[1][q]);
          acc[2][q] = fmaf(pv.z, wv, acc[2][q]);
          acc[3][q] = fmaf(pv.w, wv, acc[3][q]);
        }
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t i = ib + ty * 4 + a;
    if (i >= p.n) continue;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = tx + 16 * q;
      if (q < CPT && c < p.s)
        p.out[i + c * p.ld] = fmaf(p.amp, acc[a][q], p.sigma * p.eps[i + c * p.ld]);
    }
  }
}

}  // namespace

int grad_blocks(int64_t m) { return static_cast<int>(ceil_div(m, TM)); }

void grad_simt(const GradParams& p, cudaStream_t st) {
  if (p.d <= 4) return launch_grad<4>(p, st);
  if (p.d <= 8) return launch_grad<8>(p, st);
  if (p.d <= 12) return launch_grad<12>(p, st);
  if (p.d <= 16) return launch_grad<16>(p, st);
  if (p.d <= 32) return launch_grad<32>(p, st);
  throw std::invalid_argument("gradient kernel supports d <= 32");
}

void grad_finalize(const double* part, int nblk, int width, double* out, cudaStream_t st) {
  grad_finalize_kernel<<<1, 128, 0, st>>>(part, nblk, width, out);
  WGP_LAUNCH_CHECK();
}

void rff_probes(const RffParams& p, cudaStream_t st) {
  if (p.s > 128) throw std::invalid_argument("rff_probes: at most 128 probes per launch");
  const int SP = ((p.s + 15) / 16) * 16;
  const size_t smem = sizeof(float) * (RF * (RT + 4) + RF * SP);
  WGP_SMEM_ATTR(rff_kernel, 64 * 1024);
  rff_kernel<<<static_cast<unsigned>(ceil_div(p.n, RT)), NT, smem, st>>>(p);
  WGP_LAUNCH_CHECK();
}

}  // namespace wgp
