// hv_f64.cu — fused Matérn-3/2 H.V with fp64 right-hand sides and fp64
// accumulation: the operator of the fp64 CG path.
//
// Why a second H.V engine.  CG's short recurrences (proj/src/solvers.cpp:112-134)
// rely on the operator being one fixed symmetric linear map.  The fp32 tcgen05
// engine (hv_tc.cu) is accurate to ~1e-6 per product, but its error is not a
// fixed linear map: fp32 storage of the direction P, the fp32 tensor-core
// accumulation and the asymmetric rounding of the Gram entries each act as
// noise of order 1e-7 |H||P|, and measured (numpy emulation at config 0's late
// hyperparameters, kappa ~ 3e4) even 1e-9 |H||P| of such noise costs CG 10-15%
// more iterations than the fp64 reference at tol 0.01; fp32 vectors + the tc
// operator cost 25-38%.  A FIXED symmetric perturbation of the entries costs
// nothing (fp32-rounded entries: 94 vs 99 iterations).  So this engine
//   * evaluates each entry k_ij in fp32 from direct coordinate differences:
//     (x_ik - x_jk)^2 = (x_jk - x_ik)^2 exactly and the same instruction
//     sequence follows, so K is bitwise symmetric and identical on every call;
//   * multiplies by fp64 V and accumulates in fp64 (DFMA), so the product is
//     exact to ~1e-16 and linear in V.
// The diagonal (sf^2 + sigma^2) is applied in the split reduction; the
// streamed sum skips j == i.
//
// Decomposition: CTA = 64 output rows x one J range ("split") of 64-point
// tiles; the split count and ranges are keyed on the global n, so row shards
// reproduce the full operator's rows bitwise.  Per-split fp64 partials are
// summed in split order by hv64_reduce (deterministic, no atomics).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "hv_f64.cuh"

namespace wgp {
namespace {

#ifndef WGP_HV64_TM
#define WGP_HV64_TM 128
#endif
constexpr int TM = WGP_HV64_TM;  // output rows per CTA: one warp per 16 rows
constexpr int TJ = 32;           // contracted points per tile
constexpr int NT = 2 * TM;       // threads (TM / 16 warps)
constexpr int NW = NT / 32;
constexpr int KS = TM + 8;   // fp32 row stride of the K^T tile: conflict-free A fragments
constexpr int VJ = TJ + 4;   // fp64 column stride of the V tile: conflict-free B fragments
constexpr int kMaxNF = 10;   // <= 80 columns per launch (8 per DMMA fragment)
// residency: <= 128 registers per thread (2 x 256 or 4 x 128 threads)
constexpr int kCtasPerSm = TM == 128 ? 2 : 3;
constexpr int RA = TM / 32;        // K phase: rows lane + 32 a, a < RA
constexpr int PB = TJ / NW;        // K phase: points PB w + b, b < PB

__host__ __device__ inline int64_t jtiles(int64_t n) { return (n + TJ - 1) / TJ; }

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// D(8x8) += A(8x4, row) B(4x8, col), fp64 on the tensor core (DMMA).
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// D(16x8) += A(16x8, row) B(8x8, col): 4x the work of m8n8k4 per instruction.
__device__ __forceinline__ void dmma1688(double (&c)[4], const double (&a)[4], double b0, double b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0), "d"(b1));
}
#ifndef WGP_HV64_MMA
#define WGP_HV64_MMA 16
#endif

// One tile's V (TJ points x 8 NF columns, column-major with stride VJ, zero
// beyond n and s) and point coordinates (TJ x dp, row-major) -> shared memory
// with cp.async (16-byte pieces; V needs an even ldv and a 16-byte aligned base).
template <int NF>
__device__ __forceinline__ void load_tile(const Hv64Params& p, int64_t jt, double* vs, float* xj) {
  constexpr int PAIRS = TJ / 2;
  for (int e = threadIdx.x; e < 8 * NF * PAIRS; e += NT) {
    const int c = e / PAIRS, j = 2 * (e % PAIRS);
    const int64_t g = jt + j;
    double* dst = vs + c * VJ + j;
    if (c < p.s && g < p.n) {
      cp_async16(dst, p.V + g + static_cast<int64_t>(c) * p.ldv, g + 1 < p.n ? 16 : 8);
    } else {
      dst[0] = 0.0;
      dst[1] = 0.0;
    }
  }
  const int nq = TJ * p.dp / 4;  // xs rows are 16-byte aligned (dp % 4 == 0) and contiguous
  const float* src = p.xs + jt * p.dp;
  for (int e = threadIdx.x; e < nq; e += NT) cp_async16(xj + 4 * e, src + 4 * e, 16);
  cp_async_commit();
}

// Per tile: (1) the K tile, TM x 32 entries, 16 per thread, in fp32 from
// direct differences, stored as K^T (fp32; lane takes rows lane + 32 a, warp
// w points PB w + b: a warp's stores are 128-byte runs); (2) the product on
// the fp64 tensor core: warp w owns rows 16 w .. 16 w + 15 and every column,
// 2 x NF m8n8k4 DMMAs per 4 points, K widened to fp64 in the A fragment.
// The next tile's V and coordinates stream in with cp.async during the
// current tile (double buffered); two CTAs per SM overlap one CTA's K phase
// (FP32 / MUFU) with the other's DMMAs.
template <int NF>
__global__ void __launch_bounds__(NT, kCtasPerSm) hv64_kernel(Hv64Params p, int64_t m_pad, int splits) {
  if (p.done && *p.done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dps = p.dp + 1;  // odd stride: conflict-free row reads of xi
  double* vsb = reinterpret_cast<double*>(smem_raw);            // 2 x [8 NF][VJ]
  float* ks = reinterpret_cast<float*>(vsb + 2 * 8 * NF * VJ);  // [TJ][KS]
  float* xjb = ks + TJ * KS;                                     // 2 x [TJ][dp]
  float* xi = xjb + 2 * TJ * p.dp;                               // [TM][dps]
  __shared__ int64_t grow_s[TM];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float hsf2 = p.hyp[0], ha = p.hyp[1];
  const int64_t rbase = static_cast<int64_t>(blockIdx.x) * TM;
  // this CTA's J range: tiles [t0, t1) of the split, keyed on the global n
  const int64_t nt = jtiles(p.n);
  const int split = blockIdx.y;
  const int64_t t0 = nt * split / splits, t1 = nt * (split + 1) / splits;
  if (t0 < t1) load_tile<NF>(p, t0 * TJ, vsb, xjb);
  for (int r = tid; r < TM; r += NT) {
    const int64_t lr = rbase + r;
    grow_s[r] = lr < p.m ? p.r0 + lr : -1;
  }
  __syncthreads();
  for (int e = tid; e < TM * p.dp; e += NT) {
    const int r = e / p.dp, k = e % p.dp;
    const int64_t g = grow_s[r];
    xi[r * dps + k] = g >= 0 ? p.xs[g * p.dp + k] : 0.f;
  }

#if WGP_HV64_MMA == 16
  double acc[NF][4];  // C fragment f: rows g, g + 8 (c0 c1 | c2 c3), columns 8 f + 2 t + {0, 1}
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0.0;
#else
  double acc[2][NF][2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[r][f][0] = acc[r][f][1] = 0.0;
#endif

  int buf = 0;
  for (int64_t t = t0; t < t1; ++t, buf ^= 1) {
    const int64_t jt = t * TJ;
    const double* vs = vsb + buf * 8 * NF * VJ;
    const float* xj = xjb + buf * TJ * p.dp;
    cp_async_wait_all();
    __syncthreads();  // tile t landed; every warp is done with tile t - 1 (ks, other buffers)
    {  // K tile: rows lane + 32 a, points PB warp + b; bitwise symmetric in (i, j)
      float r2[RA][PB];
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < PB; ++b) r2[a][b] = 0.f;
      for (int k = 0; k < p.d; ++k) {  // the padded coordinates are zero: skip them
        float xa[RA], xb[PB];
#pragma unroll
        for (int a = 0; a < RA; ++a) xa[a] = xi[(lane + 32 * a) * dps + k];
#pragma unroll
        for (int b = 0; b < PB; ++b) xb[b] = xj[(PB * warp + b) * p.dp + k];
#pragma unroll
        for (int a = 0; a < RA; ++a)
#pragma unroll
          for (int b = 0; b < PB; ++b) {
            const float df = xa[a] - xb[b];
            r2[a][b] = fmaf(df, df, r2[a][b]);
          }
      }
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        const int64_t gj = jt + PB * warp + b;
        const bool valid = gj < p.n;
#pragma unroll
        for (int a = 0; a < RA; ++a) {
          const float kv = matern_from_u(sqrt_approx(r2[a][b]), hsf2, ha);
          ks[(PB * warp + b) * KS + lane + 32 * a] = (valid && gj != grow_s[lane + 32 * a]) ? kv : 0.f;
        }
      }
    }
    __syncthreads();  // K^T tile complete
    if (t + 1 < t1) load_tile<NF>(p, jt + TJ, vsb + (buf ^ 1) * 8 * NF * VJ, xjb + (buf ^ 1) * TJ * p.dp);
#if WGP_HV64_MMA == 16
    // product, m16n8k8 (g = lane / 4, t = lane % 4): A = K rows 16 w + g (+ 8),
    // points 8 kk + t (+ 4); B = V points 8 kk + t (+ 4), columns 8 f + g
    const float* ka = ks + (lane & 3) * KS + 16 * warp + (lane >> 2);
    const double* vb = vs + (lane >> 2) * VJ + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < TJ / 8; ++kk) {
      const double a[4] = {ka[8 * kk * KS], ka[8 * kk * KS + 8], ka[(8 * kk + 4) * KS], ka[(8 * kk + 4) * KS + 8]};
      double b0[NF], b1[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        b0[f] = vb[8 * f * VJ + 8 * kk];
        b1[f] = vb[8 * f * VJ + 8 * kk + 4];
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) dmma1688(acc[f], a, b0[f], b1[f]);
    }
#else
    // product: A = K rows (16 w + 8 r + lane / 4), points 4 kk + lane % 4;
    // B = V points 4 kk + lane % 4, columns 8 f + lane / 4
    const float* ka = ks + (lane & 3) * KS + 16 * warp + (lane >> 2);
    const double* vb = vs + (lane >> 2) * VJ + (lane & 3);
#pragma unroll 2
    for (int kk = 0; kk < TJ / 4; ++kk) {
      const double a0 = ka[4 * kk * KS], a1 = ka[4 * kk * KS + 8];
      double b[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) b[f] = vb[8 * f * VJ + 4 * kk];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        dmma884(acc[0][f], a0, b[f]);
        dmma884(acc[1][f], a1, b[f]);
      }
    }
#endif
  }
  // partials: part[(split s + c) m_pad + local row]; C fragment: row lane / 4,
  // columns 2 (lane % 4) + {0, 1}
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t lr = rbase + 16 * warp + 8 * r + (lane >> 2);
    if (lr >= p.m) continue;
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * f + 2 * (lane & 3) + e;
#if WGP_HV64_MMA == 16
        if (c < p.s) p.part[(static_cast<int64_t>(split) * p.s + c) * m_pad + lr] = acc[f][2 * r + e];
#else
        if (c < p.s) p.part[(static_cast<int64_t>(split) * p.s + c) * m_pad + lr] = acc[r][f][e];
#endif
      }
  }
}

// out = sum over splits (in split order) + diag V; store or residual.
__global__ void hv64_reduce_kernel(Hv64Params p, int64_t m_pad, int splits) {
  if (p.done && *p.done) return;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= p.m) return;
  const int64_t g = p.r0 + r;
  double v = 0.0;
  for (int k = 0; k < splits; ++k) v += p.part[(static_cast<int64_t>(k) * p.s + c) * m_pad + r];
  v = fma(static_cast<double>(p.hyp[2]), p.V[g + c * p.ldv], v);
  double* o = p.out + r + c * p.ldo;
  *o = p.mode == kHv64Residual ? p.B[g + c * p.ldb] - v : v;
}

template <int NF>
size_t smem_bytes(int dp) {
  return sizeof(double) * 2 * 8 * NF * VJ + sizeof(float) * (TJ * KS + 2 * TJ * dp + TM * (dp + 1));
}

template <int NF>
void launch(const Hv64Params& p, int64_t m_pad, int splits, cudaStream_t st) {
  const size_t smem = smem_bytes<NF>(p.dp);
  WGP_SMEM_ATTR(hv64_kernel<NF>, 200 * 1024);
  const dim3 grid(static_cast<unsigned>(ceil_div(p.m, TM)), static_cast<unsigned>(splits));
  hv64_kernel<NF><<<grid, NT, smem, st>>>(p, m_pad, splits);
  WGP_LAUNCH_CHECK();
}

}  // namespace

int hv64_splits(int64_t n) {
  // Whole waves for the full operator: the smallest split count giving at
  // least two waves of 148 x kCtasPerSm CTAs over ceil(n / 64) row tiles
  // with the last wave >= 90% full (at least 4 tiles per split).  A function
  // of n only, so row shards sum in the same order as the full launch.
  const int64_t rt = ceil_div(n, TM), nt = jtiles(n);
  const int64_t wave = 148 * kCtasPerSm;
  const int64_t smax = std::max<int64_t>(1, nt / 4);
  for (int64_t s = 1; s <= smax; ++s) {
    const int64_t ctas = rt * s;
    if (ctas < 2 * wave) continue;
    const double waves = static_cast<double>(ctas) / wave;
    if (waves / std::ceil(waves) >= 0.9) return static_cast<int>(s);
  }
  // small operators (fewer than two waves even at 4 tiles per split): one
  // wave, as many CTAs as fit (config 0: 32 row tiles x 13 splits = 416 of 444)
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(smax, wave / rt)));
}

// The operator engine: the exact integer-slice product on the int8 tensor
// core (hv_i8.cu) from n = 4096 points on (config-2-shaped data, s = 65, per
// CG iteration: 92 vs 128 us at n = 4096, 625 vs 1456 us at 16384,
// scripts/time_cg64_sizes.py), the DMMA kernel below for smaller n (its
// latency is lower: 39.5 vs 49.3 us at config 0, n = 2048) and d > 16.  Keyed on
// the global n, so every row shard uses the same engine.
// WGP_HV64_ENGINE=dmma | i8 forces one (A/B, tests).
static bool use_i8(int64_t n, int d, int s) {
  static const int force = [] {
    const char* e = getenv("WGP_HV64_ENGINE");
    if (!e) return 0;
    return std::string(e) == "dmma" ? -1 : std::string(e) == "i8" ? 1 : 0;
  }();
  if (!hv_i8_supported(d, s) || force < 0) return false;
  return force > 0 || n >= 4096;
}

size_t hv64_workspace_bytes(int64_t n, int64_t m, int s) {
  return std::max(sizeof(double) * static_cast<size_t>(hv64_splits(n)) * s * round_up(m, TM),
                  hv_i8_workspace_bytes(n, m, std::min(s, 8 * kMaxNF)));
}

static void hv64_launch(const Hv64Params& p, cudaStream_t st, bool reduce, int* splits_out, int64_t* m_pad_out) {
  if (p.s <= 0 || p.m <= 0) return;
  if (p.s > 8 * kMaxNF) {  // column chunks of <= 80 (accumulator registers)
    for (int c0 = 0; c0 < p.s; c0 += 8 * kMaxNF) {
      Hv64Params q = p;
      q.s = p.s - c0 < 8 * kMaxNF ? p.s - c0 : 8 * kMaxNF;
      q.V = p.V + c0 * p.ldv;
      q.out = p.out + c0 * p.ldo;
      if (p.B) q.B = p.B + c0 * p.ldb;
      hv64_launch(q, st, true, nullptr, nullptr);
    }
    return;
  }
  int splits = 0;
  int64_t m_pad = 0;
  if (use_i8(p.n, p.d, p.s) && hv_i8_partials(p, st, &splits, &m_pad)) {
    if (splits_out) *splits_out = splits;
    if (m_pad_out) *m_pad_out = m_pad;
    if (!reduce) return;
    hv64_reduce_kernel<<<dim3(static_cast<unsigned>(ceil_div(p.m, 256)), p.s), 256, 0, st>>>(p, m_pad, splits);
    WGP_LAUNCH_CHECK();
    return;
  }
  if ((p.ldv & 1) || (reinterpret_cast<uintptr_t>(p.V) & 15) || (p.dp & 3))
    throw std::invalid_argument("hv64: V needs an even leading dimension and 16-byte alignment");
  splits = hv64_splits(p.n);
  m_pad = round_up(p.m, TM);
  switch ((p.s + 7) / 8) {
    case 1: launch<1>(p, m_pad, splits, st); break;
    case 2: launch<2>(p, m_pad, splits, st); break;
    case 3: launch<3>(p, m_pad, splits, st); break;
    case 4: launch<4>(p, m_pad, splits, st); break;
    case 5: launch<5>(p, m_pad, splits, st); break;
    case 6: launch<6>(p, m_pad, splits, st); break;
    case 7: launch<7>(p, m_pad, splits, st); break;
    case 8: launch<8>(p, m_pad, splits, st); break;
    case 9: launch<9>(p, m_pad, splits, st); break;
    default: launch<10>(p, m_pad, splits, st); break;
  }
  if (splits_out) *splits_out = splits;
  if (m_pad_out) *m_pad_out = m_pad;
  if (!reduce) return;
  hv64_reduce_kernel<<<dim3(static_cast<unsigned>(ceil_div(p.m, 256)), p.s), 256, 0, st>>>(p, m_pad, splits);
  WGP_LAUNCH_CHECK();
}

void hv64(const Hv64Params& p, cudaStream_t st) { hv64_launch(p, st, true, nullptr, nullptr); }

bool hv64_partials(const Hv64Params& p, cudaStream_t st, int* splits, int64_t* m_pad) {
  if (p.s <= 0 || p.m <= 0 || p.s > 8 * kMaxNF) return false;
  hv64_launch(p, st, false, splits, m_pad);
  return true;
}

}  // namespace wgp
