// grad_tc.cu — gradient contraction on the tensor core (the
// derivative_contractions of proj/src/kernel.cpp:199-262).
//
// Per entry (i, j) the gradient needs
//   W^B_ij = sum_c L_ic R_jc            (an s-long dot product: GEMM-shaped)
//   u_ij, decay 2^-u, k_ij, (x_ik - x_jk)^2 per lengthscale   (O(d) CUDA-core work)
// and accumulates, per lengthscale k and for the signal,
//   A_k = sum W^A decay dx_k^2,  B_k = sum W^B decay dx_k^2,
//   A_s = sum W^A k,             B_s = sum W^B k,   W^A = vy_i vy_j / 2.
// The SIMT kernel (grad_rff.cu) spends ~64 of its ~100 FP ops per entry on
// W^B.  Here the tensor core forms W^B (3xTF32, ~2^-21 per product: L_I from
// TMEM, R_J from shared memory, fp32 accumulation over s <= 64 terms) and the
// epilogue warps do only the O(d) part: ~5d + 6 FP ops and 2 MUFU per entry.
// The distances are formed from direct coordinate differences (not a Gram),
// exactly as the SIMT kernel does: they are needed for the per-lengthscale
// terms anyway and keep r^2 >= 0 and bit-identical to grad_simt.
//
// CTA = 128 rows (TMEM lanes) x a J range in 64-point tiles.  Warps 0..11:
// three epilogue groups (group w takes tiles t = w mod 3; warp w % 4 owns
// TMEM lanes 32 (w % 4) .. +31 = its 32 rows); warp 12 TMA / bulk producer;
// warp 13 MMA issuer; warp 14 TMEM allocator.  TMEM: six W buffers of 64
// fp32 columns [0, 384), L_I hi [384, 448), L_I lo [448, 512).  Rings:
// R_J planes (consumed by the MMA, freed by its commit) and the epilogue's
// per-point data x_j | vy_j (freed by the epilogue).  Reductions: fp32 per
// row over 4 tiles (256 entries), then a per-row fp64 sum in shared memory,
// fp64 warp / CTA sums in fixed order, one fp64 partial per CTA -- the
// [2 (d + 1)] partial format grad_finalize sums (bitwise deterministic).
#include "common.cuh"
#include "hv_tc.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace wgp {
namespace {

constexpr int gTI = 128;             // rows per CTA (MMA M, TMEM lanes)
constexpr int gTJ = 64;              // points per J tile (MMA N)
constexpr int gThreads = 512;
constexpr int gEpiGroups = 3, gEpiWarps = 12, gEpiThreads = 384;
constexpr int gWarpProd = 12, gWarpMma = 13, gWarpAlloc = 14;
constexpr int gBufs = 6;                    // W buffers (64 TMEM columns each)
constexpr uint32_t gLhi = 384, gLlo = 448;  // L_I planes, <= 64 columns each
constexpr int gRing = 8;                    // MMA-done barrier ring (> gBufs)
constexpr int gNE = 8;                      // epilogue-data ring (>= gBufs + 2)
constexpr int gMaxNM = 6;
constexpr int gFlushTiles = 4;              // fp32 row sums span 4 tiles (256 entries)
constexpr int gSmemLimit = 232448 - 4096;   // 227 KB opt-in minus static smem
constexpr uint32_t gTfMask = 0xFFFFE000u;

__host__ __device__ constexpr int ep_of(int d) { return ((d + 1 + 3) / 4) * 4; }  // x_j[0..d) | vy_j | 0..

struct GradTcArgs {
  int64_t n;
  int d, dp, s, spk;  // spk: K extent of W^B (32 or 64: multiples of one 128-byte swizzle row)
  int num_jt, splits, nm;
  uint32_t mstage, estage, acc_off;
  const float* xs;   // prepared points [n][dp]
  const float* vy;   // [n]
  const float* xv;   // [n_pad][ep]: x_j | vy_j, zero rows past n
  const float* L;
  int64_t ld;
  float sf2, a, coef_b;
  double* part;      // [gridDim.x][2 (d + 1)]
};

template <int D>
__global__ void __launch_bounds__(gThreads, 1)
    grad_tc_kernel(const __grid_constant__ CUtensorMap mRhi, const __grid_constant__ CUtensorMap mRlo,
                   const GradTcArgs p) {
  constexpr int EP = ep_of(D);
  constexpr int NW = 2 * (D + 1);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // rfull[s]: R_J planes of stage s landed; efull[s]: x_j | vy_j of stage s
  // landed; mdone[t % 8]: W(t) in TMEM and R stage of t free; wfree[b]: the
  // epilogue read W buffer b; efree[s]: the epilogue read stage s; lready: L_I in TMEM.
  __shared__ __align__(8) uint64_t bar_rfull[gMaxNM], bar_efull[gNE], bar_mdone[gRing], bar_wfree[gBufs],
      bar_efree[gNE], bar_lready;
  __shared__ double wacc[gEpiWarps][NW];
  __shared__ uint32_t tmem_slot;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sR = smem;                                                 // nm x [R_hi | R_lo]
  const float* sE = reinterpret_cast<const float*>(sR + static_cast<size_t>(p.nm) * p.mstage);  // gNE x [64][EP]
  double* sAcc = reinterpret_cast<double*>(smem + p.acc_off);        // [NW][384] per-row fp64 sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt = blockIdx.x / p.splits, sp = blockIdx.x % p.splits;
  const int jt_begin = static_cast<int>(static_cast<int64_t>(p.num_jt) * sp / p.splits);
  const int jt_end = static_cast<int>(static_cast<int64_t>(p.num_jt) * (sp + 1) / p.splits);
  const int T = jt_end - jt_begin;
  const int NM = p.nm;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NM; ++i) mbar_init(&bar_rfull[i], 1);
    for (int i = 0; i < gNE; ++i) {
      mbar_init(&bar_efull[i], 1);
      mbar_init(&bar_efree[i], 4);
    }
    for (int i = 0; i < gRing; ++i) mbar_init(&bar_mdone[i], 1);
    for (int i = 0; i < gBufs; ++i) mbar_init(&bar_wfree[i], 4);
    mbar_init(&bar_lready, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == gWarpAlloc) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_slot;

  if (warp == gWarpProd) {
    // ------------------------------------------------------------ producer
    // Ring slots / phases advance incrementally (no runtime divisions in the
    // single-warp loops).
    int sm = 0, se = 0, eround = 0;
    const uint32_t plane = p.mstage / 2;
    for (int t = 0; t < T; ++t) {
      const int pt = (jt_begin + t) * gTJ;
      if (t >= NM) mbar_wait(&bar_mdone[(t - NM) & (gRing - 1)], ((t - NM) >> 3) & 1);
      uint8_t* rb = sR + static_cast<size_t>(sm) * p.mstage;
      mbar_expect_tx_warp(&bar_rfull[sm], p.mstage);
      for (int kb = 0; kb < p.spk / 32; ++kb) {
        tma_load_2d_warp(rb + kb * 8192, &mRhi, &bar_rfull[sm], 32 * kb, pt);
        tma_load_2d_warp(rb + plane + kb * 8192, &mRlo, &bar_rfull[sm], 32 * kb, pt);
      }
      if (eround > 0) mbar_wait(&bar_efree[se], (eround - 1) & 1);
      mbar_expect_tx_warp(&bar_efull[se], p.estage);
      bulk_load_warp(const_cast<float*>(sE) + se * (p.estage / 4), p.xv + static_cast<int64_t>(pt) * EP, p.estage,
                     &bar_efull[se]);
      if (++sm == NM) sm = 0;
      if (++se == gNE) se = 0, ++eround;
    }
  } else if (warp == gWarpMma) {
    // ------------------------------------------------------------ MMA issuer
    // W(t) = L_I R_J^T into buffer t % 6: spk / 8 K steps of 3xTF32, A (L_I
    // hi / lo) from TMEM, B (R_J hi / lo, 64 points x 8 K, 128-byte swizzle) from shared memory.
    if (T > 0) {
      constexpr uint32_t idesc = idesc_tf32(gTI, gTJ);
      mbar_wait(&bar_lready, 0);
      tc_after();
      const int nk = p.spk / 8;
      const uint32_t plane = p.mstage / 2;
      int sm = 0, b = 0, bround = 0;
      uint32_t rph = 0;
      for (int t = 0; t < T; ++t) {
        if (bround > 0) mbar_wait(&bar_wfree[b], (bround - 1) & 1);
        mbar_wait(&bar_rfull[sm], rph);
        tc_after();
        const uint8_t* rb = sR + static_cast<size_t>(sm) * p.mstage;
        const uint32_t dcol = tmem + static_cast<uint32_t>(b) * gTJ;
#pragma unroll 8
        for (int k = 0; k < nk; ++k) {
          const uint64_t dh = umma_desc(rb + (k >> 2) * 8192) + 2 * (k & 3);
          const uint64_t dl = umma_desc(rb + plane + (k >> 2) * 8192) + 2 * (k & 3);
          mma3_ts(dcol, tmem + gLhi + 8 * k, tmem + gLlo + 8 * k, dh, dl, idesc, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar_mdone[t & (gRing - 1)]);
        if (++sm == NM) sm = 0, rph ^= 1u;
        if (++b == gBufs) b = 0, ++bround;
      }
    }
  } else if (warp < gEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3, w = warp >> 2;
    const int row = q * 32 + lane;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int64_t gi = static_cast<int64_t>(rt) * gTI + row;
    const bool valid = gi < p.n;
    float xi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) xi[k] = valid ? p.xs[gi * p.dp + k] : 0.f;
    const float hvy = valid ? 0.5f * p.vy[gi] : 0.f;
    if (w == 0 && T > 0) {
      // L_I (row gi, columns [0, spk), zero past s and past n) -> TMEM hi / lo planes
      for (int kb = 0; kb < p.spk / 32; ++kb) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int col = 32 * kb + c;
          const float v = (valid && col < p.s) ? p.L[gi + static_cast<int64_t>(col) * p.ld] : 0.f;
          hi[c] = __float_as_uint(v) & gTfMask;
          lo[c] = __float_as_uint(v - __uint_as_float(hi[c]));
        }
        __syncwarp();
        tmem_st32(tmem + lanes + gLhi + 32 * kb, hi);
        tmem_st32(tmem + lanes + gLlo + 32 * kb, lo);
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_lready);
    }
    double* acc64 = sAcc + warp * 32 + lane;  // slot k at acc64[k * 384]
#pragma unroll
    for (int k = 0; k < NW; ++k) acc64[k * gEpiThreads] = 0.0;
    const float sf2 = p.sf2, ac = p.a;
    float A[D + 1], B[D + 1];
#pragma unroll
    for (int k = 0; k <= D; ++k) A[k] = B[k] = 0.f;
    auto flush = [&]() {
#pragma unroll
      for (int k = 0; k <= D; ++k) {
        acc64[k * gEpiThreads] += static_cast<double>(A[k]);
        acc64[(D + 1 + k) * gEpiThreads] += static_cast<double>(B[k]);
        A[k] = B[k] = 0.f;
      }
    };
    int since = 0;
    for (int t = w; t < T; t += gEpiGroups) {
      const int b = t % gBufs, se = t % gNE;
      mbar_wait(&bar_mdone[t & (gRing - 1)], (t >> 3) & 1);
      mbar_wait(&bar_efull[se], (t / gNE) & 1);
      tc_after();
      const float* ev = sE + se * (p.estage / 4);
#pragma unroll 1
      for (int h = 0; h < gTJ / 16; ++h) {
        uint32_t wr[16];
        __syncwarp();
        tmem_ld16(tmem + lanes + static_cast<uint32_t>(b * gTJ + 16 * h), wr);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float* xj = ev + (16 * h + e) * EP;  // warp-uniform: shared-memory broadcast
          float xv[EP];
#pragma unroll
          for (int c = 0; c < EP / 4; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(xj + 4 * c);
            xv[4 * c] = v.x, xv[4 * c + 1] = v.y, xv[4 * c + 2] = v.z, xv[4 * c + 3] = v.w;
          }
          float dq[D];
          float r2 = 0.f;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const float df = xi[k] - xv[k];
            r2 = fmaf(df, df, r2);
            dq[k] = df * df;
          }
          const float u = sqrt_approx(r2);
          const float dec = ex2_approx(-u);
          const float kv = fmaf(ac, u, sf2) * dec;
          const float vyj = xv[D];
          const float wb = __uint_as_float(wr[e]);
          const float dA = dec * vyj, dB = dec * wb;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            A[k] = fmaf(dq[k], dA, A[k]);
            B[k] = fmaf(dq[k], dB, B[k]);
          }
          A[D] = fmaf(kv, vyj, A[D]);
          B[D] = fmaf(kv, wb, B[D]);
        }
      }
      tc_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bar_wfree[b]);
        mbar_arrive(&bar_efree[se]);
      }
      if (++since == gFlushTiles) {
        flush();
        since = 0;
      }
    }
    flush();
    // row scale (W^A = vy_i vy_j / 2: the vy_i / 2 factor; coef_b for W^B),
    // then the fixed-order warp sums
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      double v = acc64[k * gEpiThreads] * (k <= D ? static_cast<double>(hvy) : static_cast<double>(p.coef_b));
      v = warp_sum(v);
      if (lane == 0) wacc[warp][k] = v;
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x < NW) {
    double s = 0.0;
    for (int w = 0; w < gEpiWarps; ++w) s += wacc[w][threadIdx.x];
    p.part[static_cast<int64_t>(blockIdx.x) * NW + threadIdx.x] = s;
  }
  if (warp == gWarpAlloc) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// R (column-major, ld) -> tf32 hi / lo planes [n_pad][spk] (point-major, K
// contiguous: the MMA's K-major B operand), and xv [n_pad][ep] = x_j | vy_j.
// 32 points per CTA through a shared-memory transpose (coalesced both ways).
__global__ void grad_tc_prep_kernel(const float* R, int64_t ld, int s, const float* xs, int dp, int d,
                                    const float* vy, int64_t n, int spk, int ep, float* rhi, float* rlo, float* xv) {
  __shared__ float tile[64][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 x 32
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int c = ty; c < spk; c += 8) tile[c][tx] = (i0 + tx < n && c < s) ? R[i0 + tx + static_cast<int64_t>(c) * ld] : 0.f;
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    for (int c = tx; c < spk; c += 32) {
      const float v = tile[c][r];
      const float h = __uint_as_float(__float_as_uint(v) & gTfMask);
      rhi[(i0 + r) * spk + c] = h;
      rlo[(i0 + r) * spk + c] = v - h;
    }
    for (int k = tx; k < ep; k += 32) {
      const int64_t i = i0 + r;
      float v = 0.f;
      if (i < n) v = k < d ? xs[i * dp + k] : (k == d ? vy[i] : 0.f);
      xv[i * ep + k] = v;
    }
  }
}

int choose_grad_splits(int64_t row_tiles, int jt, int sms) {
  constexpr double kCtaOverheadTiles = 8.0;
  int best = 1;
  double best_cost = 1e300;
  for (int sp = 1; sp <= 64; ++sp) {
    if (sp > 1 && jt / sp < 8) break;
    const double waves = std::ceil(static_cast<double>(row_tiles * sp) / sms);
    const double cost = waves * (std::ceil(static_cast<double>(jt) / sp) + kCtaOverheadTiles);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

template <int D>
void launch_grad_tc(const CUtensorMap& mh, const CUtensorMap& ml, const GradTcArgs& a, unsigned grid, int smem,
                    cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    WGP_CUDA(cudaFuncSetAttribute(grad_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, gSmemLimit));
    configured = true;
  }
  grad_tc_kernel<D><<<grid, gThreads, smem, st>>>(mh, ml, a);
  WGP_LAUNCH_CHECK();
}

}  // namespace

bool grad_tc_supported(int d, int s) { return d >= 1 && d <= 12 && s >= 1 && s <= 64; }

GradTcPlan grad_tc_plan(int64_t n, int d, int s) {
  GradTcPlan pl;
  pl.n_pad = round_up(std::max<int64_t>(n, 1), gTJ);
  pl.spk = s <= 32 ? 32 : 64;
  pl.ep = ep_of(d);
  const int64_t row_tiles = ceil_div(n, gTI);
  const int jt = static_cast<int>(ceil_div(n, gTJ));
  static const int force = [] {
    const char* e = getenv("WGP_GRAD_SPLITS");
    return e ? atoi(e) : 0;
  }();
  pl.splits = force > 0 ? std::min(force, jt) : choose_grad_splits(row_tiles, jt, tc_sm_count());
  pl.nblk = static_cast<int>(row_tiles * pl.splits);
  pl.ws_bytes = sizeof(float) * static_cast<size_t>(pl.n_pad) * (2 * pl.spk + pl.ep);
  return pl;
}

void grad_tc(const GradParams& p, const GradTcPlan& pl, void* ws, cudaStream_t st) {
  if (!grad_tc_supported(p.d, p.s)) throw std::invalid_argument("grad_tc: needs 1 <= d <= 12 and 1 <= s <= 64");
  float* rhi = static_cast<float*>(ws);
  float* rlo = rhi + pl.n_pad * pl.spk;
  float* xv = rlo + pl.n_pad * pl.spk;
  grad_tc_prep_kernel<<<static_cast<unsigned>(pl.n_pad / 32), 256, 0, st>>>(p.R, p.ld, p.s, p.xs, p.dp, p.d, p.vy,
                                                                             p.n, pl.spk, pl.ep, rhi, rlo, xv);
  WGP_LAUNCH_CHECK();
  const CUtensorMap mh = tc_tensor_map(rhi, pl.spk, pl.n_pad, pl.spk * 4, 32, gTJ);
  const CUtensorMap ml = tc_tensor_map(rlo, pl.spk, pl.n_pad, pl.spk * 4, 32, gTJ);
  GradTcArgs a{};
  a.n = p.n;
  a.d = p.d;
  a.dp = p.dp;
  a.s = p.s;
  a.spk = pl.spk;
  a.num_jt = static_cast<int>(ceil_div(p.n, gTJ));
  a.splits = pl.splits;
  a.mstage = 2u * static_cast<uint32_t>(pl.spk / 32) * 8192u;
  a.estage = static_cast<uint32_t>(gTJ * pl.ep * 4);
  const int acc_bytes = 2 * (p.d + 1) * gEpiThreads * 8;
  const int fixed = gNE * static_cast<int>(a.estage) + acc_bytes + 1024;
  a.nm = std::min(gMaxNM, (gSmemLimit - fixed) / static_cast<int>(a.mstage));
  if (a.nm < 2) throw DeviceError("grad_tc: shared memory too small for the R ring");
  a.acc_off = static_cast<uint32_t>(a.nm) * a.mstage + gNE * a.estage;
  const int smem = static_cast<int>(a.acc_off) + acc_bytes + 1024;
  a.xs = p.xs;
  a.vy = p.vy;
  a.xv = xv;
  a.L = p.L;
  a.ld = p.ld;
  a.sf2 = p.sf2;
  a.a = p.a;
  a.coef_b = p.coef_b;
  a.part = p.part;
  const unsigned grid = static_cast<unsigned>(pl.nblk);
  switch (p.d) {
#define WGP_GRAD_CASE(D) \
  case D:                \
    return launch_grad_tc<D>(mh, ml, a, grid, smem, st);
    WGP_GRAD_CASE(1)
    WGP_GRAD_CASE(2)
    WGP_GRAD_CASE(3)
    WGP_GRAD_CASE(4)
    WGP_GRAD_CASE(5)
    WGP_GRAD_CASE(6)
    WGP_GRAD_CASE(7)
    WGP_GRAD_CASE(8)
    WGP_GRAD_CASE(9)
    WGP_GRAD_CASE(10)
    WGP_GRAD_CASE(11)
    WGP_GRAD_CASE(12)
#undef WGP_GRAD_CASE
    default:
      throw std::invalid_argument("grad_tc: unsupported d");
  }
}

}  // namespace wgp
