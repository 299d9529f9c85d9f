// hv_i8.cu — the fp64 CG operator as an exact integer-slice product on the
// 5th-generation tensor core (tcgen05.mma kind::i8, int32 accumulation).
//
// What it computes: the same fixed symmetric linear map as hv_f64.cu's DMMA
// engine, H V with entries k_ij from direct coordinate differences (bitwise
// symmetric) -- but K.V is done exactly in integers instead of in fp64:
//   * entries: k_ij in fp32 bit for bit as the DMMA engine forms them, as the
//     39-bit integer K_ij = rint(k_ij 2^eK) (sf^2 2^eK in [2^38, 2^39)): k_ij
//     itself for k_ij >= sf^2 2^-15, within 2^-39 sf^2 below -- the same
//     FIXED symmetric operator up to those tiny entries (fixed
//     symmetric perturbations cost CG nothing; noise that is not a fixed
//     linear map does), split into five unsigned bytes K = sum_i K_i 256^i;
//   * V: each column scaled by a power of two 2^e_c so its max |v| lands in
//     [2^53, 2^54), rounded to an integer (2^-53 of the column max) and split
//     into seven balanced signed bytes V = sum_j V_j 256^j;
//   * K.V = sum_ij 256^(i+j) K_i V_j: every byte product is exact and every
//     int32 accumulation is exact (drained to fp64 every 192 tiles, before it
//     could overflow).  Classes i + j = 3..10 are kept (29 byte pairs); the
//     dropped classes 0..2 weigh < 2^-60 of the result, so the product is
//     linear in V to fp64 rounding and deterministic.  (Keeping only classes
//     5..10 -- linear to ~1e-12 -- cost CG 5-11% more iterations than the
//     DMMA engine on fixed config-2 systems: scripts/diag_cg_engines.py.)
// Eight classes of N = s padded to 16 int32 columns fill TMEM for s <= 64;
// the 65th column (the configs' s = 65: 64 probes + y) runs on the fp64 pipe
// in the entry warps (one DFMA per entry, exactly the DMMA engine's
// arithmetic); wider V is done in column chunks (each re-evaluates K).
// One MMA per K byte covers up to 256 / N consecutive V bytes (their classes
// are consecutive accumulators): 18 kind::i8 MMAs (M = 128, K = 32) per
// 64-point tile at s = 65.
//
// Warp roles (320 threads): warps 0..7 evaluate the entries (warp w: rows
// 32 (w % 4) .. +31 = its TMEM lane quarter, points 32 (w / 4) .. +31 of each
// tile, all 32 at once for independent dependency chains) and write K's bytes
// into the 64-byte-swizzled K-major A operand in shared memory (one 8 KB block
// per byte), accumulate the 65th column, and drain / re-zero the accumulators
// into the fp64 split partials; warp 8 streams the per-tile V byte images
// (pre-swizzled by i8_vimg_kernel) and the tile's negated coordinates with 1-D
// bulk copies; warp 9 issues the MMAs.
// Output: fp64 split partials in hv64's layout (hv64_reduce_kernel / the
// CG fold add the diagonal and sum the splits in order).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "hv_f64.cuh"
#include "tc_ptx.cuh"

namespace wgp {
namespace {

constexpr int TI = 128;          // output rows per CTA (MMA M, TMEM lanes)
constexpr int TJ = 64;           // points per tile (two K steps of 32 bytes)
constexpr int kNCls = 8;         // accumulator classes i + j = 3 .. 10
constexpr int kNVB = 7;          // V bytes 0..6
constexpr int kMaxSm = 64;       // columns on the tensor core (8 x 64 TMEM columns)
constexpr int kTailMax = 1;      // column 64 on the fp64 pipe (4 columns: register spills in the entry loop)
constexpr int kChunk = 192;      // tiles between drains (int32 headroom: < 2^31 / (5 x 64 x 255 x 128) = 205)
constexpr int kMaxD = 16;        // coordinates kept in registers
#ifndef WGP_I8_ABLATE
#define WGP_I8_ABLATE 0
#endif
#ifndef WGP_I8_NBK
#define WGP_I8_NBK 3  // 4.23 vs 4.33 ms per config-2 CG iteration with 2 (interleaved A/B, before the tail fixes)
#endif
constexpr int NBK = WGP_I8_NBK, NV = 3;   // K buffers, V / coordinate stages
#ifndef WGP_I8_EPI
#define WGP_I8_EPI 8  // with 32-point groups: 3.31 ms per config-2 CG iteration vs 3.47 for 16 warps x 16-point groups (interleaved A/B)
#endif
constexpr int kEpiWarps = WGP_I8_EPI;                 // entry warps: 4 lane quarters x kEpiWarps / 4 point slices
constexpr int kWarpProd = kEpiWarps, kWarpMma = kEpiWarps + 1, kThreads = 32 * (kEpiWarps + 2);
constexpr int kPW = 4 * TJ / kEpiWarps;               // points per entry warp per tile (32 or 16)
#ifndef WGP_I8_G
#define WGP_I8_G 32  // one group per warp-tile: 16-point groups 3.43 vs 8-point 3.87 ms (16 warps), 32 with 8 warps 3.31 ms -- independent chains
#endif
constexpr int kG = WGP_I8_G;                          // points per entry group (8 or 16)
static_assert(kPW % kG == 0 && kG % 4 == 0, "entry groups of whole quads");
static_assert(kPW % 16 == 0, "16-byte K chunks per warp");
constexpr int kNKB = 5;                            // K bytes (39-bit K)
constexpr uint32_t kKBlk = TI * 64u;           // one K byte: 128 rows x 64 points, 64-byte swizzle
constexpr uint32_t kKBuf = kNKB * kKBlk;       // 40 KB

// V stage: bytes j = 0..6, each spad rows (columns of V) x 64 points, 64-byte
// swizzle, stacked so that consecutive bytes form one B operand of N = L spad;
// then the tail columns in fp64, [tail][64]
__host__ __device__ inline uint32_t vstage_bytes(int spad, int tail) {  // (1024-aligned stages)
  return (static_cast<uint32_t>(kNVB) * static_cast<uint32_t>(spad) * 64u + static_cast<uint32_t>(tail) * 64u * 8u +
          1023u) & ~1023u;
}
// UMMA shared-memory descriptor, K-major, 64-byte swizzle (8-row atoms of 512 bytes)
__device__ __forceinline__ uint64_t umma_desc_sw64(const void* p) {
  const uint32_t a = smem_u32(p);
  return static_cast<uint64_t>((a >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(4) << 61);
}

struct I8Args {
  const float* xs;     // [n_pad][dp] prepared points
  const float* xtile;  // [num_jt][D][64] the tiles' points, negated, coordinate-major
  int dp, d;
  int64_t n, r0, m;  // contracted points, first output row (global), rows
  int num_jt, splits, s, spad;  // s: columns of the whole partial buffer
  int s_mma, tail, c_off;        // this launch: columns c_off .. + s_mma on MMAs, then tail on DFMA
  const uint8_t* vimg;   // [num_jt] x vstage_bytes(spad, tail) swizzled V byte images + fp64 tail
  const double* vscale;  // [s_mma] 2^-e_c
  const float* hyp;      // device [sf2, a, diag]
  double* part;          // [splits][s][m_pad] fp64 partials
  int64_t m_pad;
  const int* done;
};

// One tile's MMAs: for K byte i its partner V bytes j = max(0, 3 - i) .. 6
// are consecutive row blocks of the V stage and their classes i + j - 3
// consecutive accumulators, so one instruction covers up to 256 / spad of
// them (the A tile is read once per group instead of once per pair -- the
// shared-memory reads of the operands bound the SS MMAs).  ka / vb: shared
// addresses of K byte 0 and V byte 0.  The accumulators are zeroed by the
// entry warps at the start and after every drain, so every MMA accumulates.
// (SPAD known at compile time: every descriptor is the tile's two base
// descriptors plus a constant, ~3 instructions per MMA for the issuing
// thread instead of ~25 with runtime group bounds and descriptor builds)
template <int SPAD>
__device__ __forceinline__ void mma_tile_i8_t(uint32_t d, uint64_t ka, uint64_t vb, uint32_t idesc_base) {
  constexpr int G = 256 / SPAD < kNVB ? 256 / SPAD : kNVB;  // bytes per instruction
#pragma unroll
  for (int i = 0; i < kNKB; ++i) {
    const int j0 = 3 - i > 0 ? 3 - i : 0;
#pragma unroll
    for (int jg = j0; jg < kNVB; jg += G) {
      const int L = kNVB - jg < G ? kNVB - jg : G;
      const uint64_t a = ka + static_cast<uint64_t>(i * (kKBlk >> 4));
      const uint64_t b = vb + static_cast<uint64_t>(jg * (SPAD * 64 >> 4));
      const uint32_t dc = d + static_cast<uint32_t>(SPAD * (i + jg - 3));
      const uint32_t idesc = idesc_base | (static_cast<uint32_t>((L * SPAD) >> 3) << 17);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dc), "l"(a + 2 * ks),
                     "l"(b + 2 * ks), "r"(idesc));
    }
  }
}
__device__ __forceinline__ void mma_tile_i8(uint32_t d, uint64_t ka, uint64_t vb, int spad, uint32_t idesc_base) {
  switch (spad) {
    case 16: mma_tile_i8_t<16>(d, ka, vb, idesc_base); break;
    case 32: mma_tile_i8_t<32>(d, ka, vb, idesc_base); break;
    case 48: mma_tile_i8_t<48>(d, ka, vb, idesc_base); break;
    default: mma_tile_i8_t<64>(d, ka, vb, idesc_base); break;
  }
}

// fp32 -> fp64 of an entry for the 65th column (F2F; the bits re-biased on
// the integer pipe instead measured the same)
__device__ __forceinline__ double f2d(float x) { return static_cast<double>(x); }

__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr), "r"(0)
               : "memory");
}

__device__ __forceinline__ void commit_one(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) hv_i8_kernel(const I8Args p) {
  if (p.done && *p.done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t vsb = vstage_bytes(p.spad, p.tail);
  uint8_t* sK = smem;                                  // NBK x 32 KB
  uint8_t* sV = sK + NBK * kKBuf;                      // NV x vsb (multiples of 1024)
  float* sX = reinterpret_cast<float*>(sV + NV * vsb); // NV x [D][TJ] negated coordinates
  __shared__ __align__(8) uint64_t bar_vfull[NV], bar_kfull[NBK], bar_mdone[8], bar_ofull, bar_odrained;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row_tiles = static_cast<int>(gridDim.x) / p.splits;
  const int rt = blockIdx.x % row_tiles, sp = blockIdx.x / row_tiles;  // split-major (L2)
  const int jt0 = static_cast<int>(static_cast<int64_t>(p.num_jt) * sp / p.splits);
  const int T = static_cast<int>(static_cast<int64_t>(p.num_jt) * (sp + 1) / p.splits) - jt0;
  constexpr uint32_t xbytes = static_cast<uint32_t>(TJ * D * 4);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NV; ++i) mbar_init(&bar_vfull[i], 1);
    for (int i = 0; i < NBK; ++i) mbar_init(&bar_kfull[i], kEpiWarps);
    for (int i = 0; i < 8; ++i) mbar_init(&bar_mdone[i], 1);
    mbar_init(&bar_ofull, 1);
    mbar_init(&bar_odrained, kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWarpProd) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_slot;

  if (warp == kWarpProd) {
    // -------------------------------------------------------------- producer
    for (int t = 0; t < T; ++t) {
      const int st = t % NV;
      if (t >= NV) mbar_wait(&bar_mdone[(t - NV) & 7], ((t - NV) >> 3) & 1);
      mbar_expect_tx_warp(&bar_vfull[st], vsb + xbytes);
      const int64_t jt = jt0 + t;
      bulk_load_warp(sV + st * vsb, p.vimg + jt * vsb, vsb, &bar_vfull[st]);
      bulk_load_warp(sX + st * TJ * D, p.xtile + jt * TJ * D, xbytes, &bar_vfull[st]);
    }
  } else if (warp == kWarpMma) {
    // -------------------------------------------------------------- MMA issuer
    const uint64_t dK0 = umma_desc_sw64(sK), dV0 = umma_desc_sw64(sV);  // + (byte offset >> 4) per buffer / stage
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) |
                           (static_cast<uint32_t>(TI >> 4) << 24);  // D s32, A u8, B s8, K-major (+ N per group)
    int nz = 0;  // accumulator zeroings (the start, then after every drain)
    for (int t = 0; t < T; ++t) {
      const int b = t % NBK, st = t % NV;
      if (t % kChunk == 0) {  // the accumulators are zero
        mbar_wait(&bar_odrained, nz & 1);
        ++nz;
      }
      mbar_wait(&bar_kfull[b], (t / NBK) & 1);
      mbar_wait(&bar_vfull[st], (t / NV) & 1);
      tc_after();
      // lane 0 issues the tile's MMAs and the commits that track them
      if (lane == 0) {
#if !(WGP_I8_ABLATE & 1)  // (ablation build: no MMAs)
        mma_tile_i8(tmem, dK0 + static_cast<uint64_t>((b * kKBuf) >> 4), dV0 + static_cast<uint64_t>((st * vsb) >> 4),
                    p.spad, idesc);
#endif
        commit_one(&bar_mdone[t & 7]);
        if ((t + 1) % kChunk == 0 || t == T - 1) commit_one(&bar_ofull);
      }
      __syncwarp();
    }
  } else {
    // -------------------------------------------------------------- entries + drains
    const int q = warp & 3, h = warp >> 2;
    const int r = 32 * q + lane;  // row in the tile = TMEM lane
    const int64_t lr = static_cast<int64_t>(rt) * TI + r;
    const int64_t g = p.r0 + lr;  // global row (n_pad rows of xs exist)
    // (x_ik, x_ik) pairs: x_i - x_j for two points per FADD2 against the
    // tile's negated coordinates; (x_i - x_j)^2 = (x_j - x_i)^2 exactly and
    // the sum runs k = 0..D-1 for both orders, so K is bitwise symmetric
    float2 xi2[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float v = p.xs[g * p.dp + k];
      xi2[k] = make_float2(v, v);
    }
    const uint32_t lanes = static_cast<uint32_t>(32 * q) << 16;
    // k_ij = (sf^2 + a u) 2^-u in fp32 exactly as the DMMA engine forms it,
    // then scaled by 2^eK (exact), sf^2 2^eK in [2^30, 2^31): K_ij is k_ij
    // itself for k_ij >= sf^2 2^-7 and within 2^-31 sf^2 below
    const float hsf2 = p.hyp[0], ha = p.hyp[1];
    const int eK = 38 - (static_cast<int>((__float_as_uint(hsf2) >> 23) & 255u) - 127);
    const float kscale = __int_as_float((127 + eK) << 23);
    // (sf^2 + a u) 2^-u 2^eK = (sf^2 2^eK + a 2^eK u) 2^-u bit for bit: power-of-two scaling is exact
    const float hsS = hsf2 * kscale, haS = ha * kscale;
    const double oscale = ldexp(1.0, -eK);
    double acct[4] = {0.0, 0.0, 0.0, 0.0};  // column 64: this row, this warp's points (point mod 4), fp64
    // zero this warp's accumulator pieces before the first MMA
    if (T > 0) {
#pragma unroll 1
      for (int c0 = 8 * h; c0 < p.spad; c0 += 8 * (kEpiWarps / 4))
#pragma unroll
        for (int c = 0; c < kNCls; ++c) tmem_zero8(tmem + lanes + static_cast<uint32_t>(c * p.spad + c0));
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_odrained);
    }
    int nd = 0;
    for (int t = 0; t < T; ++t) {
      const int b = t % NBK, st = t % NV;
      mbar_wait(&bar_vfull[st], (t / NV) & 1);
      if (t >= NBK) mbar_wait(&bar_mdone[(t - NBK) & 7], ((t - NBK) >> 3) & 1);  // K buffer b is free
      const uint32_t xt_s = smem_u32(sX + st * TJ * D + kPW * h);  // [k][64] negated, this warp's points
      const int64_t pbase = static_cast<int64_t>(jt0 + t) * TJ + kPW * h;  // this warp's first point
      // warp-uniform: do any of the warp's entries need zeroing?
      const bool edge = pbase + kPW > p.n || __any_sync(0xffffffffu, g >= pbase && g < pbase + kPW);
      uint32_t w[kNKB][kPW / 4];  // digit i: kPW bytes (points 4 c .. 4 c + 3 in word c)
#if WGP_I8_ABLATE & 2  // (ablation build: no entry math)
#pragma unroll
      for (int i = 0; i < kNKB; ++i)
#pragma unroll
        for (int c = 0; c < kPW / 4; ++c) w[i][c] = 0u;
#else
#pragma unroll
      for (int grp = 0; grp < kPW / kG; ++grp) {  // kG points at a time, packed in pairs
        float2 r2[kG / 2];
#pragma unroll
        for (int e = 0; e < kG / 2; ++e) r2[e] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          // explicit shared-space loads (a generic load through the cast
          // pointer waits on the long scoreboard)
#pragma unroll
          for (int qd = 0; qd < kG / 4; ++qd) {
            float4 a;
            const uint32_t ad = xt_s + static_cast<uint32_t>((k * TJ + kG * grp + 4 * qd) * 4);
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                         : "r"(ad));
            const float2 d0 = __fadd2_rn(xi2[k], make_float2(a.x, a.y));
            const float2 d1 = __fadd2_rn(xi2[k], make_float2(a.z, a.w));
            r2[2 * qd] = __ffma2_rn(d0, d0, r2[2 * qd]);
            r2[2 * qd + 1] = __ffma2_rn(d1, d1, r2[2 * qd + 1]);
          }
        }
        float kp[kG];  // the entries scaled by 2^eK, zero where excluded
#pragma unroll
        for (int e = 0; e < kG; ++e) {
          const float rr = (e & 1) ? r2[e >> 1].y : r2[e >> 1].x;
          kp[e] = matern_from_u(sqrt_approx(rr), hsS, haS);
        }
        if (edge) {  // the diagonal (H_ii V_i is added exactly in the reduction) and points >= n
#pragma unroll
          for (int e = 0; e < kG; ++e) {
            const int64_t gj = pbase + kG * grp + e;
            if (gj >= p.n || gj == g) kp[e] = 0.f;
          }
        }
        uint32_t K[kG], KH[kG];  // low 32 bits, bits 32..38
#pragma unroll
        for (int e = 0; e < kG; ++e) {
          // (the float's bits shifted on the integer pipe instead: 4.7 vs
          // 4.2 ms per config-2 CG iteration -- issue slots, not the
          // conversion pipe, bind)
          unsigned long long kv;
          asm("cvt.rni.sat.u64.f32 %0, %1;" : "=l"(kv) : "f"(kp[e]));
          K[e] = static_cast<uint32_t>(kv);
          KH[e] = static_cast<uint32_t>(kv >> 32);
        }
        if (p.tail > 0) {  // column 64: fp64 FMA of the fp32 entry (the DMMA engine's arithmetic), four chains
          const uint32_t vt = smem_u32(sV + st * vsb + kNVB * p.spad * 64) + 8u * (kPW * h + kG * grp);
#pragma unroll
          for (int e = 0; e < kG; e += 2) {
            double v0, v1;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v0), "=d"(v1) : "r"(vt + 8u * e));
            acct[e & 3] = fma(f2d(kp[e]), v0, acct[e & 3]);
            acct[(e + 1) & 3] = fma(f2d(kp[e + 1]), v1, acct[(e + 1) & 3]);
          }
        }
        // 4 x 4 byte transposes: w[i][.] holds byte i of 4 consecutive points
#pragma unroll
        for (int hq = 0; hq < kG / 4; ++hq) {
          const uint32_t t0 = __byte_perm(K[4 * hq], K[4 * hq + 1], 0x5140);
          const uint32_t t1 = __byte_perm(K[4 * hq], K[4 * hq + 1], 0x7362);
          const uint32_t t2 = __byte_perm(K[4 * hq + 2], K[4 * hq + 3], 0x5140);
          const uint32_t t3 = __byte_perm(K[4 * hq + 2], K[4 * hq + 3], 0x7362);
          const int wi = (kG / 4) * grp + hq;
          w[0][wi] = __byte_perm(t0, t2, 0x5410);
          w[1][wi] = __byte_perm(t0, t2, 0x7632);
          w[2][wi] = __byte_perm(t1, t3, 0x5410);
          w[3][wi] = __byte_perm(t1, t3, 0x7632);
          w[4][wi] = __byte_perm(__byte_perm(KH[4 * hq], KH[4 * hq + 1], 0x0040),
                                 __byte_perm(KH[4 * hq + 2], KH[4 * hq + 3], 0x0040), 0x5410);
        }
      }
#endif
      // K bytes -> the A operand: byte i's block, row r, 16-byte chunk c (of 4
      // per 64-point row) at (c ^ ((r % 8) / 2)) (64-byte swizzle)
      uint8_t* kb = sK + b * kKBuf + (r >> 3) * 512 + (r & 7) * 64;
#pragma unroll
      for (int i = 0; i < kNKB; ++i)
#pragma unroll
        for (int u = 0; u < kPW / 16; ++u) {
          const int c = (kPW / 16) * h + u;
          uint4 v = make_uint4(w[i][4 * u], w[i][4 * u + 1], w[i][4 * u + 2], w[i][4 * u + 3]);
          *reinterpret_cast<uint4*>(kb + i * kKBlk + ((c ^ ((r & 7) >> 1)) << 4)) = v;
        }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_kfull[b]);
      if ((t + 1) % kChunk == 0 || t == T - 1) {
        // drain: class sums -> fp64, this warp's share of the columns
        mbar_wait(&bar_ofull, nd & 1);
        tc_after();
        // 8-column pieces dealt round-robin to the warps sharing the lane quarter
#pragma unroll 1
        for (int c0 = 8 * h; c0 < p.spad; c0 += 8 * (kEpiWarps / 4)) {
          double vs[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int hf = 1; hf >= 0; --hf) {  // classes 7..4, then 3..0: high first, fixed order
            uint32_t cv[kNCls / 2][8];
#pragma unroll
            for (int c = 0; c < kNCls / 2; ++c)
              tmem_ld8(tmem + lanes + static_cast<uint32_t>((4 * hf + c) * p.spad + c0), cv[c]);
            tmem_wait_ld();
            if (t + 1 < T)  // the next chunk accumulates from zero
#pragma unroll
              for (int c = 0; c < kNCls / 2; ++c)
                tmem_zero8(tmem + lanes + static_cast<uint32_t>((4 * hf + c) * p.spad + c0));
#pragma unroll
            for (int e = 0; e < 8; ++e)
#pragma unroll
              for (int c = kNCls / 2 - 1; c >= 0; --c)
                vs[e] += ldexp(static_cast<double>(static_cast<int>(cv[c][e])), 8 * (4 * hf + c + 3));
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = c0 + e;
            if (col < p.s_mma && lr < p.m) {
              double* dst = p.part + (static_cast<int64_t>(sp) * p.s + p.c_off + col) * p.m_pad + lr;
              const double val = vs[e] * p.vscale[col] * oscale;
              *dst = nd == 0 ? val : *dst + val;
            }
          }
        }
        tmem_wait_st();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_odrained);
        ++nd;
      }
    }
    if (p.tail > 0) {
      // column 64: the kEpiWarps / 4 warps of a lane quarter summed in
      // a fixed order through shared memory (the K buffers are free: every
      // MMA completed before the final drain)
      double* scr = reinterpret_cast<double*>(sK);
      scr[h * TI + r] = (acct[0] + acct[1]) + (acct[2] + acct[3]);
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
      if (h == 0 && lr < p.m) {
        double v = 0.0;
        for (int hh = 0; hh < kEpiWarps / 4; ++hh) v += scr[hh * TI + r];
        p.part[(static_cast<int64_t>(sp) * p.s + p.c_off + p.s_mma) * p.m_pad + lr] = v * oscale;
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == kWarpProd) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Per column: max |v| (fp64 bits are monotone in |v|) -> colbits[c].
__global__ void i8_colmax_kernel(const double* V, int64_t ldv, int64_t n, unsigned long long* colbits) {
  const int c = blockIdx.y;
  unsigned long long m = 0ull;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, static_cast<unsigned long long>(__double_as_longlong(V[j + c * ldv])) & 0x7FFFFFFFFFFFFFFFull);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(colbits + c, m);
}

// Column exponent: max |v| 2^e in [2^53, 2^54) (e = 0 for a zero or
// non-finite column: its digits are then 0 / garbage-free, see below).
__device__ __forceinline__ int col_exp(unsigned long long mbits) {
  const double m = __longlong_as_double(static_cast<long long>(mbits));
  if (!(m > 0.0) || !isfinite(m)) return 0;
  int E;
  frexp(m, &E);  // m = f 2^E, f in [0.5, 1)
  return max(-1000, min(1000, 54 - E));
}

// V -> per-tile images: bytes j = 0..6 of the balanced base-256 digits of
// V 2^e_c for the s_mma MMA columns, [7][spad][64] (row = column of V, 64
// points, 16-byte chunks at (chunk ^ ((row % 8) / 2)): the UMMA 64-byte
// swizzle, K-major B operand), then the tail columns in fp64 [tail][64];
// vscale[c] = 2^-e_c.  One thread per 16-byte chunk of bytes / per tail value.
__global__ void i8_vimg_kernel(const double* V, int64_t ldv, int64_t n, int s_mma, int tail, int spad, int num_jt,
                               const unsigned long long* colbits, uint8_t* img, double* vscale) {
  // one thread per (tile, column, 16-point chunk): all seven digits of its 16
  // values (each value converted once), then the tail values
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nchunk = static_cast<int64_t>(spad) * 4, per_tile = nchunk + static_cast<int64_t>(tail) * TJ;
  if (idx >= per_tile * num_jt) return;
  const int64_t t = idx / per_tile;
  const int rem = static_cast<int>(idx - t * per_tile);
  uint8_t* timg = img + t * static_cast<int64_t>(vstage_bytes(spad, tail));
  if (rem >= nchunk) {  // a tail value
    const int q = rem - static_cast<int>(nchunk), c = q / TJ, pt = q % TJ;
    const int64_t j = t * TJ + pt;
    reinterpret_cast<double*>(timg + kNVB * spad * 64)[c * TJ + pt] = j < n ? V[j + (s_mma + c) * ldv] : 0.0;
    return;
  }
  const int row = rem / 4, chunk = rem % 4;
  const int c = row;
  const int p0 = 16 * chunk;
  uint32_t w[kNVB][4] = {};
  if (c < s_mma) {
    const int e = col_exp(colbits[c]);
    const double sc = ldexp(1.0, e);
    if (t == 0 && chunk == 0) {  // a non-finite column propagates NaN like the fp64 product
      const double m = __longlong_as_double(static_cast<long long>(colbits[c]));
      vscale[c] = isfinite(m) ? ldexp(1.0, -e) : __longlong_as_double(0x7FF8000000000000LL);
    }
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      const int64_t j = t * TJ + p0 + k;
      long long vi = 0;
      if (j < n) {
        const double x = V[j + c * ldv] * sc;
        vi = isfinite(x) ? __double2ll_rn(x) : 0ll;
      }
#pragma unroll
      for (int q = 0; q < kNVB; ++q) {  // balanced base-256 digits, least significant first
        const int dq = static_cast<int>(static_cast<signed char>(vi & 0xFF));
        vi = (vi - dq) >> 8;
        w[q][k / 4] |= (static_cast<uint32_t>(dq) & 0xFFu) << (8 * (k % 4));
      }
    }
  }
  uint8_t* dst = timg + (row >> 3) * 512 + (row & 7) * 64 + ((chunk ^ ((row & 7) >> 1)) << 4);
#pragma unroll
  for (int q = 0; q < kNVB; ++q)
    *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(q) * spad * 64) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
}

// xtile[t][k][p] = -xs[64 t + p][k] (points past n_pad read as zero rows of
// xs' padding; the entries of points >= n are zeroed in the kernel anyway).
__global__ void i8_xtile_kernel(const float* xs, int dp, int d, int64_t n_pad, int num_jt, float* xtile) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(num_jt) * d * TJ) return;
  const int64_t t = idx / (d * TJ);
  const int k = static_cast<int>((idx / TJ) % d), pt = static_cast<int>(idx % TJ);
  const int64_t j = t * TJ + pt;
  xtile[idx] = j < n_pad ? -xs[j * dp + k] : 0.f;
}

int i8_splits(int64_t n) {
  // keyed on the global n (row shards reproduce the full operator's rows):
  // whole waves of 148 CTAs, >= 4 tiles per split
  static const int force = [] {
    const char* e = getenv("WGP_I8_SPLITS");
    return e ? atoi(e) : 0;
  }();
  static const double fill = [] {
    const char* e = getenv("WGP_I8_FILL");
    return e ? atof(e) : 0.95;  // config 2: 4 splits (8.7 waves), 2.75 vs 2.96 ms per CG iteration with 2
  }();
  const int64_t rt = ceil_div(n, TI), nt = ceil_div(n, TJ);
  if (force > 0) return static_cast<int>(std::min<int64_t>(force, nt));
  const int64_t wave = 148;
  const int64_t smax = std::max<int64_t>(1, nt / 4);
  for (int64_t s = 1; s <= smax; ++s) {
    const int64_t ctas = rt * s;
    if (ctas < wave) continue;
    const double waves = static_cast<double>(ctas) / wave;
    if (waves / std::ceil(waves) >= fill) return static_cast<int>(s);
  }
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(smax, wave / rt)));
}

}  // namespace

bool hv_i8_supported(int d, int s) { return d >= 1 && d <= kMaxD && s >= 1; }

size_t hv_i8_workspace_bytes(int64_t n, int64_t m, int s) {
  const size_t part = sizeof(double) * static_cast<size_t>(i8_splits(n)) * s * round_up(m, TI);
  const size_t img = static_cast<size_t>(ceil_div(n, TJ)) * vstage_bytes(kMaxSm, kTailMax);
  const size_t xt = sizeof(float) * static_cast<size_t>(ceil_div(n, TJ)) * kMaxD * TJ;
  return round_up(part, 1024) + round_up(img, 1024) + 2 * 8 * 128 + round_up(xt, 1024);
}

// One launch over columns [c_off, c_off + s_mma + tail) of the partials.
static void i8_launch(const Hv64Params& hp, int c_off, int s_mma, int tail, int splits, int64_t m_pad,
                      uint8_t* img, unsigned long long* colbits, double* vscale, const float* xtile, cudaStream_t st) {
  const int spad = static_cast<int>(round_up(s_mma, 16));
  const int num_jt = static_cast<int>(ceil_div(hp.n, TJ));
  const double* V = hp.V + static_cast<int64_t>(c_off) * hp.ldv;
  WGP_CUDA(cudaMemsetAsync(colbits, 0, sizeof(unsigned long long) * kMaxSm, st));
  i8_colmax_kernel<<<dim3(static_cast<unsigned>(std::min<int64_t>(64, ceil_div(hp.n, 256))), s_mma), 256, 0,
                     st>>>(V, hp.ldv, hp.n, colbits);
  WGP_LAUNCH_CHECK();
  const int64_t items = (static_cast<int64_t>(spad) * 4 + static_cast<int64_t>(tail) * TJ) * num_jt;
  i8_vimg_kernel<<<static_cast<unsigned>(ceil_div(items, 256)), 256, 0, st>>>(V, hp.ldv, hp.n, s_mma, tail, spad,
                                                                            num_jt, colbits, img, vscale);
  WGP_LAUNCH_CHECK();
  I8Args a{};
  a.xs = hp.xs;
  a.xtile = xtile;
  a.dp = hp.dp;
  a.d = hp.d;
  a.n = hp.n;
  a.r0 = hp.r0;
  a.m = hp.m;
  a.num_jt = num_jt;
  a.splits = splits;
  a.s = hp.s;
  a.spad = spad;
  a.s_mma = s_mma;
  a.tail = tail;
  a.c_off = c_off;
  a.vimg = img;
  a.vscale = vscale;
  a.hyp = hp.hyp;
  a.part = hp.part;
  a.m_pad = m_pad;
  a.done = hp.done;
  const int smem = 1024 + NBK * static_cast<int>(kKBuf) + NV * static_cast<int>(vstage_bytes(spad, tail)) +
                   NV * TJ * hp.d * 4;
  const unsigned grid = static_cast<unsigned>(ceil_div(hp.m, TI) * splits);
  switch (hp.d) {
#define WGP_I8_CASE(D)                                            \
  case D:                                                         \
    WGP_SMEM_ATTR(hv_i8_kernel<D>, 225 * 1024);                   \
    hv_i8_kernel<D><<<grid, kThreads, smem, st>>>(a);             \
    break;
    WGP_I8_CASE(1) WGP_I8_CASE(2) WGP_I8_CASE(3) WGP_I8_CASE(4) WGP_I8_CASE(5) WGP_I8_CASE(6) WGP_I8_CASE(7)
    WGP_I8_CASE(8) WGP_I8_CASE(9) WGP_I8_CASE(10) WGP_I8_CASE(11) WGP_I8_CASE(12) WGP_I8_CASE(13)
    WGP_I8_CASE(14) WGP_I8_CASE(15) WGP_I8_CASE(16)
#undef WGP_I8_CASE
    default:
      throw std::invalid_argument("hv_i8: d > 16");
  }
  WGP_LAUNCH_CHECK();
}

bool hv_i8_partials(const Hv64Params& hp, cudaStream_t st, int* splits_out, int64_t* m_pad_out) {
  if (!hv_i8_supported(hp.d, hp.s) || hp.m <= 0) return false;
  const int num_jt = static_cast<int>(ceil_div(hp.n, TJ));
  const int splits = i8_splits(hp.n);
  const int64_t m_pad = round_up(hp.m, TI);
  uint8_t* ws = reinterpret_cast<uint8_t*>(hp.part);
  const size_t part_b = round_up(sizeof(double) * static_cast<size_t>(splits) * hp.s * m_pad, 1024);
  uint8_t* img = ws + part_b;
  const size_t img_b = round_up(static_cast<size_t>(num_jt) * vstage_bytes(kMaxSm, kTailMax), 1024);
  auto* colbits = reinterpret_cast<unsigned long long*>(img + img_b);
  double* vscale = reinterpret_cast<double*>(colbits + 128);
  float* xtile = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(colbits) + 2 * 8 * 128);
  {
    const int64_t nx = static_cast<int64_t>(num_jt) * hp.d * TJ;
    i8_xtile_kernel<<<static_cast<unsigned>(ceil_div(nx, 256)), 256, 0, st>>>(hp.xs, hp.dp, hp.d,
                                                                             round_up(hp.n, 128), num_jt, xtile);
    WGP_LAUNCH_CHECK();
  }
  // column chunks: 64 on the tensor core + up to kTailMax on the fp64 pipe
  for (int c0 = 0; c0 < hp.s;) {
    const int rest = hp.s - c0;
    const int s_mma = std::min(rest, kMaxSm);
    const int tail = rest - s_mma <= kTailMax ? rest - s_mma : 0;
    i8_launch(hp, c0, s_mma, tail, splits, m_pad, img, colbits, vscale, xtile, st);
    c0 += s_mma + tail;
  }
  if (splits_out) *splits_out = splits;
  if (m_pad_out) *m_pad_out = m_pad;
  return true;
}

}  // namespace wgp
