// hv_tc.cu — fused Matern-3/2 H.V on the 5th-generation tensor cores.
//
// Replaces the dense products H * V of the reference solvers
// (proj/src/solvers.cpp:71,92,110,120,169,186,188,211,242) without forming H.
// One CTA owns a 128-row tile I and streams 32-point tiles J (FlashAttention
// shape, no online-softmax state); the default engine is 3xTF32 throughout:
//
//   MMA-1  S[I,J]  = A_I . B_J^T           (tcgen05.mma kind::tf32, M=128, N=64:
//                    two J tiles per instruction, 3xTF32 hi.hi + hi.lo + lo.hi;
//                    a_i = [x_i, |x_i|^2, 1], b_j = [-2 x_j, 1, |x_j|^2] so
//                    S = u^2, the squared scaled distance, lands in TMEM; for
//                    d <= 19 the three passes are packed along K)
//   epilogue       k = sf^2 (1 + u ln2) 2^-u from S (tcgen05.ld -> registers,
//                    sqrt + ex2 on the MUFU), the diagonal entry zeroed
//                    (H_ii V_i = (sf^2 + sigma^2) V_i is added exactly at the end),
//                    k split into tf32 k_hi | k_lo, tcgen05.st back to TMEM in place
//   MMA-2  O[I,:] += K[I,J] . V[J,:]       (kind::tf32, A = K from TMEM, N = s
//                    padded to 16, 3xTF32 k_hi v_hi + k_hi v_lo + k_lo v_hi)
//
// Warp roles (512 threads): warps 0..11 epilogue (three warpgroups; group w
// takes tiles t = w, w+3, ...), warp 12 TMA producer of A_I and the B_J ring,
// 13 MMA-1 issuer, 14 TMA producer of the V_J ring (+ TMEM allocation), 15
// MMA-2 issuer.  TMEM (layout 2): two fp32 accumulators O0 | O1
// (double-buffered chunk drains), A_I hi/lo, and two 128-column groups each
// holding S(t) | S(t+1) and then, in place, their K planes -- 4 tiles in
// flight, so MMA-1 runs ahead of MMA-2 and one tile's epilogue hides behind
// the MMAs of the next (the fp16 engine: four epilogue warpgroups, 640
// threads, A_I in shared memory and five 64-point tiles in flight).  MMA-2
// accumulates in fp32 chunks of 32 tiles that the
// epilogue folds into a shared-memory fp32 sum and an fp64 CTA sum (error
// independent of n).  J tiles of a row tile may be split across CTAs (split
// count keyed on the global n, partials summed in fixed order ->
// deterministic and shard-invariant).  WGP_HV_TC_F16 selects the fp16x3 K.V
// engine (kind::f16, 64-point tiles, k1 v1 + k1 v2 + k2 v1 over V scaled per
// column by a power of two; bench.py's headline engine).

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <mutex>
#include <vector>
#include <utility>
#include <cstdlib>
#include <cstdio>

#include "common.cuh"
#include "hv_tc.cuh"
#include "tc_ptx.cuh"

namespace wgp {
namespace {

constexpr int kTI = 128;   // rows per tile (MMA M)
constexpr int kKA = 32;    // augmented Gram dimension (d + 2 <= 32)
#ifndef WGP_TC_EPI
#define WGP_TC_EPI 3
#endif
// fp16 engine: four epilogue warpgroups (its conversion keeps half a tile
// live, ~96 registers: no spills at 640 threads) and A_I in shared memory,
// so five tiles are in flight (TMEM: O0 | O1 + 5 x 64 columns); measured
// 0.1618 vs 0.1653 ms at config 1 for three groups with A_I in TMEM.
#ifndef WGP_TC_EPI16
#define WGP_TC_EPI16 4
#endif
#ifndef WGP_TC_F16_ATMEM
#define WGP_TC_F16_ATMEM 0
#endif
template <bool H16>
constexpr int kEpiGroupsT = H16 ? WGP_TC_EPI16 : WGP_TC_EPI;  // epilogue warpgroups
template <bool H16>
constexpr int kThreadsT = 128 * kEpiGroupsT<H16> + 128;  // + 4 control warps
constexpr uint32_t kTfMask = 0xFFFFE000u;  // keep sign, exponent, 10 mantissa bits
constexpr int kSmemLimit = 232448 - 2048;  // 227 KB opt-in minus static smem (barriers)
constexpr int kMaxStages = 8;              // smem ring depth cap (barrier arrays)
constexpr int kDoneRing = 8;               // MMA completion rings (>= kMaxStages, NBUF)

// 32 squared scaled distances -> tf32 hi / lo planes of k (k_hi keeps sign,
// exponent and 10 mantissa bits; k_lo = k - k_hi is exact); the diagonal
// entry (dg in [0, 32)) is zeroed: H_ii V_i is applied exactly at the end.
template <bool DIAG>
__device__ __forceinline__ void to_k(const uint32_t (&r)[32], uint32_t (&khi)[32], uint32_t (&klo)[32],
                                     float sf2, float ac, int dg) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float k = matern_from_u(sqrt_approx(fabsf(__uint_as_float(r[i]))), sf2, ac);
    khi[i] = __float_as_uint(k) & kTfMask;
    klo[i] = __float_as_uint(k - __uint_as_float(khi[i]));
    if (DIAG && dg == i) {
      khi[i] = 0u;
      klo[i] = 0u;
    }
  }
}

// 32 squared distances (one half of a 64-point tile) -> 32 packed f16x2
// words: w[c] = k1 pair c = f16(k'), w[16 + c] = k2 pair c = f16(k' - k1)
// (lower K index in the low half), k' = 2^14 (1 + u ln2) 2^-u = 2^14 k / sf^2
// in (0, 2^14]: the signal variance is applied to the output, and the 2^14
// lifts k' so that k2 stays a normal fp16 number down to k' ~ 2^-3, i.e.
// k / sf^2 >= 2^-17 (below that its absolute error is < 2^-39 sf^2).  fp16
// keeps 11 significant bits like tf32, so k1 + k2 carries 22 bits.  POLY
// evaluates 2^-u of the odd entries on the FMA pipe (ex2_poly) instead of the
// MUFU.  The squared distance from the tensor core can be a tiny negative
// number for (near-)duplicate points; sqrt(|u^2|) keeps it finite and folds
// the abs into the MUFU operand.  DIAG is a separate instantiation for the
// rare tiles that contain the diagonal, so the common path carries no
// per-entry index compares.
constexpr float kKScale = 16384.f;  // 2^14
template <bool POLY, bool DIAG>
__device__ __forceinline__ void to_k_f16(const uint32_t (&r)[32], uint32_t (&w)[32], int dg) {
  constexpr float ks = kKScale, ka = kKScale * 0.69314718055994531f;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    float k0 = matern_from_u(sqrt_approx(fabsf(__uint_as_float(r[2 * c]))), ks, ka);
    const float ub = sqrt_approx(fabsf(__uint_as_float(r[2 * c + 1])));
    float k1 = POLY ? fmaf(ka, ub, ks) * ex2_poly(-ub) : matern_from_u(ub, ks, ka);
    if (DIAG) {
      if (dg == 2 * c) k0 = 0.f;
      if (dg == 2 * c + 1) k1 = 0.f;
    }
    const __half2 h = __floats2half2_rn(k0, k1);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(k0 - hf.x, k1 - hf.y);
    w[c] = *reinterpret_cast<const uint32_t*>(&h);
    w[16 + c] = *reinterpret_cast<const uint32_t*>(&l);
  }
}

struct TcArgs {
  int64_t m;         // output rows
  int a_row0;        // first A-map row of this launch
  int64_t j0, j1;    // contracted points
  int num_jt;        // J tiles in [j0, j1)
  int splits;
  int chunk;         // tiles per fp32 accumulation chunk
  int s, s_pad;
  int nb, nv;              // B-ring and V-ring stages
  uint32_t vstage_bytes;   // V planes of one tile (2 x s_pad rows of 128 bytes)
  uint32_t a_region;       // shared bytes of A_I (+ the running sum R)
  const int* row_idx;
  int64_t r0;
  const float* V;
  int v_late;  // 1: V itself is written by the split kernel of this launch chain (zero-copy upload)
  int64_t ldv;
  float* out;
  int64_t ldo;
  const float* B;
  int64_t ldb;
  int mode;
  float sf2, a, diag;
  const float* hyp;  // device [sf2, a, diag] (overrides the three above when set)
  const float* vscale;  // H16: per column 2^-e_c, the inverse of the power of two that scaled V's fp16 planes
  float* part;       // [splits][s_pad][m_pad] fp32 split partials (splits > 1)
  int tma_part;      // 1: the final partial tile goes out as one TMA store (mPart)
  double* flush;     // [splits][s_pad][m_pad] fp64 running sums (T > flush_every * chunk)
  int flush_every;   // chunks per fp32 running sum before it is flushed to fp64
  int64_t m_pad;
  const int* done;
  long long* trace;  // WGP_TC_TRACE: per-tile clock64 stamps of CTA 0 ([T][16])
  long long* ctatime;  // WGP_TC_TRACE: per CTA {smid, globaltimer at start, after the tile loop, at exit}
  int nk1;  // packed Gram K steps (TcOperands::nk1), 0: 12 hi / lo MMAs
  int dbg;  // ablation bits (WGP_TC_DEBUG): 1 no epilogue math, 2 no MMA-2, 4 no MMA-1, 8 no V loads,
            // 16 no epilogue TMEM traffic, 32 no B loads, 128 (H16) FMA-pipe ex2 for odd entries
};

// Two K.V precisions share the pipeline:
//   H16 = false (default, WGP_HV_TC): K.V in 3xTF32 (k_hi v_hi + k_hi v_lo +
//     k_lo v_hi, ~2^-21 per product), 32-point J tiles.  TMEM: O0 [0, 96),
//     O1 [96, 192), A_I hi/lo [192, 256) (MMA-1 reads A from TMEM), two
//     128-column groups from 256.  A group serves two tiles: MMA-1 writes
//     S(t) | S(t+1) (64 fp32 columns, one N = 64 instruction per K step: a
//     tf32 MMA costs >= 35 clk whatever its size, so N = 32 ran at half the
//     tensor rate, measured), the epilogue overwrites each S in place with
//     k_hi and writes k_lo 64 columns further.
//   H16 = true (WGP_HV_TC_F16): K.V in fp16x3 (k1 v1 + k1 v2 + k2 v1, 11 + 11
//     significant bits per operand; k' = 2^14 k / sf^2 and V scaled per column
//     by a power of two keep both halves normal -- to_k_f16, split_v_f16_kernel;
//     half the tensor work of 3xTF32), 64-point J tiles.  TMEM (layout 2): O0,
//     O1, A_I hi/lo, four 64-column groups from 256 of one tile each (S: 64
//     fp32 columns, overwritten by the packed k1 | k2 pairs).
// The Gram (MMA-1) is 3xTF32 in both, over 64 points per instruction.
// tf32 TMEM layout (compile-time WGP_TC_LAYOUT): 0 = single O [0, 96), A_I in
// shared memory, three groups from 96; 1 = O0 | O1 [0, 192), A_I in shared
// memory, two groups from 192 (4 tiles in flight, no chunk-drain stall of
// MMA-2); 2 = O0 | O1, A_I in TMEM [192, 256), two groups from 256.
#ifndef WGP_TC_LAYOUT
#define WGP_TC_LAYOUT 2
#endif
constexpr bool kTfSingleO = WGP_TC_LAYOUT == 0;
constexpr bool kTfATmem = WGP_TC_LAYOUT == 2;
constexpr int kTfGroups = kTfSingleO ? 3 : 2;
template <bool H16>
struct Cfg {
  static constexpr int kTJ = H16 ? 64 : 32;        // points per J tile (MMA-2 K, epilogue)
  static constexpr int kP = H16 ? 1 : 2;           // tiles per MMA-1 group
  static constexpr int kN1 = kP * kTJ;            // MMA-1 N = points per B stage (64)
  static constexpr int kGroups = H16 ? (WGP_TC_F16_ATMEM ? 4 : 5) : kTfGroups;  // MMA-1 groups in flight (TMEM)
  static constexpr int kTilesInFlight = kP * kGroups;
  static constexpr uint32_t kGW = H16 ? 64u : 128u;  // TMEM columns per group
  // tf32 layout variant (kTfSingleO): one O accumulator [0, 96) whose chunk
  // drains stall MMA-2, A_I in shared memory (SS Gram), three groups from 96
  // (6 tiles in flight); otherwise O0 | O1, A_I in TMEM, two groups from 256.
  static constexpr bool kATmem = H16 ? (WGP_TC_F16_ATMEM != 0) : kTfATmem;
  static constexpr int kOBufs = (H16 || !kTfSingleO) ? 2 : 1;
  static constexpr uint32_t kOStride = kOBufs == 2 ? 96u : 0u;
  static constexpr uint32_t kAhi = 192, kAlo = 224;  // kATmem only
  static constexpr uint32_t kBufFirst = kATmem ? 256u : (H16 || !kTfSingleO ? 192u : 96u);
  static constexpr uint32_t kBStage = 2u * kN1 * 128u;  // B_hi | B_lo planes
  static constexpr uint32_t kLoOff = 64;                // H16 = false: k_lo column offset
  static __device__ __forceinline__ uint32_t grp_col(int gi) { return kBufFirst + kGW * static_cast<uint32_t>(gi); }
  // TMEM column of tile t's S / k_hi (H16: S / packed k1 | k2)
  static __device__ __forceinline__ uint32_t tile_col(int t) {
    return grp_col((t / kP) % kGroups) + 32u * static_cast<uint32_t>(t % kP);
  }
};

// Warp roles.  The warp scheduler prefers the highest warp id among eligible
// warps, so the latency-critical control warps get the top ids and the 12
// always-eligible epilogue warps (0..11; warp w reads TMEM lanes 32 (w % 4))
// cannot starve them.

// Accumulation precision.  MMA-2 accumulates into fp32 TMEM, and every
// K-step instruction rounds the running sum: with ~3 n / 8 roundings per
// output the error of one long accumulation grows like sqrt(n) 2^-24 |O|
// (measured 1e-5 relative at n = 20000 on dense data, beyond the 1e-5 bar at
// the reference's larger sizes).  The J tiles of a CTA are therefore
// accumulated in chunks of `chunk` tiles (1024 points), alternating between
// O0 and O1; the epilogue warps add each finished chunk into an fp32 running
// sum R in shared memory (row-private, no synchronisation) while MMA-2 fills
// the other accumulator, and every `flush_every` chunks R is moved to a
// CTA-private fp64 sum in global memory.  Error per output: ~sqrt(roundings
// per chunk) + sqrt(flush_every) roundings, independent of n; the
// shared-memory drain costs no L2 traffic (an fp64 global drain per chunk
// measured +20% time).
template <bool H16>
__global__ void __launch_bounds__(kThreadsT<H16>, 1)
    hv_tc_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                 const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                 const __grid_constant__ CUtensorMap mVhi, const __grid_constant__ CUtensorMap mVlo,
                 const __grid_constant__ CUtensorMap mPart, const TcArgs p) {
  using K = Cfg<H16>;
  constexpr int kEpiGroups = kEpiGroupsT<H16>;
  constexpr int kDrainK = (96 + 8 * kEpiGroups - 1) / (8 * kEpiGroups);  // 8-column pieces per group drain
  constexpr int kEpiWarps = 4 * kEpiGroups;
  constexpr int kWarpBProd = kEpiWarps, kWarpM1 = kEpiWarps + 1, kWarpVProd = kEpiWarps + 2, kWarpM2 = kEpiWarps + 3;
  constexpr int NBUF = K::kTilesInFlight;  // kfull ring
  constexpr int TJ = K::kTJ;
  constexpr int P = K::kP;
  if (p.done && *p.done) return;
  // Instrumentation (WGP_TC_TRACE stamps, per-CTA timers, WGP_TC_DEBUG
  // ablations) only in -DWGP_TC_ABLATE builds: the checks cost the
  // latency-critical control warps a few percent.
#ifdef WGP_TC_ABLATE
  long long* const trace = p.trace;
  long long* const ctatime = p.ctatime;
  const int dbg = p.dbg;
#else
  long long* const trace = nullptr;
  long long* const ctatime = nullptr;
  constexpr int dbg = 0;
#endif
  long long gt0 = 0;
  if (ctatime && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // m1done[t % 8]: MMA-1(t) complete (S_t ready; B slot of t free);
  // m2done[t % 8]: MMA-2(t) complete (K buffer and V slot of t free).  One
  // commit per tile and MMA warp: each commit costs ~175 clk of issue in the
  // MMA warp (measured), two per tile bounded the loop.  Ring depth 8 >= every
  // waiter's lag (NB, NV, NBUF <= 8), so no waiter aliases a phase.
  __shared__ __align__(8) uint64_t bar_bfull[kMaxStages], bar_vfull[kMaxStages], bar_m1done[kDoneRing],
      bar_m2done[kDoneRing];
  __shared__ __align__(8) uint64_t bar_a, bar_atm, bar_kfull[NBUF], bar_ofull[2], bar_odrained[2];
  __shared__ uint32_t tmem_slot;
  // bar_turn[w][q]: epilogue warp q of group w may start its tile's math (the
  // previous tile's warp q on the same SMSP is done with the MUFU)
  __shared__ __align__(8) uint64_t bar_turn[kEpiGroups][4];
  // H16: per epilogue warp, 2^-e of the columns [cb, ce) it finishes (cp.async prefetch)
  __shared__ float sColScale[H16 ? kEpiWarps : 1][8 * kDrainK];

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sAhi = smem;
  uint8_t* sAlo = smem + 16384;
  // R: [s_pad][128] fp32 running sum; with A_I in TMEM it reuses
  // A's staging area, which is dead once A has been copied to TMEM.
  float* sR = reinterpret_cast<float*>(K::kATmem ? smem : smem + 32768);
  uint8_t* sB = smem + p.a_region;                            // nb x [B_hi | B_lo]
  uint8_t* sV = sB + static_cast<size_t>(p.nb) * K::kBStage;  // nv x vstage
  // [s_pad][128] fp32: V[g_row, c] of this CTA's rows for the exact diagonal
  // term, prefetched with cp.async at the start (splits == 1 only)
  float* sVd = reinterpret_cast<float*>(sV + static_cast<size_t>(p.nv) * p.vstage_bytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // split-major grid: the CTAs running together share one J range (split),
  // which stays L2-resident while all row tiles pass over it
  const int row_tiles = static_cast<int>(gridDim.x) / p.splits;
  const int rt = blockIdx.x % row_tiles, sp = blockIdx.x / row_tiles;
  const int jt_begin = static_cast<int>(static_cast<int64_t>(p.num_jt) * sp / p.splits);
  const int jt_end = static_cast<int>(static_cast<int64_t>(p.num_jt) * (sp + 1) / p.splits);
  const int T = jt_end - jt_begin;
  const int C = p.chunk;
  const int NB = p.nb, NV = p.nv;
  const int spad = p.s_pad;
  const uint32_t vbox = static_cast<uint32_t>(spad) * 128u;  // one V plane (128-byte rows)

  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&bar_bfull[i], 1);
    for (int i = 0; i < NV; ++i) mbar_init(&bar_vfull[i], 1);
    for (int i = 0; i < kDoneRing; ++i) {
      mbar_init(&bar_m1done[i], 1);
      mbar_init(&bar_m2done[i], 1);
    }
    mbar_init(&bar_a, 1);
    for (int i = 0; i < kEpiGroups * 4; ++i) mbar_init(&bar_turn[i / 4][i % 4], 1);
    mbar_init(&bar_atm, 4);
    // tf32: the V tile of slot b completes on kfull[b] too (NV == NBUF): 4
    // epilogue arrivals + the producer's expect_tx arrival, so MMA-2 checks
    // one barrier per tile (each check costs ~90 clk of its loop, measured)
    for (int i = 0; i < NBUF; ++i) mbar_init(&bar_kfull[i], H16 ? 4 : 5);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_ofull[i], 1);
      mbar_init(&bar_odrained[i], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWarpVProd) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_slot;

  if (warp == kWarpBProd) {
    // ------------------------------------------------------------ TMA producer: A, B ring
    if (T > 0) {  // whole warp, one elected lane issues
      const int arow = p.a_row0 + rt * kTI;
      mbar_expect_tx_warp(&bar_a, 2 * 16384);
      tma_load_2d_warp(sAhi, &mAhi, &bar_a, 0, arow);
      tma_load_2d_warp(sAlo, &mAlo, &bar_a, 0, arow);
      // one stage per MMA-1 group (kN1 = 64 points)
      const int G = (T + P - 1) / P;
      int st = 0;
      for (int gr = 0; gr < G; ++gr, st = (st + 1 == NB) ? 0 : st + 1) {
        if (gr >= NB) mbar_wait(&bar_m1done[(gr - NB) & (kDoneRing - 1)], ((gr - NB) >> 3) & 1);
        uint8_t* base = sB + static_cast<size_t>(st) * K::kBStage;
        if (dbg & 32) {
          mbar_arrive_warp(&bar_bfull[st]);
          continue;
        }
        mbar_expect_tx_warp(&bar_bfull[st], K::kBStage);
        const int pt = static_cast<int>(p.j0) + (jt_begin + gr * P) * TJ;
        tma_load_2d_warp(base, &mBhi, &bar_bfull[st], 0, pt);
        tma_load_2d_warp(base + K::kBStage / 2, &mBlo, &bar_bfull[st], 0, pt);
      }
    }
  } else if (warp == kWarpVProd) {
    // ------------------------------------------------------------ TMA producer: V ring
    // (separate warp so the two rings never block each other); one box of
    // 128-byte rows (32 tf32 / 64 bf16 points) per plane and tile
    if (T > 0) {
      if constexpr (H16) asm volatile("griddepcontrol.wait;" ::: "memory");  // V planes from the split kernel
      // ring slots and phases advance incrementally: runtime divisions by
      // NV / NB / C cost tens of clk each in these single-warp loops
      int st = 0;
      for (int t = 0; t < T; ++t, st = (st + 1 == NV) ? 0 : st + 1) {
        if (t >= NV) mbar_wait(&bar_m2done[(t - NV) & (kDoneRing - 1)], ((t - NV) >> 3) & 1);
        uint8_t* base = sV + static_cast<size_t>(st) * p.vstage_bytes;
        const int vp = (jt_begin + t) * TJ;
        uint64_t* vbar = H16 ? &bar_vfull[st] : &bar_kfull[st];  // tf32: st == t % NBUF
        if (dbg & 8) {
          mbar_arrive_warp(vbar);
          continue;
        }
        mbar_expect_tx_warp(vbar, p.vstage_bytes);
        tma_load_2d_warp(base, &mVhi, vbar, vp, 0);
        tma_load_2d_warp(base + vbox, &mVlo, vbar, vp, 0);
      }
    }
  } else if (warp == kWarpM1) {
    // ------------------------------------------------------------ MMA-1 issuer
    // Two issuing warps: tcgen05.mma issue blocks while the tensor pipe is
    // busy (queue depth ~1, measured), so one warp's barrier waits and
    // commits would idle the pipe.  This warp issues MMA-1 (Gram, 3xTF32) and
    // kWarpM2 MMA-2 (K.V); each one's waits overlap the other's MMAs.
    // MMA-1(t) reuses buffer t % NBUF only after MMA-2(t - NBUF) committed
    // m2done.  The whole warp runs the loop (uniform operands); elect.sync
    // picks the issuing lane.
    if (T > 0) {
      constexpr uint32_t id1 = idesc_tf32(kTI, K::kN1);
      if constexpr (!K::kATmem) {
        mbar_wait(&bar_a, 0);
      } else {
        mbar_wait(&bar_atm, 0);  // A_I copied into TMEM by epilogue group 0
      }
      tc_after();
      const uint64_t dAhi = umma_desc(sAhi), dAlo = umma_desc(sAlo);
      const int G = (T + P - 1) / P;
      int st = 0, gi = 0;
      uint32_t bph = 0;
      for (int gr = 0; gr < G; ++gr) {
        const int t = gr * P;  // first tile of the group (trace index)
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 6] = clock64();
        // the group's columns are free once MMA-2 read the last tile of group gr - kGroups
        if (gr >= K::kGroups) {
          const int u = (gr - K::kGroups) * P + P - 1;
          mbar_wait(&bar_m2done[u & (kDoneRing - 1)], (u >> 3) & 1);
        }
        mbar_wait(&bar_bfull[st], bph);
        tc_after();
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 7] = clock64();
        uint8_t* base = sB + static_cast<size_t>(st) * K::kBStage;
        const uint64_t dBhi = umma_desc(base), dBlo = umma_desc(base + K::kBStage / 2);
        const uint32_t d = tmem + K::grp_col(gi);
        if (!(dbg & 4)) {
          if constexpr (!K::kATmem) {
            if (p.nk1)
              mma1_packed_tf32(d, dAhi, dAlo, dBhi, dBlo, id1, p.nk1);
            else
              mma1_group_tf32(d, dAhi, dAlo, dBhi, dBlo, id1);
          } else {
            static_assert(K::kAlo == K::kAhi + 32, "packed Gram: A K columns contiguous in TMEM");
            if (p.nk1)
              mma1_packed_tf32_ts(d, tmem + K::kAhi, dBhi, dBlo, id1, p.nk1);
            else
              mma1_group_tf32_ts(d, tmem + K::kAhi, tmem + K::kAlo, dBhi, dBlo, id1);
          }
        }
        mma_commit(&bar_m1done[gr & (kDoneRing - 1)]);
        if (gr == 0 && ctatime && lane == 0) {
          long long gt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          ctatime[blockIdx.x * 12 + 11] = gt;  // first Gram group issued
        }
        if (trace && blockIdx.x == 0 && lane == 0)
          for (int h = 0; h < P; ++h) trace[(t + h) * 16 + 0] = clock64();
        if (++st == NB) st = 0, bph ^= 1u;
        if (++gi == K::kGroups) gi = 0;
      }
    }
  } else if (warp == kWarpM2) {
    // ------------------------------------------------------------ MMA-2 issuer
    if (T > 0) {
      const uint32_t id2 = H16 ? idesc_f16(kTI, spad) : idesc_tf32(kTI, spad);
      const uint64_t box = vbox >> 4;
      int b = 0, st = 0, c = 0, tc = 0;
      uint32_t kph = 0, vph = 0;
      for (int t = 0; t < T; ++t) {
        const uint32_t o = tmem + static_cast<uint32_t>(c & 1) * K::kOStride;
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 4] = clock64();
        // chunk c reuses its accumulator once the epilogue drained chunk c - kOBufs
        if (tc == 0 && c >= K::kOBufs) {
          const int cp = c - K::kOBufs;
          mbar_wait(&bar_odrained[cp & 1], (cp >> 1) & 1);
        }
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 12] = clock64();
        if (H16) mbar_wait(&bar_vfull[st], vph);
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 13] = clock64();
        mbar_wait(&bar_kfull[b], kph);
        tc_after();
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 3] = clock64();
        uint8_t* base = sV + static_cast<size_t>(st) * p.vstage_bytes;
        const uint32_t kb = tmem + K::tile_col(t);
        const uint64_t dv = umma_desc(base);
        if (dbg & 2) {  // (ablation: no K.V)
        } else if constexpr (H16) {
          // per 32-point half h: k1 pairs in columns [32h, 32h+16), k2 in
          // [32h+16, 32h+32); 12 MMAs from one asm block
          mma2_tile_f16(o, kb, dv, dv + box, id2, tc > 0 ? 1u : 0u);
        } else {
          static_assert(H16 || K::kLoOff == 64, "mma2_tile_tf32 assumes k_lo 64 columns after k_hi");
          mma2_tile_tf32(o, kb, dv, dv + box, id2, tc > 0 ? 1u : 0u);
        }
        if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 5] = clock64();
        if (t == 0 && ctatime && lane == 0) {
          long long gt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          ctatime[blockIdx.x * 12 + 10] = gt;  // first MMA-2 issued
        }
        mma_commit(&bar_m2done[t & (kDoneRing - 1)]);
        if (tc == C - 1 || t == T - 1) mma_commit(&bar_ofull[c & 1]);
        if (t == T - 1 && ctatime && lane == 0) {
          long long gt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          ctatime[blockIdx.x * 12 + 6] = gt;  // last MMA-2 issued
        }
        if (++st == NV) st = 0, vph ^= 1u;
        if (++b == NBUF) b = 0, kph ^= 1u;
        if (++tc == C) tc = 0, ++c;
      }
    }
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    // Warpgroup w handles tiles t = w, w+3, ...; warp w%4
    // of the group reads TMEM lanes 32 (w%4) .. +31 (= its 32 output rows).
    const int ew = warp, q = ew & 3, w = ew >> 2;
    const int row = q * 32 + lane;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int64_t lr = static_cast<int64_t>(rt) * kTI + row;
    const bool valid = lr < p.m;
    int64_t g = -1;
    if (valid) g = p.row_idx ? static_cast<int64_t>(p.row_idx[lr]) : p.r0 + lr;
    const float sf2 = p.hyp ? p.hyp[0] : p.sf2, ac = p.hyp ? p.hyp[1] : p.a;
    const float hdiag = p.hyp ? p.hyp[2] : p.diag;
    const bool nomath = dbg & 1;
    const int nch = (T + C - 1) / C;
    const bool diag = g >= p.j0 && g < p.j1;
    if (K::kATmem && w == 0 && T > 0) {
      // Copy this row of A_I (hi, lo: 32 fp32 each) from the 128B-swizzled
      // TMA tile into TMEM: MMA-1 then reads A from TMEM (with A in shared
      // memory MMA-1 is smem-bandwidth bound, 48 clk per MMA, measured).
      mbar_wait(&bar_a, 0);
      uint32_t ah[32], al[32];
      const uint8_t* rh = sAhi + (row >> 3) * 1024 + (row & 7) * 128;
      const uint8_t* rl = sAlo + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int pc = (c ^ (row & 7)) * 16;
        const uint4 vh = *reinterpret_cast<const uint4*>(rh + pc);
        const uint4 vl = *reinterpret_cast<const uint4*>(rl + pc);
        ah[4 * c] = vh.x, ah[4 * c + 1] = vh.y, ah[4 * c + 2] = vh.z, ah[4 * c + 3] = vh.w;
        al[4 * c] = vl.x, al[4 * c + 1] = vl.y, al[4 * c + 2] = vl.z, al[4 * c + 3] = vl.w;
      }
      __syncwarp();
      tmem_st32(tmem + lanes + K::kAhi, ah);
      tmem_st32(tmem + lanes + K::kAlo, al);
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_atm);
    }
    // Drain chunk c: R (+)= O[c & 1] over this group's columns; every
    // flush_every chunks R moves into the fp64
    // global sum F.  The accumulator is released to MMA-2 as soon as it has
    // been read.  The last chunk finishes the row: the exact diagonal term and
    // the output mode, or the fp32 partial when the J tiles are split across
    // CTAs.
    double* F = p.flush + static_cast<int64_t>(sp) * spad * p.m_pad + lr;  // column c at F[c * m_pad]
    float* R = sR + row;                                                   // column c at R[c * 128]
    const int FE = p.flush_every;
    float* Vd = sVd + row;  // column c at Vd[c * 128]
    // Group w owns the contiguous column block [cb, ce) (<= 32 columns,
    // multiples of 8): one TMEM round trip per drain.
    const int cpg = ((spad + kEpiGroups * 8 - 1) / (kEpiGroups * 8)) * 8;
    const int cb = min(spad, w * cpg), ce = min(spad, (w + 1) * cpg);
    // Intermediate chunk c: R (+)= O[c & 1] (every flush_every chunks R moves
    // into the fp64 sum F instead); O[c & 1] is released to MMA-2 once read.
    auto drain = [&](int c) {
      mbar_wait(&bar_ofull[c & 1], (c >> 1) & 1);
      tc_after();
      const uint32_t ocol = static_cast<uint32_t>(c & 1) * K::kOStride;
      const bool fresh = c % FE == 0;  // R starts over with this chunk
      const bool flush = (c + 1) % FE == 0;
      uint32_t o[kDrainK][8];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kDrainK; ++k)
        if (cb + 8 * k < ce) tmem_ld8(tmem + lanes + ocol + cb + 8 * k, o[k]);
      tmem_wait_ld();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_odrained[c & 1]);
#pragma unroll
      for (int k = 0; k < kDrainK; ++k) {
        if (cb + 8 * k >= ce) break;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int col = cb + 8 * k + i;
          const float r = (fresh ? 0.f : R[col * 128]) + __uint_as_float(o[k][i]);
          if (!flush) {
            R[col * 128] = r;
          } else if (valid && col < p.s) {
            double* f = F + static_cast<int64_t>(col) * p.m_pad;
            *f = (c + 1 == FE ? 0.0 : *f) + static_cast<double>(r);
          }
        }
      }
    };
    // Last chunk c: this row's outputs -- the exact diagonal term and the
    // output mode, or the fp32 partial when the J tiles are split across CTAs.
    // Kept compact and free of dependent global loads on the common path: it
    // runs once per CTA from a cold instruction cache, and an unrolled version
    // with per-column global loads cost 8-12 us per CTA (measured).  The
    // diagonal's V entries come from sVd (cp.async prefetch at the start).
    auto finish = [&](int c) {
      mbar_wait(&bar_ofull[c & 1], (c >> 1) & 1);
      tc_after();
      if (ctatime && threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        ctatime[blockIdx.x * 12 + 4] = gt;  // last ofull observed
      }
      const uint32_t ocol = static_cast<uint32_t>(c & 1) * K::kOStride;
      const bool fresh = c % FE == 0;
      uint32_t o[kDrainK][8];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kDrainK; ++k)
        if (cb + 8 * k < ce) tmem_ld8(tmem + lanes + ocol + cb + 8 * k, o[k]);
      tmem_wait_ld();
      if (ctatime && threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        ctatime[blockIdx.x * 12 + 7] = gt;  // last accumulator read
      }
      // split partial as one TMA store of R (all 384 epilogue threads fold
      // their rows first; rows past m land in the padding rows of `part`)
      const bool tma_out = p.tma_part && c < FE;
      // H16: O carries sf^2-free k' = 2^14 k / sf^2 times V 2^e_c (to_k_f16, split_v_f16_kernel)
      float osc = 1.f;
      if constexpr (H16) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();  // (before any lane leaves: the column scales come from the whole warp)
        osc = sf2 * (1.f / kKScale);
      }
      if (!valid && !tma_out) return;
      auto colsc = [&](int col) { return H16 ? osc * sColScale[warp][col - cb] : 1.f; };
      // Fold the accumulator into R (one short unrolled block), then a rolled
      // loop over the row's columns: this code runs once per CTA from a cold
      // instruction cache, so its length, not its arithmetic, sets its time
      // (measured: ~4 us for the fully unrolled form, ~40 clk per instruction).
#pragma unroll
      for (int k = 0; k < kDrainK; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int col = cb + 8 * k + i;
          if (col < ce) {
            const float r = (fresh ? 0.f : R[col * 128]) + __uint_as_float(o[k][i]);
            R[col * 128] = (H16 && tma_out) ? r * colsc(col) : r;
          }
        }
      if (ctatime && threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        ctatime[blockIdx.x * 12 + 8] = gt;  // folded into R
      }
      if (tma_out) {
        // 27 coalesced column stores per thread cost ~3 us per CTA, 4% of the
        // kernel (measured, WGP_TC_DEBUG 256); one bulk tensor store of the
        // [s_pad][128] tile replaces them.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (warp == 0 && lane == 0) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&mPart),
                       "r"(rt * kTI), "r"(sp * spad), "r"(smem_u32(sR))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // sR is read before the CTA exits
        }
        return;
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      if (ctatime && threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        ctatime[blockIdx.x * 12 + 9] = gt;  // prefetch complete
      }
      const int cend = min(ce, dbg & 256 ? cb : p.s);  // dbg 256: no final stores (ablation)
      if (p.splits > 1) {
        float* part = p.part + static_cast<int64_t>(sp) * spad * p.m_pad + lr;
#pragma unroll 1
        for (int col = cb; col < cend; ++col) {
          float r = R[col * 128];
          if (c >= FE) r = static_cast<float>(__ldcg(F + static_cast<int64_t>(col) * p.m_pad) + static_cast<double>(r));
          if (H16) r *= colsc(col);
          part[static_cast<int64_t>(col) * p.m_pad] = r;
        }
        return;
      }
      const float dscale = diag ? hdiag : 0.f;
#pragma unroll 1
      for (int col = cb; col < cend; ++col) {
        float r = R[col * 128];
        if (c >= FE) r = static_cast<float>(__ldcg(F + static_cast<int64_t>(col) * p.m_pad) + static_cast<double>(r));
        if (H16) r *= colsc(col);
        r = fmaf(dscale, diag ? Vd[col * 128] : 0.f, r);
        float* dst = p.out + lr + static_cast<int64_t>(col) * p.ldo;
        if (p.mode == kHvStore)
          *dst = r;
        else if (p.mode == kHvResidual)
          *dst = p.B[g + static_cast<int64_t>(col) * p.ldb] - r;
        else
          *dst -= r;
      }
    };
    // prefetch the diagonal's V entries (overlaps the whole tile loop)
    if constexpr (H16) {
      if (p.v_late) asm volatile("griddepcontrol.wait;" ::: "memory");  // V comes from the split kernel too
    }
    if (valid && diag && p.splits == 1) {
      for (int col = cb; col < ce && col < p.s; ++col)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(Vd + col * 128)),
                     "l"(p.V + g + static_cast<int64_t>(col) * p.ldv)
                     : "memory");
    }
    if constexpr (H16) {
      // (programmatic dependent launch: the column scales come from the split
      // kernel still running when this grid starts)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int c = cb + lane; c < ce; c += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&sColScale[warp][c - cb])),
                     "l"(p.vscale + c)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // Chunk dc is drained `lag` tiles after it ended, so its last MMA-2 has
    // retired by then; every group still drains it before MMA-2 reaches
    // chunk dc + 2 (lag + 2 <= C), so MMA-2 never waits for a drain.
    // (single O: drained as soon as possible, MMA-2 waits for it)
    const int lag = K::kOBufs == 1 ? 0 : max(2, C / 2);
    int dc = 0;  // next chunk to drain
    const bool turns = dbg & 512;
    uint32_t turn_ph = 0;
    for (int t = w; t < T; t += kEpiGroups) {
      while (dc < nch - 1 && t >= (dc + 1) * C + lag) drain(dc++);
      const int b = t % NBUF;
      const uint32_t bcol = K::tile_col(t);
      const int gr = t / P;
      const int64_t tstart = p.j0 + static_cast<int64_t>(jt_begin + t) * TJ;
      const int64_t dg = valid ? g - tstart : -1;
      const bool diag_tile = __any_sync(0xffffffffu, dg >= 0 && dg < TJ);
      mbar_wait(&bar_m1done[gr & (kDoneRing - 1)], (gr >> 3) & 1);
      tc_after();
      if (trace && blockIdx.x == 0 && q == 0 && lane == 0) trace[t * 16 + 1] = clock64();
      const int dgi = static_cast<int>(dg < 0 || dg >= TJ ? -1 : dg);
      if (!(dbg & 16)) {
        if constexpr (H16) {
          // each 32-column half of S is read, converted and overwritten in
          // place by [k1 pairs (16 cols) | k2 pairs (16 cols)]; the second
          // half's load is issued before the first half's stores, and only
          // one half's values are live at a time (the 128-register epilogue
          // spilled with both)
          uint32_t r[32], wds[32];
          __syncwarp();
          tmem_ld32(tmem + lanes + bcol, r);
          tmem_wait_ld();
          if (turns && t > 0) {
            mbar_wait(&bar_turn[w][q], turn_ph & 1);
            ++turn_ph;
          }
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            const int dh = dgi - 32 * half;
            if (nomath) {
#pragma unroll
              for (int i = 0; i < 32; ++i) wds[i] = r[i];
            } else if (diag_tile) {
              to_k_f16<false, true>(r, wds, dh);
            } else if (dbg & 128) {
              to_k_f16<true, false>(r, wds, dh);
            } else {
              to_k_f16<false, false>(r, wds, dh);
            }
            __syncwarp();
            if (half == 0) tmem_ld32(tmem + lanes + bcol + 32, r);
            tmem_st32(tmem + lanes + bcol + 32 * half, wds);
            if (half == 0) tmem_wait_ld();
          }
          if (turns && lane == 0 && t + 1 < T) mbar_arrive(&bar_turn[w == kEpiGroups - 1 ? 0 : w + 1][q]);
        } else {
          // S (32 columns) -> k_hi in place, k_lo kLoOff columns further
          uint32_t r[32], khi[32], klo[32];
          __syncwarp();
          tmem_ld32(tmem + lanes + bcol, r);
          tmem_wait_ld();
          if (turns && t > 0) {
            mbar_wait(&bar_turn[w][q], turn_ph & 1);
            ++turn_ph;
          }
          if (nomath) {
#pragma unroll
            for (int i = 0; i < 32; ++i) khi[i] = r[i], klo[i] = 0u;
          } else if (diag_tile) {
            to_k<true>(r, khi, klo, sf2, ac, dgi);
          } else {
            to_k<false>(r, khi, klo, sf2, ac, dgi);
          }
          if (turns && t + 1 < T) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_turn[w == kEpiGroups - 1 ? 0 : w + 1][q]);
          }
          __syncwarp();
          tmem_st32(tmem + lanes + bcol, khi);
          tmem_st32(tmem + lanes + bcol + K::kLoOff, klo);
        }
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_kfull[b]);
      if (trace && blockIdx.x == 0 && q == 0 && lane == 0) trace[t * 16 + 2] = clock64();
      if (trace && blockIdx.x == 0 && lane == 0) trace[t * 16 + 8 + q] = clock64();
    }
    if (ctatime && threadIdx.x == 0) {
      long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      ctatime[blockIdx.x * 12 + 2] = gt;  // epilogue tile loop done (before the last drain)
    }
    while (dc < nch - 1) drain(dc++);
    if (nch > 0) {
      finish(dc++);
      if (ctatime && threadIdx.x == 0) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        ctatime[blockIdx.x * 12 + 5] = gt;  // final drain done
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (ctatime && threadIdx.x == 0) {
    uint32_t smid;
    long long gt;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    ctatime[blockIdx.x * 12 + 0] = smid;
    ctatime[blockIdx.x * 12 + 1] = gt0;
    ctatime[blockIdx.x * 12 + 3] = gt;
  }
  if (warp == kWarpVProd) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Sum of the split partials (in fp64, fixed order) + the kernel's row epilogue.
__global__ void tc_reduce_kernel(const TcArgs p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (launched programmatically after the H.V grid)
  if (p.done && *p.done) return;
  const int64_t lr = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (lr >= p.m) return;
  // the split partials' loads are issued together (a serial loop waited one
  // L2 round trip per split); summed in split order as before
  const float* src = p.part + static_cast<int64_t>(c) * p.m_pad + lr;
  const int64_t sstride = static_cast<int64_t>(p.s_pad) * p.m_pad;
  double acc = 0.0;
  int sp = 0;
  for (; sp + 4 <= p.splits; sp += 4) {
    float x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = __ldcg(src + (sp + i) * sstride);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc += static_cast<double>(x[i]);
  }
  for (; sp < p.splits; ++sp) acc += static_cast<double>(__ldcg(src + sp * sstride));
  float v = static_cast<float>(acc);
  const int64_t g = p.row_idx ? static_cast<int64_t>(p.row_idx[lr]) : p.r0 + lr;
  if (g >= p.j0 && g < p.j1) v = fmaf(p.hyp ? p.hyp[2] : p.diag, p.V[g + c * p.ldv], v);
  float* dst = p.out + lr + c * p.ldo;
  if (p.mode == kHvStore)
    *dst = v;
  else if (p.mode == kHvResidual)
    *dst = p.B[g + c * p.ldb] - v;
  else
    *dst -= v;
}

// V[j0:j1, :s] -> tf32 hi / lo planes [s][ldw] (point index j - j0).
// src / copy (optional): read V from src (the caller's page-locked host buffer) and keep
// a copy in `copy` (the device V the H.V kernel's diagonal term reads).
__global__ void split_v_kernel(const float* V, int64_t ldv, int64_t j0, int64_t nv, float* hi, float* lo,
                               int64_t ldw, const float* src, float* copy) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (j >= nv) return;
  const float v = (src ? src : V)[j0 + j + c * ldv];
  if (copy) copy[j0 + j + c * ldv] = v;
  const float vh = __uint_as_float(__float_as_uint(v) & kTfMask);
  hi[c * ldw + j] = vh;
  lo[c * ldw + j] = v - vh;
}

// Power of two 2^e_c putting the column max into [2^14, 2^15): the fp16 planes
// of the scaled column are then normal down to 2^-28 of its max (hi) and the
// lo residual down to 2^-17 of it; below, their absolute error is < 2^-39 of
// the max.  Zero and non-finite columns keep e = 0 (NaN / Inf propagate).
__device__ __forceinline__ float col_scale(unsigned mbits) {
  const int E = static_cast<int>(mbits >> 23);
  int e = 0;
  if (E == 0 && mbits) e = 100;
  else if (E > 0 && E < 255) e = min(100, max(-100, 141 - E));
  return __int_as_float((127 + e) << 23);
}

// V[j0:j1, :s] -> fp16 planes v1 = f16(2^e_c v), v2 = f16(2^e_c v - v1)
// [s][ldw] and vscale[c] = 2^-e_c (exact: |e_c| <= 100).  One cluster of
// kSplitCl CTAs per column, each CTA a contiguous slice of its rows: the
// slice's max |v| (float bits are monotone in |v|, NaN sorts above every
// finite value), the column max over the cluster through distributed shared
// memory, then the planes -- one launch; the slice stays in registers when
// it fits (kSplitKeep values per thread), otherwise it is re-read.  (One CTA
// per column walking the column serially: 8.8 us at config 1, ncu.)
constexpr int kSplitCl = 8, kSplitThreads = 256, kSplitKeep = 8;
__global__ void __cluster_dims__(kSplitCl, 1, 1) __launch_bounds__(kSplitThreads)
    split_v_f16_kernel(const float* V, int64_t ldv, int64_t j0, int64_t nv, __half* v1, __half* v2, int64_t ldw,
                       float* vscale, const float* src, float* copy) {
  // the H.V grid may start its fill (A / B loads, Gram, K conversion) now;
  // it waits for this grid before touching V's planes and scales
  asm volatile("griddepcontrol.launch_dependents;");
  const int c = blockIdx.y;
  const uint32_t rank = cluster_ctarank();
  const int64_t b0 = nv * rank / kSplitCl, b1 = nv * (rank + 1) / kSplitCl;
  // src / copy as in split_v_kernel: the first pass reads the host buffer once (every
  // load of the grid in flight at once) and stores the device copy
  const float* col = (src ? src : V) + j0 + static_cast<int64_t>(c) * ldv;
  float* ccol = copy ? copy + j0 + static_cast<int64_t>(c) * ldv : nullptr;
  const bool keep = b1 - b0 <= static_cast<int64_t>(kSplitKeep) * kSplitThreads;
  float x[kSplitKeep];
  unsigned m = 0u;
  if (keep) {
#pragma unroll
    for (int i = 0; i < kSplitKeep; ++i) {
      const int64_t j = b0 + threadIdx.x + static_cast<int64_t>(i) * kSplitThreads;
      x[i] = j < b1 ? col[j] : 0.f;
    }
    if (ccol) {
#pragma unroll
      for (int i = 0; i < kSplitKeep; ++i) {
        const int64_t j = b0 + threadIdx.x + static_cast<int64_t>(i) * kSplitThreads;
        if (j < b1) ccol[j] = x[i];
      }
    }
#pragma unroll
    for (int i = 0; i < kSplitKeep; ++i) m = max(m, __float_as_uint(x[i]) & 0x7FFFFFFFu);
  } else {
    for (int64_t j = b0 + threadIdx.x; j < b1; j += kSplitThreads * kSplitKeep) {
#pragma unroll
      for (int i = 0; i < kSplitKeep; ++i) {
        const int64_t jj = j + static_cast<int64_t>(i) * kSplitThreads;
        x[i] = jj < b1 ? col[jj] : 0.f;
        if (ccol && jj < b1) ccol[jj] = x[i];
      }
#pragma unroll
      for (int i = 0; i < kSplitKeep; ++i) m = max(m, __float_as_uint(x[i]) & 0x7FFFFFFFu);
    }
    if (ccol) col = ccol;  // the second pass re-reads this thread's own device copies
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ unsigned sm[kSplitThreads / 32];
  __shared__ unsigned scta;
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0u;
#pragma unroll
    for (int w = 0; w < kSplitThreads / 32; ++w) t = max(t, sm[w]);
    scta = t;
  }
  cluster_sync_all();  // every CTA's slice max is visible to the cluster
  unsigned mc = 0u;
#pragma unroll
  for (int r = 0; r < kSplitCl; ++r) mc = max(mc, ld_shared_cluster_u32(&scta, static_cast<uint32_t>(r)));
  const float sc = col_scale(mc);
  if (rank == 0 && threadIdx.x == 0) vscale[c] = 1.f / sc;
  __half* h1 = v1 + static_cast<int64_t>(c) * ldw;
  __half* h2 = v2 + static_cast<int64_t>(c) * ldw;
  auto put = [&](int64_t j, float xv) {
    const float v = xv * sc;
    const __half h = __float2half_rn(v);
    h1[j] = h;
    h2[j] = __float2half_rn(v - __half2float(h));
  };
  if (keep) {
#pragma unroll
    for (int i = 0; i < kSplitKeep; ++i) {
      const int64_t j = b0 + threadIdx.x + static_cast<int64_t>(i) * kSplitThreads;
      if (j < b1) put(j, x[i]);
    }
  } else {  // re-read, kSplitKeep loads in flight per thread (a serial loop: 58 us per AP block at config 3)
    for (int64_t j = b0 + threadIdx.x; j < b1; j += kSplitThreads * kSplitKeep) {
#pragma unroll
      for (int i = 0; i < kSplitKeep; ++i) {
        const int64_t jj = j + static_cast<int64_t>(i) * kSplitThreads;
        x[i] = jj < b1 ? col[jj] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < kSplitKeep; ++i) {
        const int64_t jj = j + static_cast<int64_t>(i) * kSplitThreads;
        if (jj < b1) put(jj, x[i]);
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still read its scta
}

__global__ void build_ops_kernel(const float* xs, int64_t n, int64_t n_pad, int dp, int d, bool packed, float* ahi,
                                 float* alo, float* bhi, float* blo) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  float a[kKA], b[kKA];
#pragma unroll
  for (int k = 0; k < kKA; ++k) a[k] = b[k] = 0.f;
  if (i < n) {
    double sq = 0.0;
    for (int k = 0; k < d; ++k) {
      const float x = xs[i * dp + k];
      sq += static_cast<double>(x) * x;
    }
    for (int k = 0; k < kKA; ++k) {
      if (k < d) {
        a[k] = xs[i * dp + k];
        b[k] = -2.f * xs[i * dp + k];
      }
    }
    a[d] = static_cast<float>(sq);
    a[d + 1] = 1.f;
    b[d] = 1.f;
    b[d + 1] = static_cast<float>(sq);
  }
  if (!packed) {
#pragma unroll
    for (int k = 0; k < kKA; ++k) {
      const float ah = __uint_as_float(__float_as_uint(a[k]) & kTfMask);
      const float bh = __uint_as_float(__float_as_uint(b[k]) & kTfMask);
      ahi[i * kKA + k] = ah;
      alo[i * kKA + k] = a[k] - ah;
      bhi[i * kKA + k] = bh;
      blo[i * kKA + k] = b[k] - bh;
    }
    return;
  }
  // packed (TcOperands::nk1): [a_hi | a_hi | a_lo] . [b_hi | b_lo | b_hi]
  const int w = d + 2;
  for (int k = 0; k < 2 * kKA; ++k) {
    const int seg = k / w, e = k - seg * w;
    float av = 0.f, bv = 0.f;
    if (seg < 3) {
      const float ah = __uint_as_float(__float_as_uint(a[e]) & kTfMask);
      const float bh = __uint_as_float(__float_as_uint(b[e]) & kTfMask);
      av = seg < 2 ? ah : a[e] - ah;
      bv = seg == 1 ? b[e] - bh : bh;
    }
    float* pa = k < kKA ? ahi : alo;
    float* pb = k < kKA ? bhi : blo;
    pa[i * kKA + (k & (kKA - 1))] = av;
    pb[i * kKA + (k & (kKA - 1))] = bv;
  }
}

__global__ void gather_rows_kernel(const float* ahi, const float* alo, const int* idx, int64_t m,
                                   float* ghi, float* glo, int64_t m_pad) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m_pad * kKA) return;
  const int64_t r = e / kKA, k = e % kKA;
  float h = 0.f, l = 0.f;
  if (r < m) {
    const int64_t g = idx[r];
    h = ahi[g * kKA + k];
    l = alo[g * kKA + k];
  }
  ghi[e] = h;
  glo[e] = l;
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  if (!fn) throw DeviceError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                     uint32_t box_out, CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_in, box_out};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(&m, dtype, 2, const_cast<void*>(base), dims, strides,
                                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

// J-split count: waves x (tiles per CTA + a fixed per-CTA cost of ~16 tile
// times for the pipeline fill, the final drain and the CTA turnover,
// measured), plus the split-reduction pass.
// min_sp: the smallest split count whose J range fits the L2 budget (below).
int choose_splits(int64_t row_tiles, int jt, int sms, int min_sp = 1) {
  constexpr double kCtaOverheadTiles = 16.0;
  int best = 1;
  double best_cost = 1e300;
  for (int sp = 1; sp <= 64; ++sp) {
    if (sp > 1 && jt / sp < 8) break;
    if (sp < min_sp) continue;
    const double waves = std::ceil(static_cast<double>(row_tiles * sp) / sms);
    const double cost = waves * (std::ceil(static_cast<double>(jt) / sp) + kCtaOverheadTiles) +
                        (sp > 1 ? 4.0 + 0.5 * sp : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

}  // namespace

struct Workspace {
  void* p = nullptr;
  size_t bytes = 0;
  void* ensure(size_t b) {
    if (b > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      WGP_CUDA(cudaMalloc(&p, b));
      bytes = b;
      alloc_generation().fetch_add(1);
    }
    return p;
  }
  ~Workspace() {
    if (p) cudaFree(p);
  }
};

struct TcWorkspaces {
  Workspace v, rows, part;
};

namespace {

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

TcOperands::~TcOperands() {
  int k = 0;
  profile_ms(&k);
  if (a_hi) cudaFree(a_hi);
  delete ws;
}

double TcOperands::profile_ms(int* launches) {
  double ms = 0.0;
  for (auto& e : events) {
    float t = 0.f;
    if (cudaEventSynchronize(e.second) == cudaSuccess && cudaEventElapsedTime(&t, e.first, e.second) == cudaSuccess)
      ms += t;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  if (launches) *launches = static_cast<int>(events.size());
  events.clear();
  return ms;
}

void TcOperands::build(const float* xs, int64_t n_, int dp, int d_, cudaStream_t st) {
  n = n_;
  d = d_;
  n_pad = round_up(n, 128);
  const size_t plane = sizeof(float) * n_pad * kKA;
  if (4 * plane > bytes) {
    if (a_hi) cudaFree(a_hi);
    a_hi = nullptr;
    WGP_CUDA(cudaMalloc(&a_hi, 4 * plane));
    bytes = 4 * plane;
  }
  a_lo = static_cast<char*>(a_hi) + plane;
  b_hi = static_cast<char*>(a_hi) + 2 * plane;
  b_lo = static_cast<char*>(a_hi) + 3 * plane;
  static const bool no_pack = getenv("WGP_TC_NOPACK") != nullptr;  // A/B switch
  nk1 = (!no_pack && 3 * (d + 2) <= 2 * kKA) ? static_cast<int>(ceil_div(3 * (d + 2), 8)) : 0;
  build_ops_kernel<<<static_cast<unsigned>(ceil_div(n_pad, 128)), 128, 0, st>>>(
      xs, n, n_pad, dp, d, nk1 > 0, static_cast<float*>(a_hi), static_cast<float*>(a_lo), static_cast<float*>(b_hi),
      static_cast<float*>(b_lo));
  WGP_LAUNCH_CHECK();
  valid = true;
}

// Programmatic dependent launch (the fp16 engine): the H.V grid starts while
// split_v_f16 runs (its fill overlaps the split), the reduction as soon as the
// H.V grid ends.  WGP_TC_NO_PDL=1: ordinary stream order (A/B).
bool tc_pdl() {
  static const bool off = getenv("WGP_TC_NO_PDL") != nullptr;
  return !off;
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, int smem, cudaStream_t st, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  WGP_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <bool H16>
void launch_tc(const CUtensorMap& mAhi, const CUtensorMap& mAlo, const CUtensorMap& mBhi, const CUtensorMap& mBlo,
               const CUtensorMap& mPart,
               const CUtensorMap& mVhi, const CUtensorMap& mVlo, const TcArgs& a, unsigned grid, int smem,
               cudaStream_t st, bool pdl) {
  WGP_SMEM_ATTR(hv_tc_kernel<H16>, kSmemLimit);
  launch_pdl(hv_tc_kernel<H16>, dim3(grid), dim3(kThreadsT<H16>), smem, st, pdl, mAhi, mAlo, mBhi, mBlo, mVhi, mVlo,
             mPart, a);
  WGP_LAUNCH_CHECK();
}

CUtensorMap tc_tensor_map(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_in,
                          uint32_t box_out) {
  return make_map(base, inner, outer, row_bytes, box_in, box_out);
}
int tc_sm_count() { return sm_count(); }

bool hv_tc_supported(int d, int s) { return d + 2 <= kKA && s >= 1 && s <= 128; }

// choose_splits' cost model of one launch over m rows and nv points, in
// J-tile units of one CTA (wgp_hv picks its row chunks with it; the L2 split
// floor as in hv_tc, partial cap left out)
double hv_tc_model_cost(int64_t m, int64_t nv, int s, bool f16) {
  const int TJ = f16 ? Cfg<true>::kTJ : Cfg<false>::kTJ;
  const int jt = static_cast<int>(ceil_div(nv, TJ));
  const int64_t rt = ceil_div(m, kTI);
  const double spad = static_cast<double>(round_up(s, 16));
  const int min_sp = std::max(1, std::min(64, static_cast<int>(std::ceil(static_cast<double>(nv) *
                                                                        (256.0 + 2.0 * (f16 ? 2 : 4) * spad) / 48e6))));
  const int sp = choose_splits(rt, jt, sm_count(), min_sp);
  return std::ceil(static_cast<double>(rt * sp) / sm_count()) * (std::ceil(static_cast<double>(jt) / sp) + 16.0) +
         (sp > 1 ? 4.0 + 0.5 * sp : 0.0);
}

// WGP_TC_TRACE report: per-tile stamps of CTA 0 (T0 steady-state tiles) and per-CTA timers.
void trace_report(const TcArgs& a, int T0, unsigned grid, cudaStream_t st) {
    std::vector<long long> h(16 * (a.num_jt + 4));
    WGP_CUDA(cudaMemcpyAsync(h.data(), a.trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    if (const char* dump = getenv("WGP_TC_TRACE_DUMP")) {  // raw stamps, 16 per tile, for offline analysis
      if (FILE* f = fopen(dump, "wb")) {
        fwrite(h.data(), sizeof(long long), h.size(), f);
        fclose(f);
      }
    }
    // per tile: [0] MMA-1 committed, [1] epilogue woke (S ready), [2] epilogue
    // arrived kfull, [3] MMA-2 passed its waits, [4] MMA-2 loop top, [5] MMA-2
    // issued, [6] MMA-1 loop top, [7] MMA-1 passed its waits.  Means over the
    // steady-state tiles of CTA 0 (clk).
    double v[14] = {0};
    int cnt = 0;
    for (int t = 8; t + 2 < T0; ++t) {
      const long long* r = &h[16 * t];
      const long long* n = &h[16 * (t + 1)];
      for (int q = 0; q < 4; ++q) v[10 + q] += r[8 + q] - r[1];  // wake -> kfull arrive, lane quarter q
      v[0] += r[1] - r[0];   // S ready -> epilogue wake
      v[1] += r[2] - r[1];   // epilogue
      v[2] += r[3] - r[2];   // kfull -> MMA-2 past waits
      v[3] += n[4] - r[4];   // MMA-2 period
      v[4] += r[3] - r[4];   // MMA-2 waiting (odrained, vfull, kfull)
      v[5] += r[5] - r[3];   // MMA-2 issuing
      v[6] += n[4] - r[5];   // MMA-2 commits + loop
      v[7] += r[7] - r[6];   // MMA-1 waiting (m2done, bfull)
      v[8] += r[0] - r[7];   // MMA-1 issuing + commits
      v[9] += n[6] - r[6];   // MMA-1 period
      ++cnt;
    }
    {
      double w_od = 0, w_v = 0, w_k = 0;
      int m = 0;
      for (int t = 8; t + 2 < T0; ++t) {
        const long long* r = &h[16 * t];
        w_od += r[12] - r[4];
        w_v += r[13] - r[12];
        w_k += r[3] - r[13];
        ++m;
      }
      if (m)
        fprintf(stderr, "[hv_tc trace] MMA-2 waits per tile: odrained %.0f  vfull %.0f  kfull %.0f clk\n", w_od / m,
                w_v / m, w_k / m);
    }
    if (cnt)
      fprintf(stderr,
              "[hv_tc trace] tiles=%d S->epi %.0f epi %.0f kfull->mma2 %.0f | MMA-2 period %.0f = wait %.0f + "
              "issue %.0f + commit %.0f | MMA-1 period %.0f: wait %.0f issue+commit %.0f clk\n",
              cnt, v[0] / cnt, v[1] / cnt, v[2] / cnt, v[3] / cnt, v[4] / cnt, v[5] / cnt, v[6] / cnt, v[9] / cnt,
              v[7] / cnt, v[8] / cnt);
    {
      std::vector<long long> c(12 * grid);
      WGP_CUDA(cudaMemcpy(c.data(), a.ctatime, sizeof(long long) * c.size(), cudaMemcpyDeviceToHost));
      long long t0 = c[1], t1 = c[3];
      double dur = 0, tail = 0, s_m2 = 0, s_of = 0, s_dr = 0, s_ex = 0, s_tl = 0, s_fo = 0, s_cw = 0;
      for (unsigned b = 0; b < grid; ++b) {
        t0 = std::min(t0, c[12 * b + 1]);
        t1 = std::max(t1, c[12 * b + 3]);
        dur += c[12 * b + 3] - c[12 * b + 1];
        tail += c[12 * b + 3] - c[12 * b + 2];
        s_m2 += c[12 * b + 6] - c[12 * b + 2];
        s_of += c[12 * b + 4] - c[12 * b + 2];
        s_dr += c[12 * b + 5] - c[12 * b + 4];
        s_tl += c[12 * b + 7] - c[12 * b + 4];
        s_fo += c[12 * b + 8] - c[12 * b + 7];
        s_cw += c[12 * b + 9] - c[12 * b + 8];
        s_ex += c[12 * b + 3] - c[12 * b + 5];
      }
      double f1 = 0, f2 = 0;
      for (unsigned b = 0; b < grid; ++b) {
        f1 += c[12 * b + 11] - c[12 * b + 1];
        f2 += c[12 * b + 10] - c[12 * b + 1];
      }
      fprintf(stderr, "[hv_tc trace] fill from CTA start: first Gram group issued %.1f us, first K.V tile issued %.1f us\n",
              f1 / grid / 1e3, f2 / grid / 1e3);
      fprintf(stderr, "[hv_tc trace] tail from epilogue loop end: last MMA-2 issued %+.1f us, ofull seen %.1f, "
              "final drain %.1f (TMEM read %.1f, fold %.1f, cp.async wait %.1f), sync+exit %.1f us\n",
              s_m2 / grid / 1e3, s_of / grid / 1e3, s_dr / grid / 1e3, s_tl / grid / 1e3, s_fo / grid / 1e3,
              s_cw / grid / 1e3, s_ex / grid / 1e3);
      // gaps between consecutive CTAs on one SM
      std::vector<std::vector<std::pair<long long, long long>>> per_sm(256);
      for (unsigned b = 0; b < grid; ++b) per_sm[c[12 * b] & 255].push_back({c[12 * b + 1], c[12 * b + 3]});
      double gap = 0;
      int ng = 0;
      for (auto& v : per_sm) {
        std::sort(v.begin(), v.end());
        for (size_t i = 1; i < v.size(); ++i) gap += v[i].first - v[i - 1].second, ++ng;
      }
      fprintf(stderr,
              "[hv_tc trace] grid %u: span %.1f us, CTA mean %.1f us (last drain+exit %.1f us), "
              "SM gap between CTAs %.1f us (%d)\n",
              grid, (t1 - t0) / 1e3, dur / grid / 1e3, tail / grid / 1e3, ng ? gap / ng / 1e3 : 0.0, ng);
    }
    if (cnt)  // quarter q shares SMSP q with control warp 12 + q (measured: the MMA-warp SMSPs lag)
      fprintf(stderr, "[hv_tc trace] epilogue per lane quarter (SMSP): %.0f %.0f %.0f %.0f clk\n", v[10] / cnt,
              v[11] / cnt, v[12] / cnt, v[13] / cnt);
  }

void hv_tc(TcOperands& ops, const HvParams& hp, cudaStream_t st, bool bf16) {
  if (hp.s > 96) {  // the V ring holds at most 96 columns: balanced column chunks
    const int chunks = static_cast<int>(ceil_div(hp.s, 96));
    for (int c = 0; c < chunks; ++c) {
      const int c0 = hp.s * c / chunks, c1 = hp.s * (c + 1) / chunks;
      HvParams q = hp;
      q.s = c1 - c0;
      q.V = hp.V + c0 * hp.ldv;
      if (hp.v_host) q.v_host = hp.v_host + c0 * hp.ldv;
      q.out = hp.out + c0 * hp.ldo;
      if (hp.B) q.B = hp.B + c0 * hp.ldb;
      q.vplanes = nullptr;
      q.reuse_vsplit = false;
      hv_tc(ops, q, st, bf16);
    }
    return;
  }
  if (!ops.ws) ops.ws = new TcWorkspaces();
  Workspace& ws_v = ops.ws->v;
  Workspace& ws_rows = ops.ws->rows;
  Workspace& ws_part = ops.ws->part;
  if (hp.m <= 0 || hp.j1 <= hp.j0) return;
  const int s = hp.s;
  const int spad = static_cast<int>(round_up(s, 16));
  const int64_t nv = hp.j1 - hp.j0;
  const int64_t ldw = round_up(nv, 8);
  const int TJ = bf16 ? Cfg<true>::kTJ : Cfg<false>::kTJ;
  // hi / lo planes of V[j0:j1]: tf32 (fp32 storage) or column-scaled fp16 (split_v_f16_kernel)
  const size_t esz = bf16 ? 2 : 4;
  // caller-maintained planes (16-byte aligned rows for TMA) or this launch's split
  const bool pre = !bf16 && hp.vplanes && hp.j0 % 4 == 0 && hp.vplanes_ld % 4 == 0 && hp.vplanes_ld >= hp.j1;
  // (the split workspace is sized even when unused: a later launch in a CUDA
  // graph capture, e.g. CG's refresh H.V of X, must not allocate)
  const size_t plane_bytes = round_up(esz * ldw * s * 2, 256);
  char* wsv = static_cast<char*>(ws_v.ensure(plane_bytes + 8 * 128));
  float* vscale = reinterpret_cast<float*>(wsv + plane_bytes);  // [128] 2^-e_c (H16)
  char* vhi = pre ? reinterpret_cast<char*>(const_cast<float*>(hp.vplanes + hp.j0)) : wsv;
  char* vlo = pre ? reinterpret_cast<char*>(const_cast<float*>(hp.vplanes + hp.j0 + hp.vplanes_ld * s))
                  : vhi + esz * ldw * s;
  const int64_t ldp = pre ? hp.vplanes_ld : ldw;  // plane leading dimension
  const dim3 vgrid(static_cast<unsigned>(ceil_div(nv, 256)), s);
  if (pre || hp.reuse_vsplit) {
  } else if (bf16) {
    split_v_f16_kernel<<<dim3(kSplitCl, s), kSplitThreads, 0, st>>>(hp.V, hp.ldv, hp.j0, nv,
                                                                     reinterpret_cast<__half*>(vhi),
                                                                     reinterpret_cast<__half*>(vlo), ldw, vscale,
                                                                     hp.v_host, hp.v_host ? const_cast<float*>(hp.V) : nullptr);
  } else
    split_v_kernel<<<vgrid, 256, 0, st>>>(hp.V, hp.ldv, hp.j0, nv, reinterpret_cast<float*>(vhi),
                                          reinterpret_cast<float*>(vlo), ldw, hp.v_host,
                                          hp.v_host ? const_cast<float*>(hp.V) : nullptr);
  WGP_LAUNCH_CHECK();
  // A rows: the operand planes directly (row range) or a gathered copy
  const float* ahi = static_cast<const float*>(ops.a_hi);
  const float* alo = static_cast<const float*>(ops.a_lo);
  int64_t a_rows = ops.n_pad;
  int a_row0 = static_cast<int>(hp.r0);
  const int64_t m_pad = round_up(hp.m, 128);
  if (hp.row_idx) {
    float* g = static_cast<float*>(ws_rows.ensure(sizeof(float) * m_pad * kKA * 2));
    gather_rows_kernel<<<static_cast<unsigned>(ceil_div(m_pad * kKA, 256)), 256, 0, st>>>(
        ahi, alo, hp.row_idx, hp.m, g, g + m_pad * kKA, m_pad);
    WGP_LAUNCH_CHECK();
    ahi = g;
    alo = g + m_pad * kKA;
    a_rows = m_pad;
    a_row0 = 0;
  }
  const CUtensorMap mAhi = make_map(ahi, kKA, a_rows, kKA * 4, kKA, kTI);
  const CUtensorMap mAlo = make_map(alo, kKA, a_rows, kKA * 4, kKA, kTI);
  const CUtensorMap mBhi = make_map(ops.b_hi, kKA, ops.n_pad, kKA * 4, kKA, 64);  // MMA-1 N = 64 points
  const CUtensorMap mBlo = make_map(ops.b_lo, kKA, ops.n_pad, kKA * 4, kKA, 64);
  // one TJ-point x s_pad box per plane (128-byte rows: 32 tf32 / 64 bf16 points)
  const CUtensorMapDataType vt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUtensorMap mVhi = make_map(vhi, nv, s, ldp * esz, TJ, spad, vt);
  const CUtensorMap mVlo = make_map(vlo, nv, s, ldp * esz, TJ, spad, vt);

  TcArgs a{};
  a.m = hp.m;
  a.a_row0 = a_row0;
  a.j0 = hp.j0;
  a.j1 = hp.j1;
  a.num_jt = static_cast<int>(ceil_div(nv, TJ));
  a.s = s;
  a.s_pad = spad;
  // Ring depths: V tiles are consumed by MMA-2 and must be prefetched far
  // enough ahead to cover the L2->SMEM latency (measured: 3 stages starve
  // MMA-2); the B ring only feeds MMA-1, which runs ahead anyway.
  static const int env_nb = [] {
    const char* e = getenv("WGP_TC_NB");
    return e ? atoi(e) : 0;
  }();
  static const int env_nv = [] {
    const char* e = getenv("WGP_TC_NV");
    return e ? atoi(e) : 0;
  }();
  a.vstage_bytes = 2u * static_cast<uint32_t>(spad) * 128u;
  // A_I (32 KB) + the running sum R (512 s_pad bytes; aliases A when A lives in TMEM)
  const bool a_tmem = bf16 ? Cfg<true>::kATmem : Cfg<false>::kATmem;
  a.a_region = a_tmem ? std::max(32768u, 512u * spad) : 32768u + 512u * spad;
  const int bstage = 2 * 64 * 128;
  a.nb = env_nb > 0 ? std::min(env_nb, kMaxStages) : 3;
  a.nv = std::min<int>(kMaxStages, (kSmemLimit - static_cast<int>(a.a_region) - 512 * spad - 1024 - a.nb * bstage) /
                                       static_cast<int>(a.vstage_bytes));
  if (env_nv > 0) a.nv = std::min(a.nv, env_nv);
  if (!bf16) a.nv = Cfg<false>::kTilesInFlight;  // V slots share the K slots' barriers
  if (a.nv < 2 || a.nb < 2) throw DeviceError("hv_tc: right-hand side too wide for the V ring");
  a.row_idx = hp.row_idx;
  a.r0 = hp.r0;
  a.V = hp.V;
  a.v_late = hp.v_host ? 1 : 0;
  a.ldv = hp.ldv;
  a.out = hp.out;
  a.ldo = hp.ldo;
  a.B = hp.B;
  a.ldb = hp.ldb;
  a.mode = hp.mode;
  a.sf2 = hp.sf2;
  a.a = hp.a;
  a.diag = hp.diag;
  a.hyp = hp.hyp;
  a.vscale = vscale;
  a.m_pad = m_pad;
  a.done = hp.done;
  static const int dbg = [] {
    const char* e = getenv("WGP_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  a.dbg = dbg;
  a.nk1 = ops.nk1;
#ifdef WGP_TC_ABLATE
  static const bool tracing = getenv("WGP_TC_TRACE") != nullptr;
#else
  static const bool tracing = [] {  // the stamps are compiled out of the default build
    if (getenv("WGP_TC_TRACE")) fprintf(stderr, "[hv_tc] WGP_TC_TRACE needs a -DWGP_TC_ABLATE build\n");
    return false;
  }();
#endif
  static Workspace ws_trace;
  a.trace = nullptr;
  if (tracing) {
    a.trace = static_cast<long long*>(ws_trace.ensure(sizeof(long long) * 16 * (a.num_jt + 4)));
    WGP_CUDA(cudaMemsetAsync(a.trace, 0, sizeof(long long) * 16 * (a.num_jt + 4), st));
  }
  const int64_t row_tiles = ceil_div(hp.m, kTI);
  const int64_t key_tiles = hp.split_rows > 0 ? ceil_div(hp.split_rows, kTI) : row_tiles;
  // L2 rasterisation: every CTA streams the operand planes of its J range
  // (B hi / lo + V hi / lo: 256 + 2 esz s_pad bytes per point).  With one
  // split the concurrently running row tiles drift apart along J over the
  // waves, and once the planes outgrow L2 they re-read them from HBM
  // (config 3, n = 391k: 463 GB of DRAM reads per H.V at a 53% L2 hit rate,
  // ncu).  Splits whose J range fits the budget, with the split-major grid,
  // keep the range L2-resident across all row tiles; the fp32 partials are
  // capped at WGP_TC_PART_GB (default 32 GB, keyed like the splits: a row
  // shard allocates its share).
  static const double l2_budget = [] {
    const char* e = getenv("WGP_TC_L2MB");
    return (e ? atof(e) : 48.0) * 1e6;
  }();
  int min_sp = 1;
  if (l2_budget > 0) {
    const double plane_bytes = static_cast<double>(nv) * (256.0 + 2.0 * static_cast<double>(esz) * spad);
    min_sp = static_cast<int>(std::ceil(plane_bytes / l2_budget));
    // the cap uses the split key's rows, so a row shard picks the full operator's splits
    const double part_row = 4.0 * spad * static_cast<double>(key_tiles * kTI);
    static const double part_cap = [] {
      const char* e = getenv("WGP_TC_PART_GB");
      return (e ? atof(e) : 32.0) * 1e9;
    }();
    min_sp = std::max(1, std::min({min_sp, static_cast<int>(part_cap / part_row), 64}));
  }
  a.splits = choose_splits(key_tiles, a.num_jt, sm_count(), min_sp);
  static const int force_splits = [] {
    const char* e = getenv("WGP_TC_SPLITS");
    return e ? atoi(e) : 0;
  }();
  if (force_splits > 0) a.splits = std::min(force_splits, a.num_jt);
  // fp32 accumulation chunk (tiles): bounds the accumulation error, see the kernel
  static const int env_chunk = [] {
    const char* e = getenv("WGP_TC_CHUNK");
    return e ? atoi(e) : 0;
  }();
  a.chunk = env_chunk >= 4 ? env_chunk : 1024 / TJ;
  static const int env_flush = [] {
    const char* e = getenv("WGP_TC_FLUSH");
    return e ? atoi(e) : 0;
  }();
  a.flush_every = env_flush >= 1 ? env_flush : 64;
  const int max_tiles = static_cast<int>(ceil_div(a.num_jt, a.splits));
  const bool flushes = max_tiles > a.flush_every * a.chunk;
  const size_t part_bytes = a.splits > 1 ? sizeof(float) * a.splits * spad * m_pad : 0;
  const size_t flush_bytes = flushes ? sizeof(double) * a.splits * spad * m_pad : 0;
  char* pw = static_cast<char*>(ws_part.ensure(round_up(part_bytes, 256) + flush_bytes + 256));
  a.part = reinterpret_cast<float*>(pw);
  a.flush = reinterpret_cast<double*>(pw + round_up(part_bytes, 256));
  // The split partial of a CTA, R = [s_pad][128] fp32 in shared memory, is one
  // box of the partial buffer viewed as [splits * s_pad] columns x [m_pad] rows.
  CUtensorMap mPart = mAhi;  // unused unless tma_part
  a.tma_part = 0;
  if (a.splits > 1) {
    mPart = make_map(a.part, static_cast<uint64_t>(m_pad), static_cast<uint64_t>(a.splits) * spad, m_pad * 4, kTI,
                     static_cast<uint32_t>(spad), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CU_TENSOR_MAP_SWIZZLE_NONE);
    a.tma_part = 1;
  }
  const int smem = static_cast<int>(a.a_region) + 1024 + a.nb * bstage + a.nv * static_cast<int>(a.vstage_bytes) +
                   512 * spad;  // + sVd
  const unsigned grid = static_cast<unsigned>(row_tiles * a.splits);
  static Workspace ws_cta;
  a.ctatime = nullptr;
  if (tracing) a.ctatime = static_cast<long long*>(ws_cta.ensure(sizeof(long long) * 12 * grid));
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ops.profiling) {
    WGP_CUDA(cudaEventCreate(&ev0));
    WGP_CUDA(cudaEventCreate(&ev1));
    WGP_CUDA(cudaEventRecord(ev0, st));
  }
  // PDL after the fp16 split only: the tf32 engine's planes may come from the
  // caller's kernels, and with gathered rows the kernel right before this one
  // writes A (the A / B producer does not wait)
  const bool pdl = bf16 && !pre && !hp.reuse_vsplit && !hp.row_idx && tc_pdl() && !ops.profiling && !tracing;
  if (bf16)
    launch_tc<true>(mAhi, mAlo, mBhi, mBlo, mPart, mVhi, mVlo, a, grid, smem, st, pdl);
  else
    launch_tc<false>(mAhi, mAlo, mBhi, mBlo, mPart, mVhi, mVlo, a, grid, smem, st, false);
  if (ops.profiling) {
    WGP_CUDA(cudaEventRecord(ev1, st));
    ops.events.emplace_back(ev0, ev1);
  }
  if (tracing) trace_report(a, static_cast<int>(static_cast<int64_t>(a.num_jt) / a.splits), grid, st);
  if (a.splits > 1) {
    launch_pdl(tc_reduce_kernel, dim3(static_cast<unsigned>(ceil_div(hp.m, 256)), s), dim3(256), 0, st,
               bf16 && tc_pdl() && !ops.profiling, a);
    WGP_LAUNCH_CHECK();
  }
}

}  // namespace wgp
