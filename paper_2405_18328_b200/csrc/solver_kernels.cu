// solver_kernels.cu — CG / AP / SGD vector kernels with fused column
// reductions.  Semantics follow proj/src/solvers.cpp:
// CG :81-139, AP :141-196, SGD :198-263; see solver_kernels.cuh.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "solver_kernels.cuh"

namespace wgp {
namespace {

constexpr int NT = 256;
constexpr int SMAX = 256;

struct Red {
  double v[NT / 32][SMAX];
};

// Per-column partial of the CTA's row range; lane 0 of each warp deposits.
__device__ __forceinline__ void deposit(Red& red, int c, double v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red.v[threadIdx.x >> 5][c] = v;
}

// Writes this CTA's partials and returns true in the last CTA to finish.
// Small n: the grid's y dimension splits the columns into groups of 4 (CTA
// (x, y) takes row block x and column groups y, y + gridDim.y, ...), so each
// CTA makes one pass instead of s / 4 serial ones.  Each (row block, column)
// partial is still produced by one CTA in the same order: results are
// identical to the one-dimensional grid.
__device__ __forceinline__ bool my_col(int c) { return ((c >> 2) % gridDim.y) == blockIdx.y; }

__device__ void block_totals(const double* part, int w, double* tot);

// Row-sharded solves (ColState::dist_loc set): the last CTA stores this
// rank's column totals in dist_loc and stops; the host exchanges the ranks'
// totals (allgather) and dist_finish runs the epilogue on their rank-order
// sum, identically on every rank.
__device__ bool publish(Red& red, int s, double* part, SolveCtrl* ctrl, double* dist_loc = nullptr) {
  __syncthreads();
  for (int c = threadIdx.x; c < s; c += blockDim.x) {
    if (!my_col(c)) continue;
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red.v[w][c];
    part[static_cast<int64_t>(blockIdx.x) * s + c] = t;
  }
  __threadfence();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&ctrl->ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return false;
  __threadfence();
  block_totals(part, s, red.v[0]);  // red's deposits are in part: reuse it
  if (dist_loc) {
    for (int c = threadIdx.x; c < s; c += blockDim.x) dist_loc[c] = red.v[0][c];
    if (threadIdx.x == 0) ctrl->ticket = 0;
    return false;
  }
  return true;
}

// All column totals at once in the last CTA: warp w takes columns w, w + 8,
// ...; its lanes stride over the CTAs' partials and a fixed shuffle tree
// combines them (fixed order: deterministic).  A thread per column walking
// ~160 partials was a chain of L2 round trips (~25 us per reduction kernel,
// 65 us for sgd_check's two, config 2).
__device__ void block_totals(const double* part, int w, double* tot) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned nb = gridDim.x;
  for (int c = warp; c < w; c += NT / 32) {
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned b = lane;
    for (; b + 96 < nb; b += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] += __ldcg(part + static_cast<int64_t>(b + 32 * u) * w + c);
    }
    for (; b < nb; b += 32) t[0] += __ldcg(part + static_cast<int64_t>(b) * w + c);
    const double v = warp_sum((t[0] + t[1]) + (t[2] + t[3]));
    if (lane == 0) tot[c] = v;
  }
  __syncthreads();
}

// Per-column partials of the CTA's rows, four columns at a time with the row
// loop outside, so the loads of four columns are in flight together (a
// column at a time serialised on memory latency: 120 us per CG update at
// n = 2048, measured).  f(c, e) returns element e's contribution to column c.
template <class F>
__device__ __forceinline__ void cols4(int s, int64_t rb, int64_t re, int64_t ld, Red& red, F f) {
  for (int c0 = 4 * static_cast<int>(blockIdx.y); c0 < s; c0 += 4 * static_cast<int>(gridDim.y)) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = rb + threadIdx.x; i < re; i += NT) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u < s) v[u] += f(c0 + u, i + static_cast<int64_t>(c0 + u) * ld);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < s) deposit(red, c0 + u, v[u]);
  }
}

// After the per-column work of the last CTA: count converged columns, promote
// "converged this iteration" to frozen, and decide whether to run another
// iteration (the while-condition of solvers.cpp:107 / :181 / :234).
__device__ void loop_check(int s, ColState cs, SolveCtrl* ctrl, bool begin_next) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->ticket = 0;
    int nconv = 0;
    for (int c = 0; c < s; ++c) nconv += cs.conv[c] != 0;
    ctrl->nconv = nconv;
    if (ctrl->status != kStatusOk) {
      ctrl->done = 1;
    } else if (begin_next) {
      if (nconv == s || ctrl->it >= ctrl->max_it)
        ctrl->done = 1;
      else
        ctrl->it += 1;
    }
  }
}

#define ROWS_OF_BLOCK                                                 \
  const int64_t rpb_ = rows_per_block(n);                             \
  const int64_t rb = static_cast<int64_t>(blockIdx.x) * rpb_;         \
  const int64_t re = rb + rpb_ < n ? rb + rpb_ : n;

template <class T>
__global__ void col_dots_kernel(const T* A, const T* B, int64_t ld, int64_t n, int s,
                                double* part, unsigned* ticket, double* out) {
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(s, rb, re, ld, red, [&](int, int64_t e) { return static_cast<double>(A[e]) * static_cast<double>(B[e]); });
  __syncthreads();
  for (int c = threadIdx.x; c < s; c += NT) {
    if (!my_col(c)) continue;
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red.v[w][c];
    part[static_cast<int64_t>(blockIdx.x) * s + c] = t;
  }
  __threadfence();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  block_totals(part, s, red.v[0]);
  for (int c = threadIdx.x; c < s; c += NT) out[c] = red.v[0][c];
  if (threadIdx.x == 0) *ticket = 0;
}

__device__ void cg_init_epi(int s, ColState cs, const double* tot, SolveCtrl* ctrl) {
  for (int c = threadIdx.x; c < s; c += NT) {
    const double rs = tot[c];
    cs.rs[c] = rs;
    const bool conv = cs.bnorm[c] == 0.0 || sqrt(rs) <= cs.tol[c] * cs.bnorm[c];
    cs.conv[c] = conv ? 1 : 0;
    cs.best[c] = rs;
    cs.stall[c] = 0;
    cs.act[c] = 1;
  }
  loop_check(s, cs, ctrl, true);
}

template <class T>
__global__ void cg_init_kernel(const T* R, int64_t ld, int64_t n, int s,
                               ColState cs, double* part, SolveCtrl* ctrl) {
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(s, rb, re, ld, red, [&](int, int64_t e) {
    const double r = R[e];
    return r * r;
  });
  if (!publish(red, s, part, ctrl, cs.dist_loc)) return;
  cg_init_epi(s, cs, red.v[0], ctrl);
}

// P = R for active columns, 0 otherwise (separate pass: needs conv flags).
// P's tf32 hi / lo planes (HvParams::vplanes) written with P, bitwise hv_tc's split.
__device__ __forceinline__ void put_planes(float*, int64_t, int64_t, double) {}  // fp64 CG: no planes
__device__ __forceinline__ void put_planes(float* pp, int64_t e, int64_t plane, float v) {
  if (!pp) return;
  const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  pp[e] = hi;
  pp[e + plane] = v - hi;
}

template <class T>
__global__ void cg_seed_direction_kernel(T* P, const T* R, int64_t ld, int64_t n, int s,
                                         const int* conv, float* pp) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= n) return;
  const T v = conv[c] ? T(0) : R[i + c * ld];
  P[i + c * ld] = v;
  put_planes(pp, i + c * ld, static_cast<int64_t>(s) * ld, v);
}

__device__ void cg_alpha_epi(int s, ColState cs, const double* tot, SolveCtrl* ctrl) {
  for (int c = threadIdx.x; c < s; c += NT) {
    if (cs.conv[c]) continue;
    const double pHp = tot[c];
    if (!(pHp > 0.0)) {
      atomicCAS(&ctrl->status, kStatusOk, kStatusNotPd);
      ctrl->fail_it = ctrl->it;
    }
    cs.alpha[c] = cs.rs[c] / pHp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->ticket = 0;
    if (ctrl->status != kStatusOk) ctrl->done = 1;
  }
}

template <class T>
__global__ void cg_alpha_kernel(const T* P, const T* HP, int64_t ld, int64_t n, int s,
                                ColState cs, double* part, SolveCtrl* ctrl) {
  if (ctrl->done) return;
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(s, rb, re, ld, red, [&](int c, int64_t e) {
    return cs.conv[c] ? 0.0 : static_cast<double>(P[e]) * static_cast<double>(HP[e]);
  });
  if (!publish(red, s, part, ctrl, cs.dist_loc)) return;
  cg_alpha_epi(s, cs, red.v[0], ctrl);
}

// restart: a refresh step (:119-120).  The reference keeps the direction
// across the residual replacement (beta = |r_true|^2 / |r_old|^2), harmless
// in fp64; in fp32, once the recursive residual has fallen below the
// attainable floor, the true residual jumps by orders of magnitude and the
// inflated beta derails the iteration (measured: residuals 1e17 at tol 1e-6).
// So when the replaced residual exceeds 4x the previous one, the direction
// restarts (beta = 0); at reachable tolerances this does not trigger.
__device__ void beta_epilogue(int s, ColState cs, const double* tot, SolveCtrl* ctrl, bool restart = false) {
  for (int c = threadIdx.x; c < s; c += NT) {
    if (cs.conv[c]) continue;
    const double rs_new = tot[c];
    if (!isfinite(rs_new)) {
      atomicCAS(&ctrl->status, kStatusOk, kStatusNaN);
      ctrl->fail_it = ctrl->it;
    }
    if (restart) cs.act[c] = 0;
    if (sqrt(rs_new) <= cs.tol[c] * cs.bnorm[c]) {
      cs.conv[c] = 2;
      cs.beta[c] = 0.0;
    } else {
      cs.beta[c] = (restart && rs_new > 4.0 * cs.rs[c]) ? 0.0 : rs_new / cs.rs[c];
      if (restart) {  // rs_new is the exact residual: keep the best iterate
        if (rs_new < cs.best[c]) {
          cs.best[c] = rs_new;
          cs.stall[c] = 0;
          cs.act[c] = 1;
        } else if (++cs.stall[c] >= 3 || rs_new > 1e4 * cs.best[c]) {
          cs.act[c] = 2;  // below the attainable accuracy: restore the best, freeze
          cs.conv[c] = 3;
          cs.beta[c] = 0.0;
        }
      }
    }
    cs.rs[c] = rs_new;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctrl->ticket = 0;
    if (ctrl->status != kStatusOk) ctrl->done = 1;
  }
}

__device__ __forceinline__ float axpy(double a, float x, float y) { return fmaf(static_cast<float>(a), x, y); }
__device__ __forceinline__ double axpy(double a, double x, double y) { return fma(a, x, y); }

template <class T>
__global__ void cg_update_kernel(T* X, T* R, const T* P, const T* HP, int64_t ld,
                                 int64_t n, int s, ColState cs, double* part, SolveCtrl* ctrl,
                                 int refresh) {
  if (ctrl->done) return;
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(s, rb, re, ld, red, [&](int c, int64_t e) {
    if (cs.conv[c]) return 0.0;
    const double a = cs.alpha[c];
    X[e] = axpy(a, P[e], X[e]);
    if (refresh) return 0.0;
    const T r = axpy(-a, HP[e], R[e]);
    R[e] = r;
    return static_cast<double>(r) * r;
  });
  if (refresh) return;
  if (!publish(red, s, part, ctrl, cs.dist_loc)) return;
  beta_epilogue(s, cs, red.v[0], ctrl);
}

template <class T>
__global__ void cg_refresh_norm_kernel(T* R, const T* Rtmp, int64_t ld, int64_t n, int s,
                                       ColState cs, double* part, SolveCtrl* ctrl) {
  if (ctrl->done) return;
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(s, rb, re, ld, red, [&](int c, int64_t e) {
    if (cs.conv[c]) return 0.0;
    const T r = Rtmp[e];
    R[e] = r;
    return static_cast<double>(r) * r;
  });
  if (!publish(red, s, part, ctrl, cs.dist_loc)) return;
  beta_epilogue(s, cs, red.v[0], ctrl, true);
}

template <class T>
__global__ void cg_direction_kernel(T* P, const T* R, int64_t ld, int64_t n, int s,
                                    ColState cs, double* part, SolveCtrl* ctrl, float* pp) {
  if (ctrl->done) return;
  ROWS_OF_BLOCK
  for (int64_t i = rb + threadIdx.x; i < re; i += NT) {
    for (int c0 = 4 * static_cast<int>(blockIdx.y); c0 < s; c0 += 4 * static_cast<int>(gridDim.y)) {
#pragma unroll
      for (int c = c0; c < c0 + 4; ++c) {
        if (c >= s) break;
        const int st = cs.conv[c];
        if (st == 1 || st == 3) continue;
        const int64_t e = i + c * ld;
        const T v = st == 2 ? T(0) : axpy(cs.beta[c], P[e], R[e]);
        P[e] = v;
        put_planes(pp, e, static_cast<int64_t>(s) * ld, v);  // skipped columns keep P and its planes
      }
    }
  }
  __syncthreads();
  __threadfence();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&ctrl->ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = threadIdx.x; c < s; c += NT)
    if (cs.conv[c] == 2) cs.conv[c] = 1;
  loop_check(s, cs, ctrl, true);
}

// Grid-wide barrier for cooperatively launched kernels (all CTAs resident).
__device__ void grid_sync(SolveCtrl* ctrl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = &ctrl->bar_gen;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(&ctrl->bar_count, 1u) == gridDim.x * gridDim.y - 1) {
      ctrl->bar_count = 0;
      __threadfence();
      atomicAdd(&ctrl->bar_gen, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// This CTA's column partials (its rows, its column groups) -> part[bx s + c].
__device__ void store_partials(Red& red, int s, double* part) {
  __syncthreads();
  for (int c = threadIdx.x; c < s; c += blockDim.x) {
    if (!my_col(c)) continue;
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red.v[w][c];
    part[static_cast<int64_t>(blockIdx.x) * s + c] = t;
  }
}

// hv64's split reduction for this CTA's rows and column group (fp64 CG,
// HvFold): HP = the fp64 split partials summed in split order + diag P,
// bitwise hv64_reduce_kernel; every split's loads are issued together.
template <class T>
__device__ __forceinline__ void fold_hv(T* HP, const T* P, int64_t ld, int s, int64_t rb, int64_t re,
                                        const HvFold& fold) {
  const double diag = static_cast<double>(fold.hyp[2]);
  const int64_t ks = static_cast<int64_t>(s) * fold.m_pad;
  for (int c0 = 4 * static_cast<int>(blockIdx.y); c0 < s; c0 += 4 * static_cast<int>(gridDim.y)) {
    const int nu = s - c0 < 4 ? s - c0 : 4;
    for (int64_t i = rb + threadIdx.x; i < re; i += NT) {
      const double* src = fold.part + static_cast<int64_t>(c0) * fold.m_pad + i;
      double h[4] = {0.0, 0.0, 0.0, 0.0};
      int k = 0;
      for (; k + 4 <= fold.splits; k += 4) {
        double x[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) x[q][u] = u < nu ? __ldcg(src + (k + q) * ks + u * fold.m_pad) : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) h[u] += x[q][u];
      }
      for (; k < fold.splits; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < nu) h[u] += __ldcg(src + k * ks + u * fold.m_pad);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < nu) {
          const int64_t e = i + static_cast<int64_t>(c0 + u) * ld;
          HP[e] = static_cast<T>(fma(diag, static_cast<double>(P[e]), h[u]));
        }
    }
  }
}

template <class T>
__global__ void cg_fused_kernel(T* X, T* R, T* P, T* HP, int64_t ld, int64_t n, int s, ColState cs,
                                double* part, SolveCtrl* ctrl, float* pp, HvFold fold) {
  if (ctrl->done) return;  // read once by every CTA; CTA 0 updates the control state last
  __shared__ Red red;
  __shared__ int sconv[SMAX], snew[SMAX];
  __shared__ double scoef[SMAX], srs[SMAX];
  __shared__ int sfail;
  ROWS_OF_BLOCK
  for (int c = threadIdx.x; c < s; c += NT) {  // CTA 0 rewrites the column state at the end
    sconv[c] = cs.conv[c];
    srs[c] = cs.rs[c];
  }
  if (threadIdx.x == 0) sfail = 0;
  // (each thread's HP elements are the ones it reads below: no barrier needed)
  if (fold.part) fold_hv(HP, P, ld, s, rb, re, fold);
  __syncthreads();
  // alpha_c = rs_c / (p_c . Hp_c)  (cg_alpha)
  cols4(s, rb, re, ld, red, [&](int c, int64_t e) {
    return sconv[c] ? 0.0 : static_cast<double>(P[e]) * static_cast<double>(HP[e]);
  });
  store_partials(red, s, part);
  grid_sync(ctrl);
  block_totals(part, s, red.v[0]);
  for (int c = threadIdx.x; c < s; c += NT) {
    if (sconv[c]) continue;
    const double pHp = red.v[0][c];
    if (!(pHp > 0.0)) sfail = kStatusNotPd;
    scoef[c] = srs[c] / pHp;
  }
  __syncthreads();
  if (sfail) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      ctrl->status = kStatusNotPd;
      ctrl->fail_it = ctrl->it;
      ctrl->done = 1;
    }
    return;
  }
  // x += alpha p, r -= alpha Hp, ||r||^2  (cg_update); rs_new totals in part + gridDim.x s
  double* part2 = part + static_cast<int64_t>(gridDim.x) * s;
  cols4(s, rb, re, ld, red, [&](int c, int64_t e) {
    if (sconv[c]) return 0.0;
    const double a = scoef[c];
    X[e] = axpy(a, P[e], X[e]);
    const T r = axpy(-a, HP[e], R[e]);
    R[e] = r;
    return static_cast<double>(r) * r;
  });
  store_partials(red, s, part2);
  grid_sync(ctrl);
  block_totals(part2, s, red.v[0]);
  // beta / convergence (beta_epilogue without restart)
  for (int c = threadIdx.x; c < s; c += NT) {
    snew[c] = sconv[c];
    if (sconv[c]) continue;
    const double rs_new = red.v[0][c];
    if (!isfinite(rs_new)) sfail = kStatusNaN;
    if (sqrt(rs_new) <= cs.tol[c] * cs.bnorm[c]) {
      snew[c] = 2;
      scoef[c] = 0.0;
    } else {
      scoef[c] = rs_new / srs[c];
    }
  }
  __syncthreads();
  const bool lead = blockIdx.x == 0 && blockIdx.y == 0;
  if (sfail) {
    if (lead && threadIdx.x == 0) {
      ctrl->status = kStatusNaN;
      ctrl->fail_it = ctrl->it;
      ctrl->done = 1;
    }
    return;
  }
  // p = r + beta p / 0 for the just-converged  (cg_direction)
  for (int64_t i = rb + threadIdx.x; i < re; i += NT) {
    for (int c0 = 4 * static_cast<int>(blockIdx.y); c0 < s; c0 += 4 * static_cast<int>(gridDim.y)) {
#pragma unroll
      for (int c = c0; c < c0 + 4; ++c) {
        if (c >= s) break;
        const int stc = snew[c];
        if (stc == 1 || stc == 3) continue;
        const int64_t e = i + c * ld;
        const T v = stc == 2 ? T(0) : axpy(scoef[c], P[e], R[e]);
        P[e] = v;
        put_planes(pp, e, static_cast<int64_t>(s) * ld, v);
      }
    }
  }
  if (!lead) return;
  // the column state and the loop check, once
  for (int c = threadIdx.x; c < s; c += NT) {
    if (sconv[c]) continue;
    cs.rs[c] = red.v[0][c];
    cs.beta[c] = scoef[c];
    cs.conv[c] = snew[c] == 2 ? 1 : 0;
  }
  loop_check(s, cs, ctrl, true);
}

// restart comment: see beta_epilogue.  The reference iterates to max_iterations
// regardless; in fp64 the tolerances it is used with are reachable, in fp32
// an unreachable one let the iterate drift and blow up between refreshes
// (measured: relative residual 7e10 after 5000 iterations at tol 1e-6), so a
// column whose exact residual has not improved for three refreshes (or grew
// 1e4x past its best) is restored to its best iterate and frozen.
template <class T>
__global__ void cg_snapshot_kernel(T* X, T* R, T* Xb, T* Rb, int64_t ld, int64_t n, int s,
                                   ColState cs, const SolveCtrl* ctrl, int at_start) {
  if (!at_start && ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= n) return;
  const int a = cs.act[c];
  const int64_t e = i + static_cast<int64_t>(c) * ld;
  if (a == 1) {
    Xb[e] = X[e];
    Rb[e] = R[e];
  } else if (a == 2) {
    X[e] = Xb[e];
    R[e] = Rb[e];
  }
}

__device__ void norms_epi(int s, ColState cs, const double* tot, SolveCtrl* ctrl, int check_nan, int begin_next) {
  for (int c = threadIdx.x; c < s; c += NT) {
    const double t = tot[c];
    if (check_nan && !isfinite(t)) {
      atomicCAS(&ctrl->status, kStatusOk, kStatusNaN);
      ctrl->fail_it = ctrl->it;
    }
    cs.rs[c] = t;
    cs.conv[c] = (cs.bnorm[c] == 0.0 || sqrt(t) <= cs.tol[c] * cs.bnorm[c]) ? 1 : 0;
  }
  loop_check(s, cs, ctrl, begin_next != 0);
}

__global__ void norms_convergence_kernel(const float* R, int64_t ld, int64_t n, int s, ColState cs,
                                         double* part, SolveCtrl* ctrl, int check_nan,
                                         int begin_next) {
  if (begin_next && ctrl->done) return;
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(s, rb, re, ld, red, [&](int, int64_t e) {
    const double r = R[e];
    return r * r;
  });
  if (!publish(red, s, part, ctrl, cs.dist_loc)) return;
  norms_epi(s, cs, red.v[0], ctrl, check_nan, begin_next);
}

// The epilogue of a row-sharded reduction: column totals = the ranks'
// totals (all[r * w + c]) summed in rank order, then the kind's epilogue.
__global__ void dist_finish_kernel(int kind, const double* all, int nranks, int w, int s, ColState cs,
                                   SolveCtrl* ctrl, double* out, int flag_a, int flag_b) {
  if (kind == kDistAlpha || kind == kDistBeta || kind == kDistRefresh) {
    if (ctrl->done) return;
  } else if (kind == kDistNorms && flag_b && ctrl->done) {
    return;
  }
  __shared__ double tot[SMAX];
  for (int c = threadIdx.x; c < w; c += NT) {
    double t = 0.0;
    for (int r = 0; r < nranks; ++r) t += all[static_cast<int64_t>(r) * w + c];
    tot[c] = t;
  }
  __syncthreads();
  switch (kind) {
    case kDistInit: cg_init_epi(s, cs, tot, ctrl); break;
    case kDistAlpha: cg_alpha_epi(s, cs, tot, ctrl); break;
    case kDistBeta: beta_epilogue(s, cs, tot, ctrl); break;
    case kDistRefresh: beta_epilogue(s, cs, tot, ctrl, true); break;
    case kDistNorms: norms_epi(s, cs, tot, ctrl, flag_a, flag_b); break;
    default:
      for (int c = threadIdx.x; c < w; c += NT) out[c] = tot[c];
  }
}

__global__ void ap_gather_kernel(const float* R, int64_t ld, int64_t start, int64_t b, int s,
                                 double* Rb, const SolveCtrl* ctrl) {
  if (ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i < b) Rb[i + c * b] = R[start + i + c * ld];
}

__global__ void ap_apply_kernel(float* X, int64_t ld, int64_t start, int64_t b, int s,
                                const double* delta, int kparts, float* dx, float* dxp, const SolveCtrl* ctrl) {
  if (ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= b) return;
  double dv = delta[i + c * b];  // split-K partials of the block solve, summed in fixed order
  for (int k = 1; k < kparts; ++k) dv += delta[static_cast<int64_t>(k) * b * s + i + c * b];
  X[start + i + c * ld] = static_cast<float>(static_cast<double>(X[start + i + c * ld]) + dv);
  const float d32 = static_cast<float>(dv);
  dx[start + i + c * ld] = d32;  // this epoch's change of block b (Delta X)
  if (dxp) {  // and its tf32 hi / lo planes (hv_tc's split of V, bitwise)
    const float hi = __uint_as_float(__float_as_uint(d32) & 0xFFFFE000u);
    dxp[start + i + c * ld] = hi;
    dxp[start + i + (s + c) * ld] = d32 - hi;
  }
}

// H[b, b] (fp64) padded to `full` x `full` with the identity (so a partial last
// block joins the uniform batched factorisation without changing its solve).
__global__ void build_block_kernel(const float* xs, int dp, int64_t start, int64_t b, int64_t full, double sf2,
                                   double a, double noise2, double* out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= full * full) return;
  const int64_t i = e % full, j = e / full;
  if (i >= b || j >= b) {
    out[e] = i == j ? 1.0 : 0.0;
    return;
  }
  const float* xa = xs + (start + i) * dp;
  const float* xb = xs + (start + j) * dp;
  double r2 = 0.0;
  for (int k = 0; k < dp; ++k) {
    const double df = static_cast<double>(xa[k]) - static_cast<double>(xb[k]);
    r2 += df * df;
  }
  const double u = sqrt(r2);
  double v = (a * u + sf2) * exp2(-u);
  if (i == j) v += noise2;
  out[e] = v;
}

// nb identity matrices of size b x b (column-major, contiguous)
__global__ void identity_kernel(double* A, int64_t b, int64_t total) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int64_t r = e % (b * b);
  A[e] = (r % b == r / b) ? 1.0 : 0.0;
}

__global__ void sgd_scatter_kernel(float* X, float* R, float* vel, int64_t ld, const int* idx,
                                   int64_t m, int s, const float* batch, float mu, float gs,
                                   float ss, float* xp, const SolveCtrl* ctrl) {
  if (ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= m) return;
  const int64_t row = idx[i];
  const int64_t e = row + c * ld;
  const float br = batch[i + c * m];
  const float v = mu * vel[e] - gs * br;
  vel[e] = v;
  const float x = X[e] - ss * v;
  X[e] = x;
  R[e] = br;
  if (xp) {  // X's tf32 hi / lo planes (hv's split of V, bitwise) follow the update
    const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    xp[e] = hi;
    xp[e + static_cast<int64_t>(s) * ld] = x - hi;
  }
}

// sgd_step: CTA (bx, c) scatters rows [256 bx, 256 bx + 256) of column c and
// deposits its column-c change of ||R||^2 and ||X||^2; the last CTA folds the
// changes in fixed order (column c: bx ascending; X: c, then bx) and runs the
// checks of sgd_check_kernel.
__global__ void sgd_step_kernel(float* X, float* R, float* vel, int64_t ld, const int* idx, int64_t m, int s,
                                const float* batch, float mu, float gs, float ss, float* xp, ColState cs,
                                double* xsq, double* part, SolveCtrl* ctrl) {
  if (ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  double dr = 0.0, dx = 0.0;
  if (i < m) {
    const int64_t row = idx[i];
    const int64_t e = row + c * ld;
    const float br = batch[i + c * m];
    const float v = mu * vel[e] - gs * br;
    vel[e] = v;
    const float x0 = X[e], r0 = R[e];
    const float x = x0 - ss * v;
    X[e] = x;
    R[e] = br;
    if (xp) {
      const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      xp[e] = hi;
      xp[e + static_cast<int64_t>(s) * ld] = x - hi;
    }
    dr = static_cast<double>(br) * br - static_cast<double>(r0) * r0;
    dx = static_cast<double>(x) * x - static_cast<double>(x0) * x0;
  }
  __shared__ double sr[NT / 32], sx[NT / 32];
  dr = warp_sum(dr);
  dx = warp_sum(dx);
  if ((threadIdx.x & 31) == 0) {
    sr[threadIdx.x >> 5] = dr;
    sx[threadIdx.x >> 5] = dx;
  }
  __syncthreads();
  const unsigned gx = gridDim.x;
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < NT / 32; ++w) {
      a += sr[w];
      b += sx[w];
    }
    part[static_cast<int64_t>(c) * gx + blockIdx.x] = a;
    part[static_cast<int64_t>(s) * gx + static_cast<int64_t>(c) * gx + blockIdx.x] = b;
  }
  __threadfence();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&ctrl->ticket, 1u) == gx * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // thread cc folds column cc's gx partials in order (column s + c: column
  // c's change of ||X||^2); the loads of all columns are in flight together
  __shared__ double sdx[SMAX];
  for (int cc = threadIdx.x; cc < 2 * s; cc += NT) {
    double t = 0.0;
    for (unsigned b = 0; b < gx; ++b) t += __ldcg(part + static_cast<int64_t>(cc) * gx + b);
    if (cc < s) {
      const double r2 = cs.rs[cc] + t;
      cs.rs[cc] = r2;
      cs.conv[cc] = (cs.bnorm[cc] == 0.0 || sqrt(fmax(r2, 0.0)) <= cs.tol[cc] * cs.bnorm[cc]) ? 1 : 0;
    } else {
      sdx[cc - s] = t;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x2 = *xsq;
    for (int cc = 0; cc < s; ++cc) x2 += sdx[cc];
    *xsq = x2;
    const double xn = sqrt(fmax(x2, 0.0));
    if (!isfinite(xn) || xn > 1e12) {
      ctrl->status = kStatusDiverged;
      ctrl->fail_it = ctrl->it;
    }
  }
  loop_check(s, cs, ctrl, true);
}

// exact re-sync of sgd_step's running norms (reduction pattern of sgd_check)
__global__ void sgd_norms_kernel(const float* X, const float* R, int64_t ld, int64_t n, int s, ColState cs,
                                 double* xsq, double* part, SolveCtrl* ctrl) {
  if (ctrl->done) return;
  __shared__ Red red;
  ROWS_OF_BLOCK
  cols4(2 * s, rb, re, ld, red, [&](int c, int64_t e) {
    const double v = c < s ? static_cast<double>(R[e]) : static_cast<double>(X[e - static_cast<int64_t>(s) * ld]);
    return v * v;
  });
  if (!publish(red, 2 * s, part, ctrl)) return;
  for (int c = threadIdx.x; c < s; c += NT) cs.rs[c] = red.v[0][c];
  if (threadIdx.x == 0) {
    double x2 = 0.0;
    for (int c = 0; c < s; ++c) x2 += red.v[0][s + c];
    *xsq = x2;
    ctrl->ticket = 0;
  }
}

__global__ void tf32_planes_kernel(const float* X, int64_t ld, int64_t n, int s, float* xp) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= n) return;
  const int64_t e = i + c * ld;
  const float x = X[e];
  const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  xp[e] = hi;
  xp[e + static_cast<int64_t>(s) * ld] = x - hi;
}

__global__ void sgd_check_kernel(const float* X, const float* R, int64_t ld, int64_t n, int s,
                                 ColState cs, double* part, SolveCtrl* ctrl) {
  if (ctrl->done) return;
  __shared__ Red red;
  ROWS_OF_BLOCK
  // 2s virtual columns: c < s ||R_c||^2, s + c ||X_c||^2 (summed to ||X||_F^2
  // in fixed order), so the column groups of the 2D grid each publish their
  // own share (a per-CTA X sum deposited once ran 65 us per step in a 1D
  // grid of ~160 CTAs walking all columns, config 2)
  // (1D grid -- enough row blocks, or s >= SMAX / 2: s + 1 columns,
  // ||X||_F^2 per CTA in column s)
  const bool split_x = gridDim.y > 1;
  const int w = split_x ? 2 * s : s + 1;
  if (split_x) {
    cols4(2 * s, rb, re, ld, red, [&](int c, int64_t e) {
      const double v = c < s ? static_cast<double>(R[e]) : static_cast<double>(X[e - static_cast<int64_t>(s) * ld]);
      return v * v;
    });
  } else {
    double xs = 0.0;
    cols4(s, rb, re, ld, red, [&](int, int64_t e) {
      const double r = R[e];
      const double x = X[e];
      xs += x * x;
      return r * r;
    });
    deposit(red, s, xs);
  }
  if (!publish(red, w, part, ctrl)) return;
  for (int c = threadIdx.x; c < s; c += NT) {
    const double t = red.v[0][c];
    cs.conv[c] = (cs.bnorm[c] == 0.0 || sqrt(t) <= cs.tol[c] * cs.bnorm[c]) ? 1 : 0;
  }
  if (threadIdx.x == 0) {
    double x2 = 0.0;
    if (split_x)
      for (int c = 0; c < s; ++c) x2 += red.v[0][s + c];
    else
      x2 = red.v[0][s];
    const double xn = sqrt(x2);
    if (!isfinite(xn) || xn > 1e12) {
      ctrl->status = kStatusDiverged;
      ctrl->fail_it = ctrl->it;
    }
  }
  loop_check(s, cs, ctrl, true);
}

__global__ void fill_zero_kernel(float* A, int64_t ld, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) A[i + blockIdx.y * ld] = 0.f;
}
__global__ void sub_kernel(const float* A, const float* B, float* out, int64_t ld, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t e = i + blockIdx.y * ld;
  if (i < n) out[e] = A[e] - B[e];
}
__global__ void copy_kernel(const float* A, int64_t lda, float* B, int64_t ldb, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) B[i + blockIdx.y * ldb] = A[i + blockIdx.y * lda];
}

inline dim3 grid2(int64_t n, int s) { return dim3(static_cast<unsigned>(ceil_div(n, NT)), s); }
// reduction kernels: row blocks x column groups of 4 while the row blocks alone
// leave SMs idle (config 0: 8 row blocks for n = 2048)
inline dim3 cgrid(int64_t n, int s) {
  // ~4 CTAs per SM: at config 2 (161 row blocks, 130 columns) one column
  // group per CTA walked 33 groups of 4 loads serially (88 us per pass)
  const int rb = reduce_blocks(n);
  const int groups = (s + 3) / 4;
  const int y = std::max(1, std::min(groups, (592 + rb - 1) / rb));
  return dim3(static_cast<unsigned>(rb), static_cast<unsigned>(y));
}
// the cooperative cg_fused kernel: every CTA resident; column groups as in
// cgrid (~4 CTAs per SM): one column group per CTA left config 2's fused fp64
// iteration latency-bound (161 CTAs walking 17 groups of 4 columns: 226 us)
inline dim3 coop_grid(int64_t n, int s) { return cgrid(n, s); }

void check_s(int s) {
  if (s < 1 || s >= SMAX) throw std::invalid_argument("solver kernels support 1 <= s < 256 columns");
}

}  // namespace

template <class T>
void cg_snapshot(T* X, T* R, T* Xb, T* Rb, int64_t ld, int64_t n, int s, ColState cs,
                 const SolveCtrl* ctrl, bool at_start, cudaStream_t st) {
  if (n <= 0) return;
  cg_snapshot_kernel<<<dim3(static_cast<unsigned>(ceil_div(n, NT)), s), NT, 0, st>>>(X, R, Xb, Rb, ld, n, s, cs,
                                                                                     ctrl, at_start ? 1 : 0);
  WGP_LAUNCH_CHECK();
}

template <class T>
void col_dots(const T* A, const T* B, int64_t ld, int64_t n, int s, double* part,
              unsigned* ticket, double* out, cudaStream_t st) {
  check_s(s);
  col_dots_kernel<<<cgrid(n, s), NT, 0, st>>>(A, B, ld, n, s, part, ticket, out);
  WGP_LAUNCH_CHECK();
}

template <class T>
void cg_init(const T* R, int64_t ld, int64_t n, int s, ColState cs, double* part, SolveCtrl* ctrl,
             cudaStream_t st) {
  check_s(s);
  cg_init_kernel<<<cgrid(n, s), NT, 0, st>>>(R, ld, n, s, cs, part, ctrl);
  WGP_LAUNCH_CHECK();
}

template <class T>
void cg_seed(T* P, const T* R, int64_t ld, int64_t n, int s, const int* conv, cudaStream_t st, float* pp) {
  if (n <= 0) return;
  cg_seed_direction_kernel<<<grid2(n, s), NT, 0, st>>>(P, R, ld, n, s, conv, pp);
  WGP_LAUNCH_CHECK();
}

template <class T>
void cg_alpha(const T* P, const T* HP, int64_t ld, int64_t n, int s, ColState cs,
              double* part, SolveCtrl* ctrl, cudaStream_t st) {
  cg_alpha_kernel<<<cgrid(n, s), NT, 0, st>>>(P, HP, ld, n, s, cs, part, ctrl);
  WGP_LAUNCH_CHECK();
}

template <class T>
void cg_update(T* X, T* R, const T* P, const T* HP, int64_t ld, int64_t n, int s,
               ColState cs, double* part, SolveCtrl* ctrl, bool refresh, cudaStream_t st) {
  cg_update_kernel<<<cgrid(n, s), NT, 0, st>>>(X, R, P, HP, ld, n, s, cs, part, ctrl,
                                                    refresh ? 1 : 0);
  WGP_LAUNCH_CHECK();
}

template <class T>
void cg_refresh_norm(T* R, const T* Rtmp, int64_t ld, int64_t n, int s, ColState cs,
                     double* part, SolveCtrl* ctrl, cudaStream_t st) {
  cg_refresh_norm_kernel<<<cgrid(n, s), NT, 0, st>>>(R, Rtmp, ld, n, s, cs, part, ctrl);
  WGP_LAUNCH_CHECK();
}

template <class T>
void cg_direction(T* P, const T* R, int64_t ld, int64_t n, int s, ColState cs,
                  double* part, SolveCtrl* ctrl, cudaStream_t st, float* pp) {
  cg_direction_kernel<<<cgrid(n, s), NT, 0, st>>>(P, R, ld, n, s, cs, part, ctrl, pp);
  WGP_LAUNCH_CHECK();
}

template <class T>
bool cg_fused(T* X, T* R, T* P, T* HP, int64_t ld, int64_t n, int s, ColState cs, double* part,
              SolveCtrl* ctrl, cudaStream_t st, float* pp, HvFold fold) {
  check_s(s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = coop_grid(n, s);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cg_fused_kernel<T>, X, R, P, HP, ld, n, s, cs, part, ctrl, pp, fold);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return true;
}

#define WGP_CG_INSTANTIATE(T)                                                                                  \
  template void cg_snapshot<T>(T*, T*, T*, T*, int64_t, int64_t, int, ColState, const SolveCtrl*, bool,     \
                               cudaStream_t);                                                                \
  template void col_dots<T>(const T*, const T*, int64_t, int64_t, int, double*, unsigned*, double*,         \
                            cudaStream_t);                                                                   \
  template void cg_init<T>(const T*, int64_t, int64_t, int, ColState, double*, SolveCtrl*, cudaStream_t);     \
  template void cg_seed<T>(T*, const T*, int64_t, int64_t, int, const int*, cudaStream_t, float*);             \
  template void cg_alpha<T>(const T*, const T*, int64_t, int64_t, int, ColState, double*, SolveCtrl*,       \
                            cudaStream_t);                                                                   \
  template void cg_update<T>(T*, T*, const T*, const T*, int64_t, int64_t, int, ColState, double*,          \
                             SolveCtrl*, bool, cudaStream_t);                                                \
  template void cg_refresh_norm<T>(T*, const T*, int64_t, int64_t, int, ColState, double*, SolveCtrl*,      \
                                   cudaStream_t);                                                            \
  template void cg_direction<T>(T*, const T*, int64_t, int64_t, int, ColState, double*, SolveCtrl*,         \
                                cudaStream_t, float*);                                                       \
  template bool cg_fused<T>(T*, T*, T*, T*, int64_t, int64_t, int, ColState, double*, SolveCtrl*,            \
                            cudaStream_t, float*, HvFold);
WGP_CG_INSTANTIATE(float)
WGP_CG_INSTANTIATE(double)
#undef WGP_CG_INSTANTIATE

__global__ void masked_rows_kernel(const float* R, int64_t ld, int64_t start, int64_t size, int64_t own0,
                                   int64_t own1, float* out, const SolveCtrl* ctrl) {
  if (ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size) return;
  const int64_t g = start + i;
  out[i + blockIdx.y * size] = (g >= own0 && g < own1) ? R[g + blockIdx.y * ld] : 0.f;
}
void masked_rows(const float* R, int64_t ld, int64_t start, int64_t size, int64_t own0, int64_t own1, int s,
                 float* out, const SolveCtrl* ctrl, cudaStream_t st) {
  masked_rows_kernel<<<grid2(size, s), NT, 0, st>>>(R, ld, start, size, own0, own1, out, ctrl);
  WGP_LAUNCH_CHECK();
}
__global__ void widen_block_kernel(const float* A, double* B, int64_t size, const SolveCtrl* ctrl) {
  if (ctrl->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < size) B[i + blockIdx.y * size] = A[i + blockIdx.y * size];
}
void widen_block(const float* A, double* B, int64_t size, int s, const SolveCtrl* ctrl, cudaStream_t st) {
  widen_block_kernel<<<grid2(size, s), NT, 0, st>>>(A, B, size, ctrl);
  WGP_LAUNCH_CHECK();
}

__global__ void widen_kernel(const float* A, int64_t lda, double* B, int64_t ldb, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) B[i + blockIdx.y * ldb] = A[i + blockIdx.y * lda];
}
__global__ void narrow_kernel(const double* A, int64_t lda, float* B, int64_t ldb, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) B[i + blockIdx.y * ldb] = static_cast<float>(A[i + blockIdx.y * lda]);
}
template <class T>
__global__ void diff_cols_kernel(const T* A, const T* B, T* out, int64_t ld, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t e = i + blockIdx.y * ld;
  if (i < n) out[e] = A[e] - B[e];
}
template <class T>
void diff_cols(const T* A, const T* B, T* out, int64_t ld, int64_t n, int s, cudaStream_t st) {
  if (n <= 0) return;
  diff_cols_kernel<<<grid2(n, s), NT, 0, st>>>(A, B, out, ld, n);
  WGP_LAUNCH_CHECK();
}
template void diff_cols<float>(const float*, const float*, float*, int64_t, int64_t, int, cudaStream_t);
template void diff_cols<double>(const double*, const double*, double*, int64_t, int64_t, int, cudaStream_t);

__global__ void axpy_cols_kernel(double a, const double* X, double* Y, int64_t ld, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) Y[i + blockIdx.y * ld] = fma(a, X[i + blockIdx.y * ld], Y[i + blockIdx.y * ld]);
}
void axpy_cols(double a, const double* X, double* Y, int64_t ld, int64_t n, int s, cudaStream_t st) {
  if (n <= 0) return;
  axpy_cols_kernel<<<grid2(n, s), NT, 0, st>>>(a, X, Y, ld, n);
  WGP_LAUNCH_CHECK();
}
void widen(const float* A, int64_t lda, double* B, int64_t ldb, int64_t n, int s, cudaStream_t st) {
  if (n <= 0) return;
  widen_kernel<<<grid2(n, s), NT, 0, st>>>(A, lda, B, ldb, n);
  WGP_LAUNCH_CHECK();
}
void narrow(const double* A, int64_t lda, float* B, int64_t ldb, int64_t n, int s, cudaStream_t st) {
  if (n <= 0) return;
  narrow_kernel<<<grid2(n, s), NT, 0, st>>>(A, lda, B, ldb, n);
  WGP_LAUNCH_CHECK();
}

void dist_finish(int kind, const double* all, int nranks, int w, int s, ColState cs, SolveCtrl* ctrl,
                 double* out, bool flag_a, bool flag_b, cudaStream_t st) {
  if (w > SMAX) throw std::invalid_argument("dist_finish: too many columns");
  dist_finish_kernel<<<1, NT, 0, st>>>(kind, all, nranks, w, s, cs, ctrl, out, flag_a ? 1 : 0, flag_b ? 1 : 0);
  WGP_LAUNCH_CHECK();
}

void norms_convergence(const float* R, int64_t ld, int64_t n, int s, ColState cs, double* part,
                       SolveCtrl* ctrl, bool check_nan, bool begin_next, cudaStream_t st) {
  check_s(s);
  norms_convergence_kernel<<<cgrid(n, s), NT, 0, st>>>(R, ld, n, s, cs, part, ctrl,
                                                            check_nan ? 1 : 0, begin_next ? 1 : 0);
  WGP_LAUNCH_CHECK();
}

void ap_gather(const float* R, int64_t ld, int64_t start, int64_t b, int s, double* Rb,
               const SolveCtrl* ctrl, cudaStream_t st) {
  ap_gather_kernel<<<grid2(b, s), NT, 0, st>>>(R, ld, start, b, s, Rb, ctrl);
  WGP_LAUNCH_CHECK();
}

void ap_apply(float* X, int64_t ld, int64_t start, int64_t b, int s, const double* delta, int kparts,
              float* dx, float* dxp, const SolveCtrl* ctrl, cudaStream_t st) {
  ap_apply_kernel<<<grid2(b, s), NT, 0, st>>>(X, ld, start, b, s, delta, kparts, dx, dxp, ctrl);
  WGP_LAUNCH_CHECK();
}

void identities(double* A, int64_t b, int64_t nb, cudaStream_t st) {
  const int64_t total = b * b * nb;
  identity_kernel<<<static_cast<unsigned>(ceil_div(total, NT)), NT, 0, st>>>(A, b, total);
  WGP_LAUNCH_CHECK();
}

void build_block(const float* xs, int dp, int64_t start, int64_t b, int64_t full, double sf2, double a,
                 double noise2, double* out, cudaStream_t st) {
  build_block_kernel<<<static_cast<unsigned>(ceil_div(full * full, NT)), NT, 0, st>>>(
      xs, dp, start, b, full, sf2, a, noise2, out);
  WGP_LAUNCH_CHECK();
}

void sgd_scatter(float* X, float* R, float* vel, int64_t ld, const int* idx, int64_t m, int s,
                 const float* batch, float momentum, float grad_scale, float step_scale, float* xp,
                 const SolveCtrl* ctrl, cudaStream_t st) {
  sgd_scatter_kernel<<<grid2(m, s), NT, 0, st>>>(X, R, vel, ld, idx, m, s, batch, momentum,
                                                 grad_scale, step_scale, xp, ctrl);
  WGP_LAUNCH_CHECK();
}

void sgd_step(float* X, float* R, float* vel, int64_t ld, const int* idx, int64_t m, int s, const float* batch,
              float momentum, float grad_scale, float step_scale, float* xp, ColState cs, double* xsq,
              double* part, SolveCtrl* ctrl, cudaStream_t st) {
  check_s(s);
  sgd_step_kernel<<<grid2(m, s), NT, 0, st>>>(X, R, vel, ld, idx, m, s, batch, momentum, grad_scale, step_scale,
                                              xp, cs, xsq, part, ctrl);
  WGP_LAUNCH_CHECK();
}

void sgd_norms(const float* X, const float* R, int64_t ld, int64_t n, int s, ColState cs, double* xsq,
               double* part, SolveCtrl* ctrl, cudaStream_t st) {
  check_s(2 * s);
  sgd_norms_kernel<<<cgrid(n, 2 * s), NT, 0, st>>>(X, R, ld, n, s, cs, xsq, part, ctrl);
  WGP_LAUNCH_CHECK();
}

void tf32_planes(const float* X, int64_t ld, int64_t n, int s, float* xp, cudaStream_t st) {
  tf32_planes_kernel<<<grid2(n, s), NT, 0, st>>>(X, ld, n, s, xp);
  WGP_LAUNCH_CHECK();
}

void sgd_check(const float* X, const float* R, int64_t ld, int64_t n, int s, ColState cs,
               double* part, SolveCtrl* ctrl, cudaStream_t st) {
  check_s(s + 1);
  // part holds reduce_blocks(n) x max(s + 2, 2 s) doubles (Ctx::ensure_solver_ws)
  const int rb = reduce_blocks(n);
  const dim3 grid = (rb < 148 && 2 * s < SMAX) ? cgrid(n, 2 * s) : dim3(static_cast<unsigned>(rb));
  sgd_check_kernel<<<grid, NT, 0, st>>>(X, R, ld, n, s, cs, part, ctrl);
  WGP_LAUNCH_CHECK();
}

void fill_zero(float* A, int64_t ld, int64_t n, int s, cudaStream_t st) {
  if (n <= 0) return;
  fill_zero_kernel<<<grid2(n, s), NT, 0, st>>>(A, ld, n);
  WGP_LAUNCH_CHECK();
}
void sub_into(const float* A, const float* B, float* out, int64_t ld, int64_t n, int s,
              cudaStream_t st) {
  if (n <= 0) return;
  sub_kernel<<<grid2(n, s), NT, 0, st>>>(A, B, out, ld, n);
  WGP_LAUNCH_CHECK();
}
void copy_cols(const float* A, int64_t lda, float* B, int64_t ldb, int64_t n, int s,
               cudaStream_t st) {
  if (n <= 0) return;
  copy_kernel<<<grid2(n, s), NT, 0, st>>>(A, lda, B, ldb, n);
  WGP_LAUNCH_CHECK();
}

}  // namespace wgp
