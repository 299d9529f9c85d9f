// solver_kernels.cuh — fused solver-vector kernels.
//
// Control state lives on the device so an iteration is a fixed launch
// sequence with no host round trip; the host polls `SolveCtrl` every few
// iterations.  All column reductions are two-phase (per-CTA fp64 partials,
// then a fixed-order sum by the last CTA to finish) so results are bitwise
// reproducible.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wgp {

struct SolveCtrl {
  int done;       // 1: the iteration loop has finished (or failed)
  int it;         // iterations / epochs / steps performed
  int status;     // kStatus*
  int fail_it;    // iteration at which a failure was detected
  int nconv;      // converged columns
  int max_it;
  unsigned ticket;
  int pad;
  unsigned bar_count;  // grid barrier of the cooperative cg_fused kernel
  unsigned bar_gen;
};

enum : int { kStatusOk = 0, kStatusNotPd = 1, kStatusNaN = 2, kStatusDiverged = 3 };

// Column state: 0 active, 1 converged (frozen), 2 converged in this iteration,
// 3 stalled below the fp32 attainable accuracy (frozen at its best iterate,
// reported not converged; CG only).
struct ColState {
  int* conv;
  double* rs;      // CG: ||r||^2
  double* alpha;   // CG
  double* beta;    // CG
  const double* bnorm;
  const double* tol;
  double* best;    // CG: smallest exact ||r||^2 seen at a refresh (or the start)
  int* stall;      // CG: refreshes since the last improvement
  int* act;        // CG: 1 snapshot the iterate, 2 restore the snapshot (refresh steps)
  double* dist_loc = nullptr;  // row-sharded solve: this rank's column totals (see dist_finish)
};

// Row-sharded reductions: with ColState::dist_loc set, a reduction kernel
// (cg_init, cg_alpha, cg_update, cg_refresh_norm, norms_convergence) leaves
// this rank's column totals in dist_loc and skips its epilogue; after the
// ranks' totals are gathered into all[nranks][w], dist_finish sums them in
// rank order and runs the epilogue of `kind` (kDistSum: out[c] = total).
enum : int { kDistSum = 0, kDistInit = 1, kDistAlpha = 2, kDistBeta = 3, kDistRefresh = 4, kDistNorms = 5 };
void dist_finish(int kind, const double* all, int nranks, int w, int s, ColState cs, SolveCtrl* ctrl,
                 double* out, bool flag_a, bool flag_b, cudaStream_t st);

// Rows per CTA of the reduction kernels: 256 (one per thread) up to a grid of
// ~2 CTAs per SM; the same function on host and device.
__host__ __device__ inline int64_t rows_per_block(int64_t n) {
  const int64_t want = (n + 295) / 296;  // 2 x 148 SMs
  const int64_t r = ((want + 255) / 256) * 256;
  return r < 256 ? 256 : r;
}
// (at least one CTA: a rank without rows still publishes zero totals)
inline int reduce_blocks(int64_t n) {
  const int b = static_cast<int>((n + rows_per_block(n) - 1) / rows_per_block(n));
  return b < 1 ? 1 : b;
}

// The CG kernels run on fp32 (the tf32 engines' solver state) or fp64 vectors
// (the fp64 CG path over hv_f64); scalars are fp64 either way.
// out[c] = sum_i A[i,c] * B[i,c]  (fp64, fixed order), all columns.
template <class T>
void col_dots(const T* A, const T* B, int64_t ld, int64_t n, int s, double* part,
              unsigned* ticket, double* out, cudaStream_t st);

// CG: before the loop.  R = rhs - H X0 must already be in R; cg_init
// computes rs = ||r||^2, convergence and the loop-entry check (row-sharded:
// dist_finish(kDistInit)); cg_seed then sets P = R (active) / 0.
// pp (optional, fp32 only, here and in cg_direction): P's tf32 planes, written
// with P (hi at pp[j + c ld], lo at pp[j + (s + c) ld]; for HvParams::vplanes).
template <class T>
void cg_init(const T* R, int64_t ld, int64_t n, int s, ColState cs, double* part, SolveCtrl* ctrl,
             cudaStream_t st);
template <class T>
void cg_seed(T* P, const T* R, int64_t ld, int64_t n, int s, const int* conv, cudaStream_t st,
             float* pp = nullptr);
// alpha_c = rs_c / (p_c . hp_c); non-positive curvature -> kStatusNotPd.
template <class T>
void cg_alpha(const T* P, const T* HP, int64_t ld, int64_t n, int s, ColState cs,
              double* part, SolveCtrl* ctrl, cudaStream_t st);
// x += alpha p; r -= alpha hp (refresh=false) or x += alpha p only (refresh=true).
template <class T>
void cg_update(T* X, T* R, const T* P, const T* HP, int64_t ld, int64_t n, int s,
               ColState cs, double* part, SolveCtrl* ctrl, bool refresh, cudaStream_t st);
// refresh: r = rtmp for active columns; then ||r||^2, convergence, beta.
template <class T>
void cg_refresh_norm(T* R, const T* Rtmp, int64_t ld, int64_t n, int s, ColState cs,
                     double* part, SolveCtrl* ctrl, cudaStream_t st);
// Refresh steps: per column, act 1 copies X, R -> Xb, Rb (new best iterate),
// act 2 copies Xb, Rb -> X, R (stalled column restored to its best).
template <class T>
void cg_snapshot(T* X, T* R, T* Xb, T* Rb, int64_t ld, int64_t n, int s, ColState cs,
                 const SolveCtrl* ctrl, bool at_start, cudaStream_t st);
// p = r + beta p (active) / 0 (just converged); then the next-iteration check.
template <class T>
void cg_direction(T* P, const T* R, int64_t ld, int64_t n, int s, ColState cs,
                  double* part, SolveCtrl* ctrl, cudaStream_t st, float* pp = nullptr);
// One non-refresh CG iteration's vector work in ONE cooperative kernel:
// cg_alpha + cg_update + cg_direction (solvers.cpp:112-134) with two grid
// barriers; every CTA forms the column totals itself from the per-CTA
// partials in the same fixed order, so results are bitwise those of the
// three kernels.  Unsharded solves only.  Returns false (nothing launched)
// when the cooperative launch is unavailable; the caller then runs the three.
// fp64 H.V split partials for cg_fused to sum first (hv64_reduce_kernel's
// sum: part[(k s + c) m_pad + r] over k < splits, in order, + hyp[2] P, for
// the CTA's own rows and columns: one launch fewer per iteration);
// part == nullptr: HP is already formed.
struct HvFold {
  const double* part = nullptr;
  int splits = 0;
  int64_t m_pad = 0;
  const float* hyp = nullptr;
};
template <class T>
bool cg_fused(T* X, T* R, T* P, T* HP, int64_t ld, int64_t n, int s, ColState cs, double* part,
              SolveCtrl* ctrl, cudaStream_t st, float* pp, HvFold fold = HvFold());
// B = A (fp32 -> fp64) / B = A rounded to fp32, n x s column blocks.
void widen(const float* A, int64_t lda, double* B, int64_t ldb, int64_t n, int s, cudaStream_t st);
// out = A - B (n x s column blocks, leading dimension ld; float or double).
template <class T>
void diff_cols(const T* A, const T* B, T* out, int64_t ld, int64_t n, int s, cudaStream_t st);
// Y += a X (fp64, n x s column blocks, leading dimension ld).
void axpy_cols(double a, const double* X, double* Y, int64_t ld, int64_t n, int s, cudaStream_t st);
void narrow(const double* A, int64_t lda, float* B, int64_t ldb, int64_t n, int s, cudaStream_t st);
// out[i + c size] = R[start + i + c ld] for rows start + i in [own0, own1), 0 elsewhere
// (a rank's share of an AP block residual, row-sharded AP).
void masked_rows(const float* R, int64_t ld, int64_t start, int64_t size, int64_t own0, int64_t own1, int s,
                 float* out, const SolveCtrl* ctrl, cudaStream_t st);
// B[i + c size] = (double) A[i + c size] for an AP block (size x s, contiguous).
void widen_block(const float* A, double* B, int64_t size, int s, const SolveCtrl* ctrl, cudaStream_t st);

// Convergence from exact residual norms (AP epochs, SGD init): conv_c =
// bnorm_c == 0 || ||R_c|| <= tol_c bnorm_c; NaN -> kStatusNaN (when check_nan);
// then the loop check (all converged or it >= max_it -> done, else ++it).
void norms_convergence(const float* R, int64_t ld, int64_t n, int s, ColState cs, double* part,
                       SolveCtrl* ctrl, bool check_nan, bool begin_next, cudaStream_t st);

// AP block step helpers.
void ap_gather(const float* R, int64_t ld, int64_t start, int64_t b, int s, double* Rb,
               const SolveCtrl* ctrl, cudaStream_t st);
// X[start:start+b] += delta, and dx[start:start+b] = delta (fp32, same ld as X);
// dxp (optional): the tf32 hi / lo planes of dx (hi at dxp[j + c ld], lo at
// dxp[j + (s + c) ld]), for hv with HvParams::vplanes.
// delta: kparts partials of b x s (ld b) at stride b s, summed in fixed order.
void ap_apply(float* X, int64_t ld, int64_t start, int64_t b, int s, const double* delta, int kparts,
              float* dx, float* dxp, const SolveCtrl* ctrl, cudaStream_t st);
// nb contiguous b x b identity matrices (fp64, column-major).
void identities(double* A, int64_t b, int64_t nb, cudaStream_t st);
// H[b, b] in fp64 from the prepared points, padded with the identity to full x full.
void build_block(const float* xs, int dp, int64_t start, int64_t b, int64_t full, double sf2, double a,
                 double noise2, double* out, cudaStream_t st);

// SGD: vel/X/R row scatter (proj/src/solvers.cpp:247-252) then divergence and
// convergence on the stored residual estimate (:254-258).
// xp (optional): X's tf32 hi / lo planes (tf32_planes layout), updated with X.
void sgd_scatter(float* X, float* R, float* vel, int64_t ld, const int* idx, int64_t m, int s,
                 const float* batch, float momentum, float grad_scale, float step_scale, float* xp,
                 const SolveCtrl* ctrl, cudaStream_t st);
// xp[j + c ld] = tf32 hi of X[j + c ld], xp[j + (s + c) ld] = the lo part
// (bitwise hv_tc's split of V; for HvParams::vplanes).
void tf32_planes(const float* X, int64_t ld, int64_t n, int s, float* xp, cudaStream_t st);
// One SGD step's vector work in one kernel: the momentum scatter of
// sgd_scatter, then the residual-estimate norms ||R_c||^2 (cs.rs) and ||X||_F^2
// (*xsq) updated by the minibatch rows' changes (fp64, fixed order; the
// minibatch rows are distinct), and sgd_check's convergence / divergence
// tests and loop check on them.  part: >= ceil(m / 256) * (s + 1) doubles.
void sgd_step(float* X, float* R, float* vel, int64_t ld, const int* idx, int64_t m, int s, const float* batch,
              float momentum, float grad_scale, float step_scale, float* xp, ColState cs, double* xsq,
              double* part, SolveCtrl* ctrl, cudaStream_t st);
// Exact ||R_c||^2 -> cs.rs and ||X||_F^2 -> *xsq (no convergence or loop
// check): re-synchronises sgd_step's running norms once per round.
void sgd_norms(const float* X, const float* R, int64_t ld, int64_t n, int s, ColState cs, double* xsq,
               double* part, SolveCtrl* ctrl, cudaStream_t st);
void sgd_check(const float* X, const float* R, int64_t ld, int64_t n, int s, ColState cs,
               double* part, SolveCtrl* ctrl, cudaStream_t st);

// Small helpers.
void fill_zero(float* A, int64_t ld, int64_t n, int s, cudaStream_t st);
void sub_into(const float* A, const float* B, float* out, int64_t ld, int64_t n, int s,
              cudaStream_t st);  // out = A - B
void copy_cols(const float* A, int64_t lda, float* B, int64_t ldb, int64_t n, int s,
               cudaStream_t st);

}  // namespace wgp
