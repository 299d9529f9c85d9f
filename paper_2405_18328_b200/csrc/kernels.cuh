// kernels.cuh — launch interfaces of the warmgp B200 device kernels.
//
// Point layout in HBM: the n x d inputs are
// stored once per hyperparameter setting as `xs`, row-major [n_pad][dp]
// fp32, centred and scaled per dimension by sqrt(3) log2(e) / lengthscale_k, so
// the squared Euclidean distance of two rows is u^2 with
// u = sqrt(3) log2(e) r and k = sf^2 (1 + u ln2) 2^-u.  Right-hand sides and
// solver state are column-major [s][ld] fp32 (Eigen's layout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wgp {

enum HvMode : int {
  kHvStore = 0,     // out[r, c]  = (H V)[row, c]
  kHvResidual = 1,  // out[r, c]  = B[row, c] - (H V)[row, c]
  kHvSubtract = 2,  // out[r, c] -= (H V)[row, c]
};

struct HvParams {
  const float* xs;       // [n_pad][dp] prepared points
  int64_t n;             // number of points
  int dp;                // padded dimension (row stride of xs)
  const int* row_idx;    // optional gather of output rows (global indices)
  int64_t r0;            // first global output row when row_idx == nullptr
  int64_t m;             // number of output rows
  int64_t j0, j1;        // contracted points [j0, j1)
  const float* V;        // V[j + c * ldv] for global j
  int64_t ldv;
  int s;                 // columns
  float* out;            // out[r + c * ldo], r = local output row
  int64_t ldo;
  const float* B;        // residual mode: B[row + c * ldb], row = global
  int64_t ldb;
  int mode;
  float sf2;             // signal^2
  float a;               // sf^2 ln 2
  float noise2;          // sigma^2
  float diag;            // sf^2 + sigma^2: the diagonal H_ii, applied in the epilogue
                         // (the streamed sum skips j == row so fp32 accumulation
                         // never carries the dominant diagonal term)
  const float* hyp;      // optional device [sf2, a, diag] overriding the three fields above
                         // (lets a captured CUDA graph follow hyperparameter changes)
  const int* done;       // optional device flag: skip the launch body when *done != 0
  int64_t split_rows;    // rows that key the J-split decomposition (0: m).  Row shards
                         // pass the global row count so every shard sums in the same
                         // order as the single-GPU launch (bitwise identical rows).
  const float* vplanes;  // optional caller-maintained tf32 planes of V (hv_tc, s <= 96):
  int64_t vplanes_ld;    // hi[j + c ld], lo[j + (s + c) ld] for global j, bitwise
                         // split_v's; the launch then skips its own split of V
  bool reuse_vsplit;     // hv_tc: the previous launch split this same V[j0:j1, :s] (row
                         // chunks of one product, wgp_hv): skip the split, reuse its planes
  const float* v_host;   // hv_tc: optional device-visible alias of the caller's page-locked V
                         // (same ldv).  The split then loads V over PCIe itself and
                         // stores what it read into V (a device buffer here), instead of
                         // a copy-engine upload before the launch (wgp_hv, zero-copy)
};

// SIMT fp32 fused H.V (direct differences; any d, s <= 128).
void hv_simt(const HvParams& p, cudaStream_t st);

// tcgen05 3xTF32 fused H.V (s <= 128 after padding; d <= 29).  Returns false
// if the shape is unsupported (caller falls back to the SIMT CUDA kernel).
struct TcPoints;  // prepared operand set, see hv_tc.cu
bool hv_tc_supported(int d, int s);
double hv_tc_model_cost(int64_t m, int64_t nv, int s, bool f16);

// Gradient contractions.  W_ij = 1/2 vy_i vy_j (A) and
// coef_b sum_c L_ic R_jc (B).  Writes per-block fp64 partials
//   part[blk][0..d]    : A contractions (d lengthscale sums, 1 signal sum)
//   part[blk][d+1..]   : B contractions
// summed in fixed order by grad_finalize.
struct GradParams {
  const float* xs;
  int64_t n;
  int dp, d;
  const float* vy;
  const float* L;
  const float* R;
  int64_t ld;
  int s;
  float coef_b;
  float sf2, a;
  double* part;   // [gridDim.x][2 (d+1)]
  int64_t r0 = 0, m = -1;  // rows [r0, r0 + m) against all n points (m < 0: all rows)
};
int grad_blocks(int64_t m);  // rows
void grad_simt(const GradParams& p, cudaStream_t st);
// Tensor-core gradient (grad_tc.cu): W^B on tcgen05, O(d) epilogue; same
// partial format as grad_simt ([plan.nblk][2 (d + 1)]).
struct GradTcPlan {
  int64_t n_pad = 0;
  int spk = 0, ep = 0, splits = 1, nblk = 0;
  int cs = 1, rt_pad = 0;  // cluster size sharing the R stream, row tiles padded to it
  size_t ws_bytes = 0;
};
bool grad_tc_supported(int d, int s);
GradTcPlan grad_tc_plan(int64_t n, int64_t m, int d, int s);  // n points, m rows
void grad_tc(const GradParams& p, const GradTcPlan& plan, void* ws, cudaStream_t st);
// out[0..2(d+1)) = sum over blocks in block order.
void grad_finalize(const double* part, int nblk, int width, double* out, cudaStream_t st);

// Pathwise RFF probes: out[i + j ld] = amp sum_f w[f + j F] cos(b_f + om_f . x_i) + sigma eps[i + j ld]
struct RffParams {
  const float* x;       // raw inputs, column-major [d][n] (x[i + k n])
  int64_t n;
  int d;
  const double* om;     // F x d row-major, omega / lengthscale (fp64)
  const double* b;      // F
  const float* w;       // F x s column-major
  const float* eps;     // ld x s
  int F, s;
  int64_t ld;
  float amp, sigma;
  float* out;
};
void rff_probes(const RffParams& p, cudaStream_t st);

// Cross kernel matrix K*[j + i ld] = k(x_j, x*_i) (train j < n, test i < m) from
// prepared points; rows n..ld-1 are zero (predict.cu).
void cross_matrix(const float* xs, int64_t n, const float* xt, int64_t m, int dp, float sf2, float a, float* out,
                  int64_t ld, cudaStream_t st);
// out[i] = K*[:, i] . alpha in fp64.
void colvec_dots(const float* K, int64_t ld, int64_t n, int64_t m, const float* alpha, double* out,
                 cudaStream_t st);

// Prepare xs from column-major raw X: xs[i][k] = (X[i,k] - mu_k) * scale_k.
void prepare_points(const float* X, int64_t n, int d, const double* mu, const double* scale,
                    float* xs, int64_t n_pad, int dp, cudaStream_t st);

}  // namespace wgp
