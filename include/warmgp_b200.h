/*
 * warmgp_b200.h — C-ABI of the B200-native iterative-GP hot path.
 *
 * This is the drop-in boundary that replaces the dense-Eigen hot path of the
 * reference library `warmgp` (/root/reference/proj).  Every entry point below
 * names the reference interface it replaces (file:line); INTEGRATION.md shows
 * the C++ adapter and the ctypes stub that bind it.
 *
 * Conventions:
 *   - plain pointers and sizes only; matrices are column-major like
 *     Eigen::MatrixXd (element (i, c) at ptr[i + c * ld]); `*_host` entry points
 *     take host memory, `*_device` ones take device memory on the context's GPU;
 *   - status codes mirror the reference's exception -> exit-code mapping
 *     (proj/tools/main.cpp:336-358): 0 ok, 2 std::invalid_argument,
 *     3 NumericalError, 4 device / IO error; wgp_last_error() returns the
 *     thread-local message, carrying the reference's message text
 *     ("...not positive definite", "...use a smaller learning rate", "step N: ...");
 *   - one context per thread/stream; the library owns all device buffers,
 *     including the warm-start state; there is NO CPU fallback: without a
 *     B200 every compute entry point returns 4.
 */
#ifndef WARMGP_B200_H
#define WARMGP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WGP_OK 0
#define WGP_INVALID 2
#define WGP_NUMERICAL 3
#define WGP_DEVICE 4

typedef struct wgp_ctx wgp_ctx;

/* Hyperparameter transform: 0 softplus (kernel.cpp:14-31), 1 log (BASELINE). */
#define WGP_TRANSFORM_SOFTPLUS 0
#define WGP_TRANSFORM_LOG 1
/* Solver kinds: solvers.hpp:13 SolverKind {Cg, Ap, Sgd}. */
#define WGP_SOLVER_CG 0
#define WGP_SOLVER_AP 1
#define WGP_SOLVER_SGD 2
/* H.V implementation (all: fp32 accumulation in chunks of 1024 points summed
 * at higher precision, so the error does not grow with n):
 *   WGP_HV_TC       tcgen05, Gram and K.V in 3xTF32 (default, ~1e-6 relative)
 *   WGP_HV_SIMT     CUDA-core fp32 kernel (direct differences, ~1e-7)
 *   WGP_HV_TC_F16   tcgen05, K.V in fp16x3 over column-scaled V (half the
 *                   K.V tensor work of 3xTF32, the same 22-bit operand split) */
#define WGP_HV_TC 0
#define WGP_HV_SIMT 1
#define WGP_HV_TC_F16 2
/* Precision of CG's solver state and operator (proj/src/solvers.cpp:81-139):
 *   WGP_CG_F64  fp64 x / r / p / Hp over the fp64-accumulating symmetric
 *               operator (hv_f64.cu): iteration counts of the fp64 reference
 *               (default)
 *   WGP_CG_F32  fp32 vectors over the selected fp32 H.V engine (faster; needs
 *               up to ~40% more iterations on ill-conditioned systems) */
#define WGP_CG_F64 0
#define WGP_CG_F32 1

/** Thread-local message of the last failing call. */
const char* wgp_last_error(void);
/** Library version string, build flags and the compiled sm target. */
const char* wgp_version(void);
/** Number of visible CUDA devices (0 on a GPU-less host; never an error). */
int wgp_device_count(void);
/** Kernels launched by this library in this process so far (all contexts). */
uint64_t wgp_launch_count(void);

/** Create a context on `device`.  Replaces nothing in the reference (which
 *  has no device); owns the stream, workspaces and warm-start buffers. */
int wgp_create(int device, wgp_ctx** out);
int wgp_destroy(wgp_ctx* ctx);
/** Select the H.V kernel (WGP_HV_TC / WGP_HV_SIMT). */
int wgp_set_hv_impl(wgp_ctx* ctx, int impl);
/** Select CG's precision (WGP_CG_F64 / WGP_CG_F32); AP and SGD always run
 *  on fp32 state over the selected H.V engine. */
int wgp_set_cg_precision(wgp_ctx* ctx, int precision);
/** The cudaStream_t the context launches on (for event timing by callers). */
void* wgp_stream(wgp_ctx* ctx);
/** Kernel timing: while enabled, CUDA events bracket every tensor-core H.V
 *  kernel launch on the context stream; wgp_profile_read syncs, returns the
 *  summed kernel time (ms) and launch count since the last read, and resets. */
int wgp_profile(wgp_ctx* ctx, int enable);
int wgp_profile_read(wgp_ctx* ctx, double* kernel_ms, int* launches);

/** Upload the n x d training inputs (host, column-major fp32).  Replaces the
 *  X argument of build_kernel_matrices (proj/src/kernel.cpp:120-139): the
 *  B200 path never materialises H. */
int wgp_set_data(wgp_ctx* ctx, const float* X_host, int64_t n, int d);
/** Constrained hyperparameters [lengthscales(d), signal, noise]
 *  (Hyperparameters::to_constrained_vector, proj/src/kernel.cpp:70-76). */
int wgp_set_hyper(wgp_ctx* ctx, const double* constrained);
/** Restrict H.V outputs to rows [r0, r1) (row-block sharding);
 *  default is all rows.  Inputs V always span all n rows. */
int wgp_set_rows(wgp_ctx* ctx, int64_t r0, int64_t r1);

/** out = H V = (K + sigma^2 I) V, V/out n x s (host).  Replaces the dense
 *  products H * P / H * X at proj/src/solvers.cpp:71,92,110,120,169,188,211
 *  and proj/src/estimator.cpp:90.  On the tcgen05 engines from
 *  8192 rows the result's download overlaps the launches (row chunks, each
 *  chunk's copy under the next chunk; WGP_HV_PIPE=1 turns it off): rows then
 *  equal wgp_hv_device's one-launch product to fp32 rounding, not bitwise.
 *  Page-locked host buffers (cudaHostAlloc / cudaHostRegister) make the copies
 *  asynchronous, and on the tcgen05 engines (s <= 96, V of 1 MB or more) a
 *  page-locked V is not copied at all: the V split kernel loads it over PCIe
 *  itself (bitwise the same result; steadier than the copy engine on hosts
 *  whose DMA read rate dips; WGP_HV_UPLOAD=ce|zc|auto), and the
 *  last row chunk is stored straight into a page-locked out_host
 *  (WGP_HV_DOWNLOAD=ce: copied).  V_host is only read. */
int wgp_hv(wgp_ctx* ctx, const float* V_host, int s, float* out_host);
/** fp64 H V on host fp64 V / out (n x s; rows of wgp_set_rows): the operator
 *  of the fp64 CG path -- entries evaluated in fp32 (bitwise symmetric),
 *  products and sums in fp64.  The Eigen::MatrixXd-facing form of the
 *  products H * X the reference writes in fp64 (same sites as wgp_hv). */
int wgp_hv_f64(wgp_ctx* ctx, const double* V_host, int s, double* out_host);
/** Device-pointer variant; `stream` may be NULL (context stream). */
int wgp_hv_device(wgp_ctx* ctx, const float* V, int64_t ldv, int s, float* out, int64_t ldo);

/* SolverConfig, proj/include/warmgp/solvers.hpp:20-32 (same defaults). */
typedef struct {
  int kind;
  double tol_mean;
  double tol_samples;
  int max_iterations;
  int block_size;
  int minibatch_size;
  double momentum;
  double learning_rate;
  uint64_t seed;
} wgp_solver_cfg;

/* SolveState, proj/include/warmgp/solvers.hpp:38-46 (caller-owned arrays). */
typedef struct {
  float* solutions;                      /* n x s */
  float* residuals;                      /* n x s, solver-tracked */
  double* per_column_relative_residual;  /* s, exact at exit */
  int* converged;                        /* s */
  int iterations_used;
} wgp_solve_state;

/** solve(H, rhs, init, config) (proj/src/solvers.cpp:265-279) with H given
 *  matrix-free by the context's X and hyperparameters.  rhs/init host n x s
 *  (init may be NULL = zeros). */
int wgp_solve(wgp_ctx* ctx, const wgp_solver_cfg* cfg, const float* rhs, const float* init, int s,
              wgp_solve_state* state);

/* SolveState in fp64 (the reference's MatrixXd / VectorXd members). */
typedef struct {
  double* solutions;                     /* n x s */
  double* residuals;                     /* n x s, solver-tracked */
  double* per_column_relative_residual;  /* s, exact at exit */
  int* converged;                        /* s */
  int iterations_used;
} wgp_solve_state_f64;

/** wgp_solve for fp64 host buffers (Eigen::MatrixXd's column-major storage:
 *  rhs.data(), init.data()).  With fp64 CG (WGP_CG_F64, the default) the fp64
 *  init and the fp64 solutions pass through unrounded; AP / SGD run on fp32
 *  state (rounded in, widened out). */
int wgp_solve_f64(wgp_ctx* ctx, const wgp_solver_cfg* cfg, const double* rhs, const double* init, int s,
                  wgp_solve_state_f64* state);

/** derivative_contractions (proj/src/kernel.cpp:216-252) for the estimator's
 *  low-rank contractions (proj/src/estimator.cpp:63-82):
 *     A = 1/2 vy vy^T,  B = coef_b L R^T      (vy: n, L/R: n x s; host)
 *  out_a/out_b (d+2): raw-space <dH/dtheta_k, A>, <dH/dtheta_k, B>, with the
 *  chain rule of `transform` at `raw`.  Uses the context's X; the context's
 *  hyperparameters are set from `raw`.  The row sums run over the context's
 *  row range (wgp_set_rows; default all rows) against all n points: the
 *  outputs of a row partition add up to the full contraction (row sharding). */
int wgp_grad(wgp_ctx* ctx, int transform, const double* raw, const float* vy, const float* L,
             const float* R, int s, double coef_b, double* out_a, double* out_b);

/** sample_probes (proj/src/estimator.cpp:21-37): host mt19937_64, bitwise the
 *  reference's values (then rounded to fp32).  dist 0 gaussian, 1 rademacher. */
int wgp_sample_probes(int64_t n, int s, int dist, uint64_t seed, float* out_host);

/** Pathwise prior-sample probes (BASELINE a12, not in the reference):
 *  z_j(x_i) = sf sqrt(2/F) sum_f w_fj cos(omega_f . x_i/ls + b_f) + sigma eps_ij,
 *  base randomness drawn on the host from mt19937_64(seed) exactly like the
 *  oracle (omega_z, chi2_3, b, w, eps order), evaluated on the GPU at the
 *  context's hyperparameters.  out host n x s. */
int wgp_rff_probes(wgp_ctx* ctx, int F, int s, uint64_t seed, float* out_host);

/* TrainConfig, proj/include/warmgp/optimizer.hpp:23-38, plus BASELINE fields. */
typedef struct {
  int steps;
  double learning_rate;
  double adam_beta1;
  double adam_beta2;
  double adam_eps;
  int num_probes;
  int probe_distribution; /* 0 gaussian, 1 rademacher */
  int mode;               /* 0 warm, 1 cold (resampled), 2 cold-fixed (TrainMode) */
  wgp_solver_cfg solver;
  double init_constrained;
  uint64_t seed;
  int transform;          /* WGP_TRANSFORM_* */
  int estimator;          /* 0 hutchinson (reference), 1 pathwise RFF */
  int rff_features;
  double init_noise;      /* <= 0: init_constrained */
  double init_signal;     /* <= 0: init_constrained */
  int warm_start_distance;/* 1: compute the diagnostic (+1 H.V per warm step) */
  int exact_gradients;    /* 1: train_exact (optimizer.hpp:83-86): exact Cholesky gradient */
  int record_solver_state;/* 1: fill wgp_trace::solver_init / solver_solutions (optimizer.hpp:35) */
} wgp_train_cfg;

/* StepRecord fields (proj/include/warmgp/optimizer.hpp:54-67), caller-owned,
 * any pointer may be NULL. */
typedef struct {
  double* raw_params;          /* steps x p (row per step) */
  double* constrained_params;  /* steps x p */
  double* gradient;            /* steps x p */
  int* solver_iterations;      /* steps */
  double* per_column_relative_residual; /* steps x (num_probes + 1) */
  double* warm_start_distance; /* steps */
  uint64_t* probe_seed;        /* steps */
  double* solver_ms;           /* steps: device time of the solve */
  double* step_ms;             /* steps: device time of the whole outer step */
  float* final_solutions;      /* n x (num_probes + 1) */
  double* warm_distance_ms;    /* steps: device time of the warm-start-distance H.V
                                  (included in step_ms; step_ms - this = the step without it) */
  float* solver_init;          /* steps x n x (num_probes + 1), with record_solver_state
                                  (StepRecord::solver_init, optimizer.hpp:65) */
  float* solver_solutions;     /* steps x n x (num_probes + 1) (StepRecord::solver_solutions, :66) */
} wgp_trace;

/** train(X, y, config) (proj/src/optimizer.cpp:175-177, run_loop :81-171):
 *  the full outer loop on the device — solves warm-started from the
 *  device-resident previous solutions, gradients, Adam on the host.
 *  Uses the context's data (wgp_set_data); y host n. */
int wgp_train(wgp_ctx* ctx, const float* y_host, const wgp_train_cfg* cfg, wgp_trace* trace);

/** exact_mll / exact_gradient (proj/src/exact.cpp:25-50) in fp64 on the device
 *  (dense H, cuSOLVER Cholesky; n <= 20000 = kDenseGuard, exact.hpp:23) for the
 *  context's data, y host n, raw (d+2) in `transform`'s space.  mll / grad
 *  (raw-space gradient, d+2) may be NULL; errors as the reference's
 *  ("...: system matrix is not positive definite", "...: n exceeds the dense guard"). */
int wgp_exact(wgp_ctx* ctx, int transform, const double* raw, const float* y, double* mll, double* grad);

/** predict(X_train, y, X_test, hyper) (proj/src/exact.cpp:52-77) through
 *  iterative solves with `cfg` for the context's data and hyperparameters:
 *  X_test host column-major m x d, y host n; means / variances (latent) host m;
 *  noise_variance may be NULL.  Beyond the dense guard (no n limit). */
int wgp_predict(wgp_ctx* ctx, const float* X_test, int64_t m, const float* y, const wgp_solver_cfg* cfg,
                double* means, double* variances, double* noise_variance);

/** adam_step (proj/src/optimizer.cpp:48-65). */
int wgp_adam_step(double* raw, const double* grad, double* m, double* v, int p, int t,
                  double lr, double beta1, double beta2, double eps);

/** Utilities of the reference's common.hpp:25-36. */
uint64_t wgp_derive_seed(uint64_t base, uint64_t stream);

/** Row permutation of split_standardize (proj/src/dataset.cpp:118-124):
 *  order = 0..n-1 shuffled by Fisher-Yates from the back with
 *  mt19937_64(derive_seed(split_seed, 0x5b117)) and uniform_below -- bitwise
 *  the reference's permutation (host-only, no device work). */
int wgp_split_order(int64_t n, uint64_t split_seed, int64_t* order);

/* ---- row sharding inside the library: one process per GPU, NCCL ----
 * Every rank creates a context on its GPU and attaches a communicator before
 * wgp_set_data (all ranks pass the same full inputs).  Rank r then owns rows
 * [own0, own1) = [r blk, (r + 1) blk) of every solver vector (blk = the
 * 128-row tiles dealt in contiguous blocks); vectors keep all rows (leading
 * dimension nranks blk), so the exchanges are in-place all-gathers:
 *   wgp_hv / wgp_hv_f64 / wgp_hv_device: the rank's rows of H V, then the
 *     all-gather of the n x s result;
 *   wgp_solve (CG, AP; SGD is single-GPU): CG all-gathers the direction every
 *     iteration and finishes its column reductions on the ranks' rank-order
 *     sums; AP sums each block's residual shares with an all-reduce; the
 *     solutions end with all rows on every rank (these collectives are
 *     captured into the CG / AP CUDA graphs);
 *   wgp_grad, wgp_train: the rank's rows of every contraction, summed over
 *     the ranks; the outer loop (Adam) runs identically on every rank.
 * Without wgp_set_comm nothing changes (the whole operator on one GPU). */
/** ncclGetUniqueId (rank 0 calls it and broadcasts the 128 bytes). */
int wgp_nccl_unique_id(unsigned char id[128]);
/** Attach a communicator (ncclCommInitRank; collective over the ranks) to the
 *  context; wgp_set_data must follow. */
int wgp_set_comm(wgp_ctx* ctx, int rank, int nranks, const unsigned char id[128]);
/** TEST INFRASTRUCTURE: a host-mediated communicator for N contexts on ONE
 *  GPU driven by N host threads (each collective: a host barrier and device
 *  copies between the contexts' buffers; no kernel waits on another rank's, no
 *  CUDA graphs).  It runs the library's multi-rank sharding logic where only
 *  one GPU is available; production uses wgp_set_comm (NCCL). */
typedef struct wgp_local_group wgp_local_group;
int wgp_local_group_create(int nranks, wgp_local_group** out);
int wgp_local_group_destroy(wgp_local_group* g);
int wgp_set_comm_local(wgp_ctx* ctx, wgp_local_group* g, int rank);
/** The context's rank, rank count, own rows and vector leading dimension. */
int wgp_shard_info(wgp_ctx* ctx, int* rank, int* nranks, int64_t* own0, int64_t* own1, int64_t* ld);
/** The row partition of n points over nranks (host only): own rows and ld. */
int wgp_shard_rows(int64_t n, int rank, int nranks, int64_t* own0, int64_t* own1, int64_t* ld);

/* ---- row-sharded solver building blocks for callers driving their own exchanges
 *      (paper_2405_18328_b200/sharded.py, torch.distributed) ---- */

/** J-split decomposition of the fused H.V for a row range: keyed on the global
 *  n (global != 0, the default: a row shard reproduces the full operator's rows
 *  bitwise at any GPU count) or on the shard's own rows (global == 0: more
 *  CTAs per GPU on small shards; rows equal to fp32 rounding). */
int wgp_set_split_global(wgp_ctx* ctx, int global);

/** out[r, :] (rows r of the context's row range, wgp_set_rows) =
 *  mode 0: H[row, j0:j1] V[j0:j1, :];  1: B[row, :] - (that);  2: out -= (that).
 *  V holds the block's rows (V[(j - j0) + c ldv], ldv >= j1 - j0), B and out
 *  the context's rows (B[(row - r0) + c ldb]).  Device pointers.
 *  The column block of the right-looking AP residual update
 *  R_I -= H[I, b] delta_b (proj/src/solvers.cpp:186). */
int wgp_hv_cols(wgp_ctx* ctx, const float* V, int64_t ldv, int s, int64_t j0, int64_t j1, float* out, int64_t ldo,
                int mode, const float* B, int64_t ldb);
/** out = H[i0:i1, j0:j1] V for any block of the full operator (independent of
 *  wgp_set_rows): V holds rows j0..j1-1 (V[(j - j0) + c ldv]), out rows
 *  i0..i1-1 (out[(i - i0) + c ldo]); the diagonal term where the ranges
 *  overlap.  Device pointers; J splits keyed on the block's own rows.  The
 *  row-sharded AP's block residual R_b = R0_b - sum over ranks of
 *  H[b, own columns before b] dX (proj/src/solvers.cpp:186 applied lazily). */
int wgp_hv_block(wgp_ctx* ctx, int64_t i0, int64_t i1, int64_t j0, int64_t j1, const float* V, int64_t ldv, int s,
                 float* out, int64_t ldo);
/** Factor every diagonal block of size block_size at the current
 *  hyperparameters (proj/src/solvers.cpp:151-165: Cholesky, errors as
 *  ap_solve's) and keep the inverses; *nblocks = ceil(n / block_size). */
int wgp_ap_factor(wgp_ctx* ctx, int block_size, int64_t* nblocks);
/** delta_b = H_bb^-1 R_b for block b of the last wgp_ap_factor
 *  (proj/src/solvers.cpp:185); device fp64, column-major size x s, ld = size. */
int wgp_ap_block_solve(wgp_ctx* ctx, int64_t block, const double* Rb, int s, double* delta);

#ifdef __cplusplus
}
#endif
#endif
