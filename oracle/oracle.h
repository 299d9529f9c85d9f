/*
 * oracle.h — CPU parity oracle for the warm-started iterative-GP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2405_18328_b200/ links, loads or
 * calls this library; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker or as the
 * timed CPU baseline.
 *
 * It is a from-scratch fp64 restatement of the reference library `warmgp`
 * (/root/reference/proj, C++20 + Eigen, unbuildable here: Eigen3 and vendor/
 * are absent, proj/CMakeLists.txt:10-11).  Every entry point cites the
 * reference function it follows.  Matrices are column-major doubles, as
 * Eigen::MatrixXd in the reference.
 *
 * Parity pin: the reference ships no golden vectors.  The
 * oracle is pinned by (a) every known-answer / closed-form / property test of
 * the reference's hot-path suites (kernel_test.cpp, solvers_test.cpp,
 * estimator_test.cpp, optimizer_test.cpp, acceptance C1/C2/C4) re-run against
 * it in tests/test_oracle_*.py, and (b) an independent dense numpy
 * restatement (oracle/dense_ref.py) of the reference's Eigen expressions.
 * Everything BASELINE.json adds beyond the reference (log transform, pathwise
 * RFF probes, separate sigma_0, config generators) is "parity unpinned": the
 * oracle defines it.
 */
#ifndef WARMGP_ORACLE_H
#define WARMGP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes, mirroring the reference's exit-code mapping
 * (proj/tools/main.cpp:336-358): 2 invalid argument, 3 NumericalError. */
#define OR_OK 0
#define OR_INVALID 2
#define OR_NUMERICAL 3

const char* or_last_error(void);

/* common.hpp:25-52 */
uint64_t or_splitmix64(uint64_t x);
uint64_t or_derive_seed(uint64_t base, uint64_t stream);
int or_split_order(int64_t n, uint64_t split_seed, int64_t* order);  // dataset.cpp:118-124
int or_synthesize_draws(int n, int d, uint64_t seed, double* X, double* xi);  // dataset.cpp:167-190

/* kernel.cpp:14-31 (softplus) plus the log transform BASELINE asks for.
 * transform: 0 = softplus (reference), 1 = log. */
double or_softplus(double x);
double or_softplus_inverse(double v);
double or_softplus_derivative(double x);
double or_to_constrained(int transform, double raw);
double or_to_raw(int transform, double constrained);
double or_chain(int transform, double raw);

/* kernel.cpp:79-93: one Matern-3/2 ARD value (constrained hyperparameters). */
double or_matern32(const double* x, const double* x2, int d, const double* ls, double sf);

/* kernel.cpp:120-139: dense system / kernel / decay matrices (n x n, column
 * major).  Any output pointer may be NULL. */
int or_build_kernel_matrices(const double* X, int64_t n, int d, const double* ls, double sf,
                             double sigma, double* system, double* kernel, double* decay);

/* Matrix-free H V = K V + sigma^2 V (the dense product at solvers.cpp:110 with
 * H evaluated per entry like scaled_sqdist, kernel.cpp:101-116).  V, out: n x s. */
int or_hv(const double* X, int64_t n, int d, const double* ls, double sf, double sigma,
          const double* V, int s, double* out, int nthreads);

/* Rows [r0, r1) of H V only (bounded CPU baseline sample); out is (r1-r0) x s. */
int or_hv_rows(const double* X, int64_t n, int d, const double* ls, double sf, double sigma,
               const double* V, int s, int64_t r0, int64_t r1, double* out, int nthreads);

/* Dense H * V for a prebuilt H (solvers.cpp:110 as Eigen evaluates it). */
int or_dense_matmul(const double* H, int64_t n, const double* V, int s, double* out, int nthreads);

/* Solver configuration, solvers.hpp:20-32. kind: 0 cg, 1 ap, 2 sgd. */
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
  /* 1: CG stores x, r, p and H p rounded to fp32 after every update (dots and
   * alpha/beta stay fp64) -- the arithmetic of the fp32 GPU path, used as the
   * reference for iteration-count parity.  0: the reference's fp64. */
  int f32_vectors;
} or_solver_cfg;

/* SolveState, solvers.hpp:38-46 (arrays supplied by the caller). */
typedef struct {
  double* solutions;        /* n x s */
  double* residuals;        /* n x s (solver-tracked) */
  double* per_column_relative_residual; /* s */
  int* converged;           /* s */
  int iterations_used;
} or_solve_state;

/* solvers.cpp:265-279 with H either dense (H != NULL) or matrix-free over X. */
int or_solve(const double* H, const double* X, int64_t n, int d, const double* ls, double sf,
             double sigma, const or_solver_cfg* cfg, const double* rhs, const double* init,
             int s, or_solve_state* state, int nthreads);

/* estimator.cpp:21-37. dist: 0 gaussian, 1 rademacher. out: n x s. */
int or_sample_probes(int64_t n, int s, int dist, uint64_t seed, double* out);

/* Pathwise probe base randomness (BASELINE a12; not in the reference).
 * omega_z F x d (f-major), chi2 F, phase_b F, w F x s (column major), eps n x s. */
int or_rff_base(int64_t n, int d, int F, int s, uint64_t seed, double* omega_z, double* chi2,
                double* phase_b, double* w, double* eps);
/* z_j(x_i) = sf sqrt(2/F) sum_f w_fj cos(omega_f . (x_i / ls) + b_f) + sigma eps_ij */
int or_rff_probes(const double* X, int64_t n, int d, const double* ls, double sf, double sigma,
                  int F, int s, const double* omega_z, const double* chi2, const double* phase_b,
                  const double* w, const double* eps, double* out, int nthreads);

/* derivative_contractions (kernel.cpp:216-252) for the low-rank contractions
 * the estimator builds (estimator.cpp:63-82):
 *   A = 1/2 vy vy^T,  B = coef_b * L R^T  (L, R: n x s)
 * out_a[p], out_b[p] are raw-space <dH/dtheta_k, A>, <dH/dtheta_k, B>. */
int or_grad_contractions(const double* X, int64_t n, int d, int transform, const double* raw,
                         const double* vy, const double* L, const double* R, int s, double coef_b,
                         double* out_a, double* out_b, int nthreads);

/* exact.cpp:36-50 (dense Cholesky gradient), exact.cpp:25-34 (MLL). */
int or_exact_gradient(const double* X, const double* y, int64_t n, int d, int transform,
                      const double* raw, double* grad, int nthreads);
int or_exact_mll(const double* X, const double* y, int64_t n, int d, int transform,
                 const double* raw, double* mll, int nthreads);

/* warm_start_distance, estimator.cpp:84-95 (matrix-free). */
int or_warm_start_distance(const double* X, int64_t n, int d, const double* ls, double sf,
                           double sigma, const double* init, const double* sol, int s,
                           double* out, int nthreads);

/* TrainConfig, optimizer.hpp:23-38, plus BASELINE extensions. */
typedef struct {
  int steps;
  double learning_rate;
  double adam_beta1;
  double adam_beta2;
  double adam_eps;
  int num_probes;
  int probe_distribution; /* 0 gaussian, 1 rademacher (hutchinson only) */
  int mode;               /* 0 warm, 1 cold (resampled), 2 cold-fixed */
  or_solver_cfg solver;
  double init_constrained;
  uint64_t seed;
  /* extensions */
  int transform;          /* 0 softplus (reference), 1 log */
  int estimator;          /* 0 hutchinson (reference), 1 pathwise RFF */
  int rff_features;
  double init_noise;      /* <= 0: use init_constrained */
  double init_signal;     /* <= 0: use init_constrained */
  int exact_gradients;    /* train_exact, optimizer.cpp:179-182 */
} or_train_cfg;

/* Per-step trace arrays (StepRecord, optimizer.hpp:54-67); all caller owned,
 * sized steps x p, steps, steps x (num_probes+1) ... Any pointer may be NULL. */
typedef struct {
  double* raw_params;        /* steps x p, row per step */
  double* constrained_params;
  double* gradient;
  int* solver_iterations;    /* steps */
  double* per_column_relative_residual; /* steps x (s+1) */
  double* warm_start_distance; /* steps */
  uint64_t* probe_seed;      /* steps */
  double* final_solutions;   /* n x (s+1) */
} or_trace;

int or_train(const double* X, const double* y, int64_t n, int d, const or_train_cfg* cfg,
             or_trace* trace, int nthreads);

/* adam_step, optimizer.cpp:48-65 */
int or_adam_step(double* raw, const double* grad, double* m, double* v, int p, int t,
                 double lr, double beta1, double beta2, double eps);

#ifdef __cplusplus
}
#endif
#endif
