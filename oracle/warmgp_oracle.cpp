// warmgp_oracle.cpp — CPU parity oracle (TEST INFRASTRUCTURE; see oracle.h).
//
// fp64 restatement of the reference `warmgp` hot path.  File:line citations
// refer to /root/reference/proj.  OpenMP parallelism is over output rows only,
// each row reduced in a fixed order, so results are bitwise independent of
// the thread count (the reference's determinism contract).

#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_last_error;

struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};

constexpr double kSqrt3 = 1.7320508075688772;
constexpr double kLog2Pi = 1.8378770664093453;
constexpr uint64_t kSolverStream = 0x736f6c7665ULL;  // optimizer.cpp:15

template <class F>
int guarded(F&& f) {
  try {
    f();
    return OR_OK;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return OR_NUMERICAL;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return OR_INVALID;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return OR_INVALID;
  }
}

void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

// common.hpp:40-47
uint64_t uniform_below(std::mt19937_64& rng, uint64_t bound) {
  const uint64_t limit = std::numeric_limits<uint64_t>::max() -
                         std::numeric_limits<uint64_t>::max() % bound;
  uint64_t v;
  do {
    v = rng();
  } while (v >= limit);
  return v % bound;
}

// common.hpp:50-52
double uniform_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

bool all_finite(const double* a, int64_t len) {
  for (int64_t i = 0; i < len; ++i)
    if (!std::isfinite(a[i])) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Kernel geometry: Xs = X / ls stored row-major for the pair loops.
struct Geometry {
  int64_t n = 0;
  int d = 0;
  std::vector<double> xs;  // n x d row-major, scaled by 1/ls
  std::vector<double> sq;  // ||xs_i||^2, kernel.cpp:105
  double sf2 = 0, noise2 = 0, sf = 0, sigma = 0;

  Geometry(const double* X, int64_t n_, int d_, const double* ls, double sf_, double sigma_)
      : n(n_), d(d_), xs(static_cast<size_t>(n_) * d_), sq(n_), sf(sf_), sigma(sigma_) {
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) {
        const double v = X[k * n + i] * (1.0 / ls[k]);  // X * ls.cwiseInverse().asDiagonal()
        xs[i * d + k] = v;
        acc += v * v;
      }
      sq[i] = acc;
    }
    sf2 = sf * sf;
    noise2 = sigma * sigma;
  }

  // kernel.cpp:101-139: D = (sq_i + sq_j) - 2 G_ij, clamped >= 0; R = sqrt(D)
  inline double dist(int64_t i, int64_t j) const {
    const double* a = &xs[i * d];
    const double* b = &xs[j * d];
    double g = 0.0;
    for (int k = 0; k < d; ++k) g += a[k] * b[k];
    double D = (sq[i] + sq[j]) - 2.0 * g;
    if (D < 0.0) D = 0.0;
    return std::sqrt(D);
  }
  inline double decay(double R) const { return std::exp(-kSqrt3 * R); }
  inline double kval(double R) const { return sf2 * (1.0 + kSqrt3 * R) * decay(R); }
  inline double hval(int64_t i, int64_t j) const {
    double v = kval(dist(i, j));
    if (i == j) v += noise2;
    return v;
  }
};

void check_hyper(int d, const double* ls, double sf, double sigma) {
  for (int k = 0; k < d; ++k)
    if (!(ls[k] > 0.0) || !std::isfinite(ls[k]))
      throw std::invalid_argument("lengthscales must be positive and finite");
  if (!(sf > 0.0) || !(sigma > 0.0)) throw std::invalid_argument("scales must be positive");
}

// ---------------------------------------------------------------------------
// System operators used by the solvers: either a dense H (the reference's own
// representation) or matrix-free over the geometry.
struct Op {
  int64_t n = 0;
  virtual ~Op() = default;
  // out (n x s) = H V
  virtual void hv(const double* V, int s, double* out) const = 0;
  // R (n x s) -= H[:, j0:j0+b] * delta (b x s)        solvers.cpp:186
  virtual void sub_cols(int64_t j0, int64_t b, const double* delta, int s, double* R) const = 0;
  // out (m x s) = H[idx, :] * Xs                         solvers.cpp:241-242
  virtual void rows(const int64_t* idx, int64_t m, const double* Xsol, int s, double* out) const = 0;
  // dense block H[j0:j0+b, j0:j0+b] column-major        solvers.cpp:161
  virtual void block(int64_t j0, int64_t b, double* out) const = 0;
};

struct DenseOp : Op {
  const double* H;
  explicit DenseOp(const double* H_, int64_t n_) : H(H_) { n = n_; }
  void hv(const double* V, int s, double* out) const override {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int c = 0; c < s; ++c) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc += H[j * n + i] * V[c * n + j];
        out[c * n + i] = acc;
      }
  }
  void sub_cols(int64_t j0, int64_t b, const double* delta, int s, double* R) const override {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int c = 0; c < s; ++c) {
        double acc = 0.0;
        for (int64_t j = 0; j < b; ++j) acc += H[(j0 + j) * n + i] * delta[c * b + j];
        R[c * n + i] -= acc;
      }
  }
  void rows(const int64_t* idx, int64_t m, const double* Xsol, int s, double* out) const override {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < m; ++r)
      for (int c = 0; c < s; ++c) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc += H[j * n + idx[r]] * Xsol[c * n + j];
        out[c * m + r] = acc;
      }
  }
  void block(int64_t j0, int64_t b, double* out) const override {
    for (int64_t j = 0; j < b; ++j)
      for (int64_t i = 0; i < b; ++i) out[j * b + i] = H[(j0 + j) * n + (j0 + i)];
  }
};

struct FreeOp : Op {
  const Geometry& g;
  explicit FreeOp(const Geometry& g_) : g(g_) { n = g_.n; }
  void hv(const double* V, int s, double* out) const override {
    std::vector<double> row;
#pragma omp parallel for schedule(static) private(row)
    for (int64_t i = 0; i < n; ++i) {
      row.assign(s, 0.0);
      for (int64_t j = 0; j < n; ++j) {
        const double h = g.hval(i, j);
        for (int c = 0; c < s; ++c) row[c] += h * V[c * n + j];
      }
      for (int c = 0; c < s; ++c) out[c * n + i] = row[c];
    }
  }
  void sub_cols(int64_t j0, int64_t b, const double* delta, int s, double* R) const override {
    std::vector<double> row;
#pragma omp parallel for schedule(static) private(row)
    for (int64_t i = 0; i < n; ++i) {
      row.assign(s, 0.0);
      for (int64_t j = 0; j < b; ++j) {
        const double h = g.hval(i, j0 + j);
        for (int c = 0; c < s; ++c) row[c] += h * delta[c * b + j];
      }
      for (int c = 0; c < s; ++c) R[c * n + i] -= row[c];
    }
  }
  void rows(const int64_t* idx, int64_t m, const double* Xsol, int s, double* out) const override {
    std::vector<double> row;
#pragma omp parallel for schedule(static) private(row)
    for (int64_t r = 0; r < m; ++r) {
      row.assign(s, 0.0);
      const int64_t i = idx[r];
      for (int64_t j = 0; j < n; ++j) {
        const double h = g.hval(i, j);
        for (int c = 0; c < s; ++c) row[c] += h * Xsol[c * n + j];
      }
      for (int c = 0; c < s; ++c) out[c * m + r] = row[c];
    }
  }
  void block(int64_t j0, int64_t b, double* out) const override {
    for (int64_t j = 0; j < b; ++j)
      for (int64_t i = 0; i < b; ++i) out[j * b + i] = g.hval(j0 + i, j0 + j);
  }
};

// ---------------------------------------------------------------------------
// Dense Cholesky (Eigen::LLT stand-in, solvers.cpp:161 / exact.cpp:17).
bool cholesky(std::vector<double>& A, int64_t b) {  // in place, lower, column-major
  for (int64_t j = 0; j < b; ++j) {
    double djj = A[j * b + j];
    for (int64_t k = 0; k < j; ++k) djj -= A[k * b + j] * A[k * b + j];
    if (!(djj > 0.0) || !std::isfinite(djj)) return false;
    const double ljj = std::sqrt(djj);
    A[j * b + j] = ljj;
    for (int64_t i = j + 1; i < b; ++i) {
      double v = A[j * b + i];
      for (int64_t k = 0; k < j; ++k) v -= A[k * b + i] * A[k * b + j];
      A[j * b + i] = v / ljj;
    }
  }
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i < j; ++i) A[j * b + i] = 0.0;
  return true;
}

void chol_solve(const std::vector<double>& L, int64_t b, double* rhs, int s) {
  for (int c = 0; c < s; ++c) {
    double* x = rhs + static_cast<int64_t>(c) * b;
    for (int64_t i = 0; i < b; ++i) {  // L y = r
      double v = x[i];
      for (int64_t k = 0; k < i; ++k) v -= L[k * b + i] * x[k];
      x[i] = v / L[i * b + i];
    }
    for (int64_t i = b - 1; i >= 0; --i) {  // L^T x = y
      double v = x[i];
      for (int64_t k = i + 1; k < b; ++k) v -= L[i * b + k] * x[k];
      x[i] = v / L[i * b + i];
    }
  }
}

// ---------------------------------------------------------------------------
// Solvers, solvers.cpp:49-284.
struct Tol {
  std::vector<double> bnorm, tol;
};

Tol column_tolerances(const double* rhs, int64_t n, int s, double tm, double ts) {  // :49-56
  Tol t;
  t.bnorm.resize(s);
  t.tol.resize(s);
  for (int c = 0; c < s; ++c) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += rhs[c * n + i] * rhs[c * n + i];
    t.bnorm[c] = std::sqrt(acc);
    t.tol[c] = c == 0 ? tm : ts;
  }
  return t;
}

double col_norm2(const double* a, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * a[i];
  return acc;
}

void finalize(const Op& op, const double* rhs, int s, or_solve_state* st, const Tol& tol) {  // :69-77
  const int64_t n = op.n;
  std::vector<double> hx(static_cast<size_t>(n) * s);
  op.hv(st->solutions, s, hx.data());
  for (int c = 0; c < s; ++c) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double e = rhs[c * n + i] - hx[c * n + i];
      acc += e * e;
    }
    st->per_column_relative_residual[c] = tol.bnorm[c] > 0.0 ? std::sqrt(acc) / tol.bnorm[c] : 0.0;
  }
}

void check_shapes(const double* rhs, const double* init, int64_t n, int s) {  // :58-67
  if (s < 1) throw std::invalid_argument("solve: rhs needs at least one column");
  if (!all_finite(rhs, n * s) || !all_finite(init, n * s))
    throw std::invalid_argument("solve: non-finite right-hand side or init");
}

inline double rnd(double v, bool f32) { return f32 ? static_cast<double>(static_cast<float>(v)) : v; }

void cg_solve(const Op& op, const double* rhs, const double* init, int s, double tm, double ts,
              int max_it, or_solve_state* st, bool f32 = false) {  // solvers.cpp:81-139
  const int64_t n = op.n;
  check_shapes(rhs, init, n, s);
  const Tol tol = column_tolerances(rhs, n, s, tm, ts);
  if (max_it <= 0) max_it = 10 * static_cast<int>(n);
  const size_t ns = static_cast<size_t>(n) * s;
  double* Xs = st->solutions;
  double* R = st->residuals;
  std::memcpy(Xs, init, ns * sizeof(double));
  std::vector<double> hx(ns);
  op.hv(Xs, s, hx.data());
  for (size_t k = 0; k < ns; ++k) R[k] = rnd(rhs[k] - rnd(hx[k], f32), f32);
  std::vector<int> conv(s, 0);
  std::vector<double> P(ns, 0.0), rs(s), HP(ns);
  for (int c = 0; c < s; ++c) {
    rs[c] = col_norm2(R + c * n, n);
    if (tol.bnorm[c] == 0.0 || std::sqrt(rs[c]) <= tol.tol[c] * tol.bnorm[c])
      conv[c] = 1;
    else
      std::memcpy(&P[c * n], R + c * n, n * sizeof(double));
  }
  auto all_conv = [&]() { return std::all_of(conv.begin(), conv.end(), [](int v) { return v != 0; }); };
  int it = 0;
  while (!all_conv() && it < max_it) {
    ++it;
    op.hv(P.data(), s, HP.data());
    if (f32)
      for (double& v : HP) v = rnd(v, true);
    const bool refresh = (it % 50 == 0);
    for (int c = 0; c < s; ++c) {
      if (conv[c]) continue;
      double* p = &P[c * n];
      double* hp = &HP[c * n];
      double pHp = 0.0;
      for (int64_t i = 0; i < n; ++i) pHp += p[i] * hp[i];
      if (!(pHp > 0.0))
        throw NumericalError("cg_solve: non-positive curvature encountered, H is not positive definite");
      const double alpha = rs[c] / pHp;
      double* x = Xs + c * n;
      double* r = R + c * n;
      const double a_v = rnd(alpha, f32);
      for (int64_t i = 0; i < n; ++i) x[i] = rnd(x[i] + a_v * p[i], f32);
      if (refresh) {
        std::vector<double> hxc(n);
        op.hv(x, 1, hxc.data());
        for (int64_t i = 0; i < n; ++i) r[i] = rnd(rhs[c * n + i] - rnd(hxc[i], f32), f32);
      } else {
        for (int64_t i = 0; i < n; ++i) r[i] = rnd(r[i] - a_v * hp[i], f32);
      }
      const double rs_new = col_norm2(r, n);
      if (!std::isfinite(rs_new))
        throw NumericalError("cg_solve: NaN in iterate at iteration " + std::to_string(it));
      if (std::sqrt(rs_new) <= tol.tol[c] * tol.bnorm[c]) {
        conv[c] = 1;
        std::fill(p, p + n, 0.0);
      } else {
        const double beta = rnd(rs_new / rs[c], f32);
        for (int64_t i = 0; i < n; ++i) p[i] = rnd(r[i] + beta * p[i], f32);
      }
      rs[c] = rs_new;
    }
  }
  st->iterations_used = it;
  for (int c = 0; c < s; ++c) st->converged[c] = conv[c];
  finalize(op, rhs, s, st, tol);
}

void ap_solve(const Op& op, const double* rhs, const double* init, int s, double tm, double ts,
              int block_size, int max_epochs, or_solve_state* st) {  // solvers.cpp:141-196
  const int64_t n = op.n;
  check_shapes(rhs, init, n, s);
  const Tol tol = column_tolerances(rhs, n, s, tm, ts);
  if (max_epochs <= 0) max_epochs = 1000;
  const int64_t bs = std::min<int64_t>(std::max(block_size, 1), n);
  struct Block {
    int64_t start, size;
    std::vector<double> L;
  };
  std::vector<Block> blocks;
  for (int64_t start = 0; start < n; start += bs) {
    Block b;
    b.start = start;
    b.size = std::min(bs, n - start);
    b.L.resize(static_cast<size_t>(b.size) * b.size);
    op.block(b.start, b.size, b.L.data());
    if (!cholesky(b.L, b.size))
      throw NumericalError("ap_solve: diagonal block factorization failed, H is not positive definite");
    blocks.push_back(std::move(b));
  }
  const size_t ns = static_cast<size_t>(n) * s;
  double* Xs = st->solutions;
  double* R = st->residuals;
  std::memcpy(Xs, init, ns * sizeof(double));
  std::vector<double> hx(ns);
  op.hv(Xs, s, hx.data());
  for (size_t k = 0; k < ns; ++k) R[k] = rhs[k] - hx[k];
  std::vector<int> conv(s, 0);
  auto update = [&]() {
    for (int c = 0; c < s; ++c)
      conv[c] = tol.bnorm[c] == 0.0 || std::sqrt(col_norm2(R + c * n, n)) <= tol.tol[c] * tol.bnorm[c];
  };
  update();
  auto all_conv = [&]() { return std::all_of(conv.begin(), conv.end(), [](int v) { return v != 0; }); };
  int epoch = 0;
  std::vector<double> delta;
  while (!all_conv() && epoch < max_epochs) {
    ++epoch;
    for (const Block& b : blocks) {
      delta.resize(static_cast<size_t>(b.size) * s);
      for (int c = 0; c < s; ++c)
        std::memcpy(&delta[c * b.size], R + c * n + b.start, b.size * sizeof(double));
      chol_solve(b.L, b.size, delta.data(), s);
      for (int c = 0; c < s; ++c)
        for (int64_t i = 0; i < b.size; ++i) Xs[c * n + b.start + i] += delta[c * b.size + i];
      op.sub_cols(b.start, b.size, delta.data(), s, R);
    }
    op.hv(Xs, s, hx.data());
    for (size_t k = 0; k < ns; ++k) R[k] = rhs[k] - hx[k];
    if (!all_finite(R, ns))
      throw NumericalError("ap_solve: NaN in iterate at epoch " + std::to_string(epoch));
    update();
  }
  st->iterations_used = epoch;
  for (int c = 0; c < s; ++c) st->converged[c] = conv[c];
  finalize(op, rhs, s, st, tol);
}

void sgd_solve(const Op& op, const double* rhs, const double* init, int s, double tm, double ts,
               int minibatch, double momentum, double lr, int max_steps, uint64_t seed,
               or_solve_state* st) {  // solvers.cpp:198-263
  const int64_t n = op.n;
  check_shapes(rhs, init, n, s);
  const Tol tol = column_tolerances(rhs, n, s, tm, ts);
  const int64_t m = std::min<int64_t>(std::max(minibatch, 1), n);
  if (max_steps <= 0) max_steps = static_cast<int>((100 * n) / m);
  const size_t ns = static_cast<size_t>(n) * s;
  double* Xs = st->solutions;
  double* R = st->residuals;
  std::memcpy(Xs, init, ns * sizeof(double));
  std::vector<double> hx(ns);
  op.hv(Xs, s, hx.data());
  for (size_t k = 0; k < ns; ++k) R[k] = rhs[k] - hx[k];
  std::vector<int> conv(s, 0);
  auto update = [&]() {
    for (int c = 0; c < s; ++c)
      conv[c] = tol.bnorm[c] == 0.0 || std::sqrt(col_norm2(R + c * n, n)) <= tol.tol[c] * tol.bnorm[c];
  };
  update();
  auto all_conv = [&]() { return std::all_of(conv.begin(), conv.end(), [](int v) { return v != 0; }); };
  std::vector<double> vel(ns, 0.0), batch(static_cast<size_t>(m) * s);
  std::vector<int64_t> pool(n);
  std::iota(pool.begin(), pool.end(), 0);
  std::mt19937_64 rng(seed);
  const double grad_scale = static_cast<double>(n) / static_cast<double>(m);
  const double step_scale = lr / static_cast<double>(n);
  int step = 0;
  while (!all_conv() && step < max_steps) {
    ++step;
    for (int64_t i = 0; i < m; ++i) {
      const int64_t j = i + static_cast<int64_t>(uniform_below(rng, static_cast<uint64_t>(n - i)));
      std::swap(pool[i], pool[j]);
    }
    op.rows(pool.data(), m, Xs, s, batch.data());
    for (int c = 0; c < s; ++c)
      for (int64_t i = 0; i < m; ++i) batch[c * m + i] = rhs[c * n + pool[i]] - batch[c * m + i];
    for (int64_t i = 0; i < m; ++i) {
      const int64_t row = pool[i];
      for (int c = 0; c < s; ++c) {
        double& v = vel[c * n + row];
        v = momentum * v - grad_scale * batch[c * m + i];
        Xs[c * n + row] -= step_scale * v;
        R[c * n + row] = batch[c * m + i];
      }
    }
    const double sol_norm = std::sqrt(col_norm2(Xs, static_cast<int64_t>(ns)));
    if (!std::isfinite(sol_norm) || sol_norm > 1e12)
      throw NumericalError("sgd_solve: iterate diverged at step " + std::to_string(step) +
                           "; use a smaller learning rate");
    update();
  }
  st->iterations_used = step;
  for (int c = 0; c < s; ++c) st->converged[c] = conv[c];
  finalize(op, rhs, s, st, tol);
}

void validate_solver(const or_solver_cfg& c) {  // solvers.cpp:31-37
  if (!(c.tol_mean > 0.0 && c.tol_mean < 1.0) || !(c.tol_samples > 0.0 && c.tol_samples < 1.0))
    throw std::invalid_argument("SolverConfig: tolerances must lie in (0, 1)");
  if (c.block_size < 1) throw std::invalid_argument("SolverConfig: block_size must be >= 1");
  if (c.minibatch_size < 1) throw std::invalid_argument("SolverConfig: minibatch_size must be >= 1");
  if (c.max_iterations < 0) throw std::invalid_argument("SolverConfig: max_iterations must be >= 0");
}

void solve_op(const Op& op, const or_solver_cfg& c, const double* rhs, const double* init, int s,
              or_solve_state* st) {  // solvers.cpp:265-279
  validate_solver(c);
  switch (c.kind) {
    case 0:
      cg_solve(op, rhs, init, s, c.tol_mean, c.tol_samples, c.max_iterations, st, c.f32_vectors != 0);
      return;
    case 1:
      ap_solve(op, rhs, init, s, c.tol_mean, c.tol_samples, c.block_size, c.max_iterations, st);
      return;
    case 2:
      sgd_solve(op, rhs, init, s, c.tol_mean, c.tol_samples, c.minibatch_size, c.momentum,
                c.learning_rate, c.max_iterations, c.seed, st);
      return;
  }
  throw std::invalid_argument("solve: unknown solver kind");
}

// ---------------------------------------------------------------------------
// Hyperparameter transforms (kernel.cpp:14-77; log added for BASELINE).
double softplus(double x) {
  if (x > 0.0) return x + std::log1p(std::exp(-x));
  return std::log1p(std::exp(x));
}
double softplus_inverse(double v) {
  if (!(v > 0.0)) throw std::invalid_argument("softplus_inverse: argument must be positive");
  if (v > 0.6931471805599453) return v + std::log1p(-std::exp(-v));
  return std::log(std::expm1(v));
}
double softplus_derivative(double x) {
  if (x > 0.0) return 1.0 / (1.0 + std::exp(-x));
  const double e = std::exp(x);
  return e / (1.0 + e);
}
double to_constrained(int tr, double raw) { return tr == 1 ? std::exp(raw) : softplus(raw); }
double to_raw(int tr, double v) {
  if (tr == 1) {
    if (!(v > 0.0)) throw std::invalid_argument("log transform: argument must be positive");
    return std::log(v);
  }
  return softplus_inverse(v);
}
double chain(int tr, double raw) { return tr == 1 ? std::exp(raw) : softplus_derivative(raw); }

struct Hyper {
  int d;
  std::vector<double> ls;
  double sf, sigma;
  Hyper(int tr, int d_, const double* raw) : d(d_), ls(d_) {
    for (int k = 0; k < d; ++k) ls[k] = to_constrained(tr, raw[k]);
    sf = to_constrained(tr, raw[d]);
    sigma = to_constrained(tr, raw[d + 1]);
  }
};

// ---------------------------------------------------------------------------
// Streamed derivative contractions with low-rank A and B
// (kernel.cpp:216-252, estimator.cpp:63-82).  Direct (x_ik - x_jk)^2 per
// entry instead of the expansion trick (same quantity; fp rounding differs).
void grad_contractions(const double* X, int64_t n, int d, int tr, const double* raw,
                       const double* vy, const double* L, const double* R, int s, double coef_b,
                       double* out_a, double* out_b) {
  const Hyper h(tr, d, raw);
  const Geometry g(X, n, d, h.ls.data(), h.sf, h.sigma);
  const int p = d + 2;
  // per-row partial sums, reduced in row order afterwards (deterministic)
  std::vector<double> part_a(static_cast<size_t>(n) * (d + 1)), part_b(static_cast<size_t>(n) * (d + 1));
  std::vector<double> lrow;
#pragma omp parallel for schedule(static) private(lrow)
  for (int64_t i = 0; i < n; ++i) {
    lrow.resize(s);
    for (int c = 0; c < s; ++c) lrow[c] = L[c * n + i];
    std::vector<double> acc_a(d + 1, 0.0), acc_b(d + 1, 0.0);
    for (int64_t j = 0; j < n; ++j) {
      const double Rd = g.dist(i, j);
      const double dec = g.decay(Rd);
      const double kv = g.sf2 * (1.0 + kSqrt3 * Rd) * dec;
      const double a = 0.5 * vy[i] * vy[j];
      double bsum = 0.0;
      for (int c = 0; c < s; ++c) bsum += lrow[c] * R[c * n + j];
      const double b = coef_b * bsum;
      for (int k = 0; k < d; ++k) {
        const double diff = X[k * n + i] - X[k * n + j];
        const double w = dec * diff * diff;
        acc_a[k] += w * a;
        acc_b[k] += w * b;
      }
      acc_a[d] += kv * a;
      acc_b[d] += kv * b;
    }
    for (int k = 0; k <= d; ++k) {
      part_a[i * (d + 1) + k] = acc_a[k];
      part_b[i * (d + 1) + k] = acc_b[k];
    }
  }
  std::vector<double> sa(d + 1, 0.0), sb(d + 1, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k <= d; ++k) {
      sa[k] += part_a[i * (d + 1) + k];
      sb[k] += part_b[i * (d + 1) + k];
    }
  for (int k = 0; k < d; ++k) {
    const double ls = h.ls[k];
    const double scale = 3.0 * h.sf * h.sf * chain(tr, raw[k]) / (ls * ls * ls);
    out_a[k] = scale * sa[k];
    out_b[k] = scale * sb[k];
  }
  const double chain_sf = chain(tr, raw[d]);
  out_a[d] = (2.0 * chain_sf / h.sf) * sa[d];
  out_b[d] = (2.0 * chain_sf / h.sf) * sb[d];
  const double dnoise = 2.0 * h.sigma * chain(tr, raw[d + 1]);
  double ta = 0.0, tb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    ta += 0.5 * vy[i] * vy[i];
    double bs = 0.0;
    for (int c = 0; c < s; ++c) bs += L[c * n + i] * R[c * n + i];
    tb += coef_b * bs;
  }
  out_a[d + 1] = dnoise * ta;
  out_b[d + 1] = dnoise * tb;
  (void)p;
}

// ---------------------------------------------------------------------------
// Probes (estimator.cpp:21-37) and pathwise RFF probes (new, BASELINE a12).
void sample_probes(int64_t n, int s, int dist, uint64_t seed, double* out) {
  if (n < 1 || s < 1) throw std::invalid_argument("sample_probes: n and s must be >= 1");
  std::mt19937_64 rng(seed);
  if (dist == 0) {
    std::normal_distribution<double> normal(0.0, 1.0);
    for (int j = 0; j < s; ++j)
      for (int64_t i = 0; i < n; ++i) out[j * n + i] = normal(rng);
  } else {
    for (int j = 0; j < s; ++j)
      for (int64_t i = 0; i < n; ++i) out[j * n + i] = (rng() & 1u) ? 1.0 : -1.0;
  }
}

void rff_base(int64_t n, int d, int F, int s, uint64_t seed, double* oz, double* chi2, double* b,
              double* w, double* eps) {
  if (n < 1 || d < 1 || F < 1 || s < 1) throw std::invalid_argument("rff_base: bad sizes");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int64_t f = 0; f < F; ++f)
    for (int k = 0; k < d; ++k) oz[f * d + k] = normal(rng);
  for (int64_t f = 0; f < F; ++f) {
    double acc = 0.0;
    for (int q = 0; q < 3; ++q) {
      const double z = normal(rng);
      acc += z * z;
    }
    chi2[f] = acc;
  }
  for (int64_t f = 0; f < F; ++f) b[f] = 2.0 * M_PI * uniform_unit(rng);
  for (int j = 0; j < s; ++j)
    for (int64_t f = 0; f < F; ++f) w[j * F + f] = normal(rng);
  for (int j = 0; j < s; ++j)
    for (int64_t i = 0; i < n; ++i) eps[j * n + i] = normal(rng);
}

void rff_probes(const double* X, int64_t n, int d, const double* ls, double sf, double sigma, int F,
                int s, const double* oz, const double* chi2, const double* b, const double* w,
                const double* eps, double* out) {
  // omega_f = z_f / sqrt(u_f / 3) (Matern-3/2 spectral density: Student-t, 3 dof)
  std::vector<double> om(static_cast<size_t>(F) * d);
  for (int f = 0; f < F; ++f) {
    const double scale = 1.0 / std::sqrt(chi2[f] / 3.0);
    for (int k = 0; k < d; ++k) om[f * d + k] = oz[f * d + k] * scale / ls[k];
  }
  const double amp = sf * std::sqrt(2.0 / static_cast<double>(F));
  std::vector<double> phi;
#pragma omp parallel for schedule(static) private(phi)
  for (int64_t i = 0; i < n; ++i) {
    phi.resize(F);
    for (int f = 0; f < F; ++f) {
      double ph = b[f];
      for (int k = 0; k < d; ++k) ph += om[f * d + k] * X[k * n + i];
      phi[f] = std::cos(ph);
    }
    for (int j = 0; j < s; ++j) {
      double acc = 0.0;
      for (int f = 0; f < F; ++f) acc += w[j * F + f] * phi[f];
      out[j * n + i] = amp * acc + sigma * eps[j * n + i];
    }
  }
}

// ---------------------------------------------------------------------------
// Exact path (exact.cpp:25-50) for small n.
void exact_parts(const double* X, const double* y, int64_t n, int d, int tr, const double* raw,
                 double* grad, double* mll) {
  const Hyper h(tr, d, raw);
  const Geometry g(X, n, d, h.ls.data(), h.sf, h.sigma);
  if (n > 20000) throw std::invalid_argument("exact: n exceeds the dense guard");  // exact.hpp:23
  std::vector<double> L(static_cast<size_t>(n) * n);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) L[j * n + i] = g.hval(i, j);
  if (!cholesky(L, n)) throw NumericalError("exact: system matrix is not positive definite");
  std::vector<double> alpha(y, y + n);
  chol_solve(L, n, alpha.data(), 1);
  if (mll) {
    double yta = 0.0, logdet = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      yta += y[i] * alpha[i];
      logdet += std::log(L[i * n + i]);
    }
    *mll = -0.5 * yta - logdet - 0.5 * static_cast<double>(n) * kLog2Pi;
  }
  if (!grad) return;
  // H^-1 via n solves against the identity (columns independent -> parallel)
  std::vector<double> Hinv(static_cast<size_t>(n) * n, 0.0);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t c = 0; c < n; ++c) {
    double* col = &Hinv[c * n];
    col[c] = 1.0;
    chol_solve(L, n, col, 1);
  }
  // g_k = <dH_k, 1/2 a a^T> - <dH_k, 1/2 H^-1>
  const int p = d + 2;
  std::vector<double> acc_q(static_cast<size_t>(n) * (d + 1)), acc_t(static_cast<size_t>(n) * (d + 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    std::vector<double> q(d + 1, 0.0), t(d + 1, 0.0);
    for (int64_t j = 0; j < n; ++j) {
      const double Rd = g.dist(i, j);
      const double dec = g.decay(Rd);
      const double kv = g.sf2 * (1.0 + kSqrt3 * Rd) * dec;
      const double a = 0.5 * alpha[i] * alpha[j];
      const double b = 0.5 * Hinv[j * n + i];
      for (int k = 0; k < d; ++k) {
        const double diff = X[k * n + i] - X[k * n + j];
        const double w = dec * diff * diff;
        q[k] += w * a;
        t[k] += w * b;
      }
      q[d] += kv * a;
      t[d] += kv * b;
    }
    for (int k = 0; k <= d; ++k) {
      acc_q[i * (d + 1) + k] = q[k];
      acc_t[i * (d + 1) + k] = t[k];
    }
  }
  std::vector<double> sq(d + 1, 0.0), st(d + 1, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k <= d; ++k) {
      sq[k] += acc_q[i * (d + 1) + k];
      st[k] += acc_t[i * (d + 1) + k];
    }
  for (int k = 0; k < d; ++k) {
    const double ls = h.ls[k];
    const double scale = 3.0 * h.sf * h.sf * chain(tr, raw[k]) / (ls * ls * ls);
    grad[k] = scale * sq[k] - scale * st[k];
  }
  const double cs = 2.0 * chain(tr, raw[d]) / h.sf;
  grad[d] = cs * sq[d] - cs * st[d];
  const double dn = 2.0 * h.sigma * chain(tr, raw[d + 1]);
  double ta = 0.0, tb = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    ta += 0.5 * alpha[i] * alpha[i];
    tb += 0.5 * Hinv[i * n + i];
  }
  grad[d + 1] = dn * ta - dn * tb;
  (void)p;
}

void adam_step(double* raw, const double* grad, double* m, double* v, int p, int t, double lr,
               double b1, double b2, double eps) {  // optimizer.cpp:48-65
  if (t < 1) throw std::invalid_argument("adam_step: t must be >= 1");
  for (int k = 0; k < p; ++k)
    if (!std::isfinite(grad[k]))
      throw NumericalError("adam_step: non-finite gradient at step " + std::to_string(t));
  const double c1 = 1.0 - std::pow(b1, t);
  const double c2 = 1.0 - std::pow(b2, t);
  for (int k = 0; k < p; ++k) {
    m[k] = b1 * m[k] + (1.0 - b1) * grad[k];
    v[k] = b2 * v[k] + (1.0 - b2) * (grad[k] * grad[k]);
    const double mh = m[k] / c1;
    const double vh = v[k] / c2;
    raw[k] += lr * mh / (std::sqrt(vh) + eps);
  }
}

// ---------------------------------------------------------------------------
// run_loop, optimizer.cpp:81-171 (+ pathwise estimator, log transform, sigma_0).
void train(const double* X, const double* y, int64_t n, int d, const or_train_cfg& c, or_trace* tr) {
  if (c.steps < 1) throw std::invalid_argument("TrainConfig: steps must be >= 1");
  if (c.num_probes < 1) throw std::invalid_argument("TrainConfig: num_probes must be >= 1");
  if (!(c.learning_rate > 0.0)) throw std::invalid_argument("TrainConfig: learning rate must be positive");
  if (!(c.init_constrained > 0.0))
    throw std::invalid_argument("TrainConfig: initial constrained value must be positive");
  validate_solver(c.solver);
  if (n < 1) throw std::invalid_argument("train: dataset is empty");
  const int p = d + 2;
  const int s = c.num_probes;
  const int sp = s + 1;
  const int T = c.transform;
  std::vector<double> raw(p), m(p, 0.0), v(p, 0.0);
  for (int k = 0; k < d; ++k) raw[k] = to_raw(T, c.init_constrained);
  raw[d] = to_raw(T, c.init_signal > 0.0 ? c.init_signal : c.init_constrained);
  raw[d + 1] = to_raw(T, c.init_noise > 0.0 ? c.init_noise : c.init_constrained);

  const bool fixed_probes = c.mode != 1;
  const bool warm = c.mode == 0;
  const bool pathwise = c.estimator == 1;
  const int F = c.rff_features > 0 ? c.rff_features : 1000;
  const size_t ns = static_cast<size_t>(n) * s;
  std::vector<double> Z(ns), oz, chi2, pb, w, eps;
  uint64_t probe_seed = 0;
  auto draw = [&](uint64_t seed) {
    probe_seed = seed;
    if (pathwise) {
      oz.resize(static_cast<size_t>(F) * d);
      chi2.resize(F);
      pb.resize(F);
      w.resize(static_cast<size_t>(F) * s);
      eps.resize(ns);
      rff_base(n, d, F, s, seed, oz.data(), chi2.data(), pb.data(), w.data(), eps.data());
    } else {
      sample_probes(n, s, c.probe_distribution, seed, Z.data());
    }
  };
  if (!c.exact_gradients && fixed_probes) draw(or_derive_seed(c.seed, 1));

  std::vector<double> prev, rhs(static_cast<size_t>(n) * sp), init(static_cast<size_t>(n) * sp);
  std::vector<double> sol(static_cast<size_t>(n) * sp), res(static_cast<size_t>(n) * sp), pcr(sp);
  std::vector<int> conv(sp);
  for (int t = 1; t <= c.steps; ++t) {
    try {
      const Hyper h(T, d, raw.data());
      std::vector<double> grad(p);
      int iters = 0;
      double wsd = 0.0;
      if (c.exact_gradients) {
        exact_parts(X, y, n, d, T, raw.data(), grad.data(), nullptr);
      } else {
        const Geometry g(X, n, d, h.ls.data(), h.sf, h.sigma);
        const FreeOp op(g);
        if (!fixed_probes) draw(or_derive_seed(c.seed, static_cast<uint64_t>(t)));
        if (pathwise)
          rff_probes(X, n, d, h.ls.data(), h.sf, h.sigma, F, s, oz.data(), chi2.data(), pb.data(),
                     w.data(), eps.data(), Z.data());
        std::memcpy(rhs.data(), y, n * sizeof(double));
        std::memcpy(rhs.data() + n, Z.data(), ns * sizeof(double));
        or_solver_cfg sc = c.solver;
        sc.seed = or_derive_seed(or_derive_seed(c.seed, kSolverStream), static_cast<uint64_t>(t));
        const bool have_warm = warm && !prev.empty();
        if (have_warm)
          init = prev;
        else
          std::fill(init.begin(), init.end(), 0.0);
        or_solve_state st{sol.data(), res.data(), pcr.data(), conv.data(), 0};
        solve_op(op, sc, rhs.data(), init.data(), sp, &st);
        iters = st.iterations_used;
        if (have_warm) {  // estimator.cpp:84-95
          std::vector<double> D(sol.size()), HD(sol.size());
          for (size_t k = 0; k < D.size(); ++k) D[k] = init[k] - sol[k];
          op.hv(D.data(), sp, HD.data());
          double acc = 0.0;
          for (int cc = 0; cc < sp; ++cc) {
            double col = 0.0;
            for (int64_t i = 0; i < n; ++i) col += D[cc * n + i] * HD[cc * n + i];
            acc += col;
          }
          const double mean_q = acc / sp / static_cast<double>(n);
          wsd = std::sqrt(std::max(mean_q, 0.0));
        }
        std::vector<double> qa(p), qb(p);
        const double* right = pathwise ? sol.data() + n : Z.data();
        grad_contractions(X, n, d, T, raw.data(), sol.data(), sol.data() + n, right, s,
                          0.5 / static_cast<double>(s), qa.data(), qb.data());
        for (int k = 0; k < p; ++k) grad[k] = qa[k] - qb[k];
        prev = sol;
        if (tr && tr->per_column_relative_residual)
          std::memcpy(tr->per_column_relative_residual + static_cast<size_t>(t - 1) * sp, pcr.data(),
                      sp * sizeof(double));
      }
      adam_step(raw.data(), grad.data(), m.data(), v.data(), p, t, c.learning_rate, c.adam_beta1,
                c.adam_beta2, c.adam_eps);
      if (tr) {
        const size_t off = static_cast<size_t>(t - 1) * p;
        if (tr->raw_params) std::memcpy(tr->raw_params + off, raw.data(), p * sizeof(double));
        if (tr->constrained_params)
          for (int k = 0; k < p; ++k) tr->constrained_params[off + k] = to_constrained(T, raw[k]);
        if (tr->gradient) std::memcpy(tr->gradient + off, grad.data(), p * sizeof(double));
        if (tr->solver_iterations) tr->solver_iterations[t - 1] = iters;
        if (tr->warm_start_distance) tr->warm_start_distance[t - 1] = wsd;
        if (tr->probe_seed) tr->probe_seed[t - 1] = probe_seed;
      }
    } catch (const NumericalError& e) {
      throw NumericalError("step " + std::to_string(t) + ": " + e.what());
    }
  }
  if (tr && tr->final_solutions && !prev.empty())
    std::memcpy(tr->final_solutions, prev.data(), prev.size() * sizeof(double));
}

}  // namespace

// ===========================================================================
extern "C" {

const char* or_last_error(void) { return g_last_error.c_str(); }

uint64_t or_splitmix64(uint64_t x) {  // common.hpp:25-30
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t or_derive_seed(uint64_t base, uint64_t stream) {  // common.hpp:34-36
  return or_splitmix64(or_splitmix64(base) ^ or_splitmix64(stream + 0x51ed2701ab0a3c11ULL));
}

// dataset.cpp:167-190 (synthesize): the random draws -- X ~ U[0,1]^d row by
// row (uniform_unit) and xi ~ N(0,1) (libstdc++ normal_distribution) from
// mt19937_64(derive_seed(seed, 0xda7a)); y = chol(H) xi is formed by the caller.
int or_synthesize_draws(int n, int d, uint64_t seed, double* X, double* xi) {
  if (n < 1 || d < 1) return 2;
  std::mt19937_64 rng(or_derive_seed(seed, 0xda7aULL));
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) X[static_cast<size_t>(i) * d + k] = uniform_unit(rng);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int i = 0; i < n; ++i) xi[i] = normal(rng);
  return 0;
}

// dataset.cpp:118-124 (split_standardize's permutation)
int or_split_order(int64_t n, uint64_t split_seed, int64_t* order) {
  if (n < 1) return 2;
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  std::mt19937_64 rng(or_derive_seed(split_seed, 0x5b117ULL));
  for (int64_t i = n - 1; i > 0; --i) {
    const int64_t j = static_cast<int64_t>(uniform_below(rng, static_cast<uint64_t>(i) + 1));
    std::swap(order[i], order[j]);
  }
  return 0;
}

double or_softplus(double x) { return softplus(x); }
double or_softplus_inverse(double v) {
  double r = std::numeric_limits<double>::quiet_NaN();
  guarded([&] { r = softplus_inverse(v); });
  return r;
}
double or_softplus_derivative(double x) { return softplus_derivative(x); }
double or_to_constrained(int t, double raw) { return to_constrained(t, raw); }
double or_to_raw(int t, double v) {
  double r = std::numeric_limits<double>::quiet_NaN();
  guarded([&] { r = to_raw(t, v); });
  return r;
}
double or_chain(int t, double raw) { return chain(t, raw); }

double or_matern32(const double* x, const double* x2, int d, const double* ls, double sf) {
  double r2 = 0.0;  // kernel.cpp:85-89
  for (int k = 0; k < d; ++k) {
    const double u = (x[k] - x2[k]) / ls[k];
    r2 += u * u;
  }
  const double r = std::sqrt(r2);
  return sf * sf * (1.0 + kSqrt3 * r) * std::exp(-kSqrt3 * r);
}

int or_build_kernel_matrices(const double* X, int64_t n, int d, const double* ls, double sf,
                             double sigma, double* system, double* kernel, double* decay) {
  return guarded([&] {
    if (n < 1) throw std::invalid_argument("build_kernel_matrices: need at least one row");
    if (!all_finite(X, n * d)) throw std::invalid_argument("build_kernel_matrices: non-finite input");
    check_hyper(d, ls, sf, sigma);
    const Geometry g(X, n, d, ls, sf, sigma);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        const double R = g.dist(i, j);
        const double dec = g.decay(R);
        const double kv = g.sf2 * (1.0 + kSqrt3 * R) * dec;
        if (decay) decay[j * n + i] = dec;
        if (kernel) kernel[j * n + i] = kv;
        if (system) system[j * n + i] = kv + (i == j ? g.noise2 : 0.0);
      }
  });
}

int or_hv(const double* X, int64_t n, int d, const double* ls, double sf, double sigma,
          const double* V, int s, double* out, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    check_hyper(d, ls, sf, sigma);
    const Geometry g(X, n, d, ls, sf, sigma);
    FreeOp(g).hv(V, s, out);
  });
}

int or_hv_rows(const double* X, int64_t n, int d, const double* ls, double sf, double sigma,
               const double* V, int s, int64_t r0, int64_t r1, double* out, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    check_hyper(d, ls, sf, sigma);
    if (r0 < 0 || r1 > n || r1 < r0) throw std::invalid_argument("or_hv_rows: bad row range");
    const Geometry g(X, n, d, ls, sf, sigma);
    std::vector<int64_t> idx(r1 - r0);
    std::iota(idx.begin(), idx.end(), r0);
    FreeOp(g).rows(idx.data(), r1 - r0, V, s, out);
  });
}

int or_dense_matmul(const double* H, int64_t n, const double* V, int s, double* out, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    DenseOp(H, n).hv(V, s, out);
  });
}

int or_solve(const double* H, const double* X, int64_t n, int d, const double* ls, double sf,
             double sigma, const or_solver_cfg* cfg, const double* rhs, const double* init, int s,
             or_solve_state* state, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    if (H) {
      solve_op(DenseOp(H, n), *cfg, rhs, init, s, state);
    } else {
      check_hyper(d, ls, sf, sigma);
      const Geometry g(X, n, d, ls, sf, sigma);
      solve_op(FreeOp(g), *cfg, rhs, init, s, state);
    }
  });
}

int or_sample_probes(int64_t n, int s, int dist, uint64_t seed, double* out) {
  return guarded([&] { sample_probes(n, s, dist, seed, out); });
}

int or_rff_base(int64_t n, int d, int F, int s, uint64_t seed, double* oz, double* chi2,
                double* b, double* w, double* eps) {
  return guarded([&] { rff_base(n, d, F, s, seed, oz, chi2, b, w, eps); });
}

int or_rff_probes(const double* X, int64_t n, int d, const double* ls, double sf, double sigma,
                  int F, int s, const double* oz, const double* chi2, const double* b,
                  const double* w, const double* eps, double* out, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    rff_probes(X, n, d, ls, sf, sigma, F, s, oz, chi2, b, w, eps, out);
  });
}

int or_grad_contractions(const double* X, int64_t n, int d, int transform, const double* raw,
                         const double* vy, const double* L, const double* R, int s, double coef_b,
                         double* out_a, double* out_b, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    grad_contractions(X, n, d, transform, raw, vy, L, R, s, coef_b, out_a, out_b);
  });
}

int or_exact_gradient(const double* X, const double* y, int64_t n, int d, int transform,
                      const double* raw, double* grad, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    exact_parts(X, y, n, d, transform, raw, grad, nullptr);
  });
}

int or_exact_mll(const double* X, const double* y, int64_t n, int d, int transform,
                 const double* raw, double* mll, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    exact_parts(X, y, n, d, transform, raw, nullptr, mll);
  });
}

int or_warm_start_distance(const double* X, int64_t n, int d, const double* ls, double sf,
                           double sigma, const double* init, const double* sol, int s,
                           double* out, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    const Geometry g(X, n, d, ls, sf, sigma);
    std::vector<double> D(static_cast<size_t>(n) * s), HD(D.size());
    for (size_t k = 0; k < D.size(); ++k) D[k] = init[k] - sol[k];
    FreeOp(g).hv(D.data(), s, HD.data());
    double acc = 0.0;
    for (int c = 0; c < s; ++c) {
      double col = 0.0;
      for (int64_t i = 0; i < n; ++i) col += D[c * n + i] * HD[c * n + i];
      acc += col;
    }
    *out = std::sqrt(std::max(acc / s / static_cast<double>(n), 0.0));
  });
}

int or_train(const double* X, const double* y, int64_t n, int d, const or_train_cfg* cfg,
             or_trace* trace, int nthreads) {
  return guarded([&] {
    set_threads(nthreads);
    train(X, y, n, d, *cfg, trace);
  });
}

int or_adam_step(double* raw, const double* grad, double* m, double* v, int p, int t, double lr,
                 double beta1, double beta2, double eps) {
  return guarded([&] { adam_step(raw, grad, m, v, p, t, lr, beta1, beta2, eps); });
}

}  // extern "C"
