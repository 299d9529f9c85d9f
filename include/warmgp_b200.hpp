// warmgp_b200.hpp — C++ adapter that keeps the reference warmgp API shape
// (proj/include/warmgp/{solvers,estimator,optimizer}.hpp) over the C-ABI in
// warmgp_b200.h.  Header-only; link against libwarmgp_b200.so.
//
// What changes for a caller of the reference: the dense `const Eigen::MatrixXd& H`
// argument of solve() (proj/include/warmgp/solvers.hpp:50-55) becomes a
// matrix-free KernelOperator (inputs X + hyperparameters, never H), and
// matrices are plain column-major std::vector<float> (Eigen::MatrixXd is
// column-major too, so `Eigen::Map<Eigen::MatrixXf>` views them without a copy).
// Exceptions are the reference's: std::invalid_argument (status 2),
// warmgp::NumericalError (status 3, same message texts), std::runtime_error
// for device failures (status 4).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "warmgp_b200.h"

namespace warmgp {

// proj/include/warmgp/common.hpp:13-16
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};

namespace b200 {

inline void check(int rc) {
  if (rc == WGP_OK) return;
  const std::string msg = wgp_last_error();
  if (rc == WGP_NUMERICAL) throw NumericalError(msg);
  if (rc == WGP_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

/// Owns one wgp_ctx (stream, device buffers, warm-start state).
class Device {
 public:
  explicit Device(int device = 0) { check(wgp_create(device, &ctx_)); }
  ~Device() { wgp_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  wgp_ctx* get() const { return ctx_; }

 private:
  wgp_ctx* ctx_ = nullptr;
};

}  // namespace b200

enum class SolverKind { Cg = WGP_SOLVER_CG, Ap = WGP_SOLVER_AP, Sgd = WGP_SOLVER_SGD };

/// proj/include/warmgp/solvers.hpp:20-32 (same fields, same defaults).
struct SolverConfig {
  SolverKind kind = SolverKind::Cg;
  double tol_mean = 0.01;
  double tol_samples = 0.1;
  int max_iterations = 0;
  int block_size = 2000;
  int minibatch_size = 1000;
  double momentum = 0.9;
  double learning_rate = 10.0;
  std::uint64_t seed = 0;

  wgp_solver_cfg c() const {
    return wgp_solver_cfg{static_cast<int>(kind), tol_mean, tol_samples, max_iterations,
                          block_size, minibatch_size, momentum, learning_rate, seed};
  }
};

/// proj/include/warmgp/solvers.hpp:38-46 (column-major n x s floats).
struct SolveState {
  std::vector<float> solutions;
  std::vector<float> residuals;
  std::vector<double> per_column_relative_residual;
  std::vector<bool> converged;
  int iterations_used = 0;
  bool all_converged() const {
    for (bool c : converged)
      if (!c) return false;
    return true;
  }
};

/// Matrix-free replacement of the dense H argument: K(X, X; theta) + sigma^2 I.
class KernelOperator {
 public:
  /// X: n x d column-major; constrained = [lengthscales (d), signal, noise].
  KernelOperator(b200::Device& dev, const std::vector<float>& X, std::int64_t n, int d,
                 const std::vector<double>& constrained)
      : dev_(dev), n_(n), d_(d) {
    b200::check(wgp_set_data(dev_.get(), X.data(), n, d));
    set_hyperparameters(constrained);
  }
  void set_hyperparameters(const std::vector<double>& constrained) {
    if (static_cast<int>(constrained.size()) != d_ + 2)
      throw std::invalid_argument("Hyperparameters: raw vector must have input_dim + 2 entries");
    b200::check(wgp_set_hyper(dev_.get(), constrained.data()));
  }
  /// out = H V (the products at proj/src/solvers.cpp:110 and friends).
  std::vector<float> apply(const std::vector<float>& V, int s) const {
    std::vector<float> out(static_cast<size_t>(n_) * s);
    b200::check(wgp_hv(dev_.get(), V.data(), s, out.data()));
    return out;
  }
  std::int64_t rows() const { return n_; }
  wgp_ctx* ctx() const { return dev_.get(); }

 private:
  b200::Device& dev_;
  std::int64_t n_;
  int d_;
};

/// solve(H, rhs, init, config) -- proj/src/solvers.cpp:265-279.
inline SolveState solve(const KernelOperator& H, const std::vector<float>& rhs, int s,
                        const std::vector<float>& init, const SolverConfig& config) {
  const size_t len = static_cast<size_t>(H.rows()) * s;
  if (rhs.size() != len) throw std::invalid_argument("solve: rhs row count mismatch");
  if (!init.empty() && init.size() != len) throw std::invalid_argument("solve: init shape must match rhs");
  SolveState st;
  st.solutions.resize(len);
  st.residuals.resize(len);
  st.per_column_relative_residual.resize(s);
  std::vector<int> conv(s);
  wgp_solve_state cs{st.solutions.data(), st.residuals.data(), st.per_column_relative_residual.data(),
                     conv.data(), 0};
  const wgp_solver_cfg cfg = config.c();
  b200::check(wgp_solve(H.ctx(), &cfg, rhs.data(), init.empty() ? nullptr : init.data(), s, &cs));
  st.converged.assign(conv.begin(), conv.end());
  st.iterations_used = cs.iterations_used;
  return st;
}

/// Zero-initialized overload (proj/src/solvers.cpp:281-284).
inline SolveState solve(const KernelOperator& H, const std::vector<float>& rhs, int s,
                        const SolverConfig& config) {
  return solve(H, rhs, s, {}, config);
}

enum class TrainMode { WarmStartFixedProbes = 0, ColdStartResampled = 1, ColdStartFixedProbes = 2 };

/// proj/include/warmgp/optimizer.hpp:23-38 plus the BASELINE extensions.
struct TrainConfig {
  int steps = 100;
  double learning_rate = 0.1;
  double adam_beta1 = 0.9;
  double adam_beta2 = 0.999;
  double adam_eps = 1e-8;
  int num_probes = 16;
  int probe_distribution = 0;  // 0 gaussian, 1 rademacher
  TrainMode mode = TrainMode::WarmStartFixedProbes;
  SolverConfig solver;
  double init_constrained = 1.0;
  std::uint64_t seed = 0;
  int transform = WGP_TRANSFORM_SOFTPLUS;
  int estimator = 0;  // 0 hutchinson, 1 pathwise RFF
  int rff_features = 1000;
  double init_noise = 0.0;
  double init_signal = 0.0;
  bool warm_start_distance = true;
};

/// proj/include/warmgp/optimizer.hpp:54-67 (device times instead of wall clock).
struct StepRecord {
  int step = 0;
  std::vector<double> raw_params, constrained_params, gradient, per_column_relative_residual;
  int solver_iterations = 0;
  double solver_ms = 0.0, step_ms = 0.0, warm_start_distance = 0.0;
  std::uint64_t probe_seed = 0;
};

struct OptTrace {
  std::vector<StepRecord> steps;
  const StepRecord& back() const { return steps.back(); }
};

namespace detail {
inline OptTrace run_loop(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                         std::int64_t n, int d, const TrainConfig& c, bool exact_gradients);
}  // namespace detail

/// train(X, y, config) -- proj/src/optimizer.cpp:175-177.
inline OptTrace train(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                      std::int64_t n, int d, const TrainConfig& c) {
  return detail::run_loop(dev, X, y, n, d, c, false);
}

/// train_exact(X, y, config) -- proj/src/optimizer.cpp:179-181: the same loop
/// with the exact Cholesky gradient (fp64 on the device, n <= 20000).
inline OptTrace train_exact(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                            std::int64_t n, int d, const TrainConfig& c) {
  return detail::run_loop(dev, X, y, n, d, c, true);
}

/// exact_mll / exact_gradient -- proj/src/exact.cpp:25-50 (raw-space gradient;
/// `transform` as TrainConfig::transform).
inline double exact_mll(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                        std::int64_t n, int d, const std::vector<double>& raw, int transform = WGP_TRANSFORM_SOFTPLUS) {
  b200::check(wgp_set_data(dev.get(), X.data(), n, d));
  double m = 0.0;
  b200::check(wgp_exact(dev.get(), transform, raw.data(), y.data(), &m, nullptr));
  return m;
}
inline std::vector<double> exact_gradient(b200::Device& dev, const std::vector<float>& X,
                                          const std::vector<float>& y, std::int64_t n, int d,
                                          const std::vector<double>& raw, int transform = WGP_TRANSFORM_SOFTPLUS) {
  b200::check(wgp_set_data(dev.get(), X.data(), n, d));
  std::vector<double> g(d + 2);
  b200::check(wgp_exact(dev.get(), transform, raw.data(), y.data(), nullptr, g.data()));
  return g;
}

inline OptTrace detail::run_loop(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                                 std::int64_t n, int d, const TrainConfig& c, bool exact_gradients) {
  if (static_cast<std::int64_t>(y.size()) != n) throw std::invalid_argument("train: X and y disagree on n");
  b200::check(wgp_set_data(dev.get(), X.data(), n, d));
  const int T = c.steps, p = d + 2, sp = c.num_probes + 1;
  std::vector<double> raw(T * p), con(T * p), grad(T * p), pcr(T * sp), wsd(T), sms(T), tms(T);
  std::vector<int> it(T);
  std::vector<std::uint64_t> seeds(T);
  wgp_train_cfg cfg{c.steps, c.learning_rate, c.adam_beta1, c.adam_beta2, c.adam_eps, c.num_probes,
                    c.probe_distribution, static_cast<int>(c.mode), c.solver.c(), c.init_constrained,
                    c.seed, c.transform, c.estimator, c.rff_features, c.init_noise, c.init_signal,
                    c.warm_start_distance ? 1 : 0, exact_gradients ? 1 : 0};
  wgp_trace tr{raw.data(), con.data(), grad.data(), it.data(), pcr.data(), wsd.data(), seeds.data(),
               sms.data(), tms.data(), nullptr};
  b200::check(wgp_train(dev.get(), y.data(), &cfg, &tr));
  OptTrace out;
  for (int t = 0; t < T; ++t) {
    StepRecord r;
    r.step = t + 1;
    r.raw_params.assign(raw.begin() + t * p, raw.begin() + (t + 1) * p);
    r.constrained_params.assign(con.begin() + t * p, con.begin() + (t + 1) * p);
    r.gradient.assign(grad.begin() + t * p, grad.begin() + (t + 1) * p);
    r.per_column_relative_residual.assign(pcr.begin() + t * sp, pcr.begin() + (t + 1) * sp);
    r.solver_iterations = it[t];
    r.solver_ms = sms[t];
    r.step_ms = tms[t];
    r.warm_start_distance = wsd[t];
    r.probe_seed = seeds[t];
    out.steps.push_back(std::move(r));
  }
  return out;
}

}  // namespace warmgp
