// warmgp_b200.hpp — C++ adapter that keeps the reference warmgp API shape
// (proj/include/warmgp/{solvers,estimator,optimizer}.hpp) over the C-ABI in
// warmgp_b200.h.  Header-only; link against libwarmgp_b200.so.
//
// What changes for a caller of the reference: the dense `const Eigen::MatrixXd& H`
// argument of solve() (proj/include/warmgp/solvers.hpp:50-55) becomes a
// matrix-free KernelOperator (inputs X + hyperparameters, never H).  Two
// spellings of every entry point:
//   * the reference's own, on fp64 dense matrices: any column-major matrix
//     type with rows(), cols() and data() over doubles -- Eigen::MatrixXd /
//     VectorXd as the reference holds them (no Eigen include needed here):
//     train(X, y, config), solve(H, rhs, init, config) -> SolveStateT<MatrixXd>;
//   * plain column-major std::vector<float> with explicit sizes (the fp32
//     storage the device computes in).
// train(X, y, config) runs on b200::default_device() (device 0, created on
// first use; set WGP_DEVICE to pick another).
// Exceptions are the reference's: std::invalid_argument (status 2),
// warmgp::NumericalError (status 3, same message texts), std::runtime_error
// for device failures (status 4).
#pragma once

#include <cstdint>
#include <cstdlib>
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
  /// CG's precision (WGP_CG_F64, the default: the reference's iteration counts;
  /// WGP_CG_F32: fp32 vectors over the tensor-core operator, faster).
  void set_cg_precision(int precision) { check(wgp_set_cg_precision(ctx_, precision)); }
  /// Join an NCCL communicator (one process per GPU); call before the data is set.
  void set_comm(int rank, int nranks, const unsigned char id[128]) { check(wgp_set_comm(ctx_, rank, nranks, id)); }

 private:
  wgp_ctx* ctx_ = nullptr;
};

/// The context behind the reference-signature entry points (one per thread:
/// the reference API is blocking and single-threaded).
inline Device& default_device() {
  thread_local Device dev([] {
    const char* e = std::getenv("WGP_DEVICE");
    return e ? std::atoi(e) : 0;
  }());
  return dev;
}

/// Column-major fp64 matrix (Eigen::MatrixXd / VectorXd) -> fp32 storage.
template <class Mat>
std::vector<float> to_f32(const Mat& m) {
  const std::size_t len = static_cast<std::size_t>(m.rows()) * static_cast<std::size_t>(m.cols());
  std::vector<float> out(len);
  const auto* p = m.data();
  for (std::size_t e = 0; e < len; ++e) out[e] = static_cast<float>(p[e]);
  return out;
}

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

  void validate() const {  // proj/src/solvers.cpp:31-37
    if (!(tol_mean > 0.0 && tol_mean < 1.0) || !(tol_samples > 0.0 && tol_samples < 1.0))
      throw std::invalid_argument("SolverConfig: tolerances must lie in (0, 1)");
    if (block_size < 1) throw std::invalid_argument("SolverConfig: block_size must be >= 1");
    if (minibatch_size < 1) throw std::invalid_argument("SolverConfig: minibatch_size must be >= 1");
    if (max_iterations < 0) throw std::invalid_argument("SolverConfig: max_iterations must be >= 0");
  }
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

/// SolveState with the reference's fp64 matrix members (solvers.hpp:38-46),
/// e.g. SolveStateT<Eigen::MatrixXd>.
template <class Mat>
struct SolveStateT {
  Mat solutions;
  Mat residuals;
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
    if (static_cast<std::int64_t>(X.size()) != n * d)
      throw std::invalid_argument("build_kernel_matrices: input dimension mismatch");
    b200::check(wgp_set_data(dev_.get(), X.data(), n, d));
    set_hyperparameters(constrained);
  }
  /// From the reference's fp64 inputs (Eigen::MatrixXd X, n x d).
  template <class Mat>
  KernelOperator(b200::Device& dev, const Mat& X, const std::vector<double>& constrained)
      : KernelOperator(dev, b200::to_f32(X), static_cast<std::int64_t>(X.rows()), static_cast<int>(X.cols()),
                       constrained) {}
  void set_hyperparameters(const std::vector<double>& constrained) {
    if (static_cast<int>(constrained.size()) != d_ + 2)
      throw std::invalid_argument("Hyperparameters: raw vector must have input_dim + 2 entries");
    b200::check(wgp_set_hyper(dev_.get(), constrained.data()));
  }
  /// out = H V (the products at proj/src/solvers.cpp:110 and friends).
  std::vector<float> apply(const std::vector<float>& V, int s) const {
    if (V.size() != static_cast<size_t>(n_) * s) throw std::invalid_argument("hv: V row count mismatch");
    std::vector<float> out(static_cast<size_t>(n_) * s);
    b200::check(wgp_hv(dev_.get(), V.data(), s, out.data()));
    return out;
  }
  /// out = H V in fp64 (the fp64 CG operator) on the reference's matrices.
  template <class Mat>
  Mat apply(const Mat& V) const {
    if (static_cast<std::int64_t>(V.rows()) != n_) throw std::invalid_argument("hv: V row count mismatch");
    Mat out(V.rows(), V.cols());
    b200::check(wgp_hv_f64(dev_.get(), V.data(), static_cast<int>(V.cols()), out.data()));
    return out;
  }
  std::int64_t rows() const { return n_; }
  wgp_ctx* ctx() const { return dev_.get(); }

 private:
  b200::Device& dev_;
  std::int64_t n_;
  int d_;
};

/// solve(H, rhs, init, config) -- proj/src/solvers.cpp:265-279 -- on the
/// reference's fp64 matrices (Eigen::MatrixXd rhs / init): wgp_solve_f64, so
/// fp64 CG takes and returns unrounded fp64.
template <class Mat>
SolveStateT<Mat> solve(const KernelOperator& H, const Mat& rhs, const Mat& init, const SolverConfig& config) {
  config.validate();
  if (static_cast<std::int64_t>(rhs.rows()) != H.rows()) throw std::invalid_argument("solve: rhs row count mismatch");
  if (rhs.cols() < 1) throw std::invalid_argument("solve: rhs needs at least one column");
  if (init.rows() != rhs.rows() || init.cols() != rhs.cols())
    throw std::invalid_argument("solve: init shape must match rhs");
  const int s = static_cast<int>(rhs.cols());
  SolveStateT<Mat> st;
  st.solutions = Mat(rhs.rows(), rhs.cols());
  st.residuals = Mat(rhs.rows(), rhs.cols());
  st.per_column_relative_residual.resize(s);
  std::vector<int> conv(s);
  wgp_solve_state_f64 cs{st.solutions.data(), st.residuals.data(), st.per_column_relative_residual.data(),
                         conv.data(), 0};
  const wgp_solver_cfg cfg = config.c();
  b200::check(wgp_solve_f64(H.ctx(), &cfg, rhs.data(), init.data(), s, &cs));
  st.converged.assign(conv.begin(), conv.end());
  st.iterations_used = cs.iterations_used;
  return st;
}
/// Zero-initialized overload (proj/src/solvers.cpp:281-284).
template <class Mat>
SolveStateT<Mat> solve(const KernelOperator& H, const Mat& rhs, const SolverConfig& config) {
  Mat init(rhs.rows(), rhs.cols());
  double* p = init.data();
  for (std::size_t e = 0, len = static_cast<std::size_t>(rhs.rows()) * rhs.cols(); e < len; ++e) p[e] = 0.0;
  return solve(H, rhs, init, config);
}

/// solve(H, rhs, init, config) on fp32 column-major storage.
inline SolveState solve(const KernelOperator& H, const std::vector<float>& rhs, int s,
                        const std::vector<float>& init, const SolverConfig& config) {
  config.validate();
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
  bool record_solver_state = false;  // keep per-step init / solutions (optimizer.hpp:35)
};

/// The constrained hyperparameters of a step (Hyperparameters' accessors,
/// proj/include/warmgp/kernel.hpp:19-50).
struct Hyperparameters {
  std::vector<double> lengthscales;
  double signal = 1.0, noise = 1.0;
  int input_dim() const { return static_cast<int>(lengthscales.size()); }
  double signal_scale() const { return signal; }
  double noise_scale() const { return noise; }
  std::vector<double> to_constrained_vector() const {
    std::vector<double> v(lengthscales);
    v.push_back(signal);
    v.push_back(noise);
    return v;
  }
};

/// proj/include/warmgp/optimizer.hpp:54-67 (device times instead of wall clock).
struct StepRecord {
  int step = 0;
  std::vector<double> raw_params, constrained_params, gradient, per_column_relative_residual;
  int solver_iterations = 0;
  double solver_ms = 0.0, step_ms = 0.0, warm_start_distance = 0.0;
  double warm_distance_ms = 0.0;  // part of step_ms spent on the warm-start-distance H.V
  std::uint64_t probe_seed = 0;
  std::vector<float> solver_init, solver_solutions;  // n x (num_probes + 1), with record_solver_state
};

struct OptTrace {
  std::vector<StepRecord> steps;
  const StepRecord& back() const { return steps.back(); }
  /// proj/src/optimizer.cpp:67-70.
  Hyperparameters final_hyperparameters(int input_dim) const {
    const std::vector<double>& c = steps.back().constrained_params;
    if (static_cast<int>(c.size()) != input_dim + 2)
      throw std::invalid_argument("Hyperparameters: raw vector must have input_dim + 2 entries");
    return Hyperparameters{std::vector<double>(c.begin(), c.begin() + input_dim), c[input_dim], c[input_dim + 1]};
  }
  /// Sum of solver iterations over 1-based steps [first, last] (clamped), :72-78.
  long total_solver_iterations(int first = 1, int last = 1 << 30) const {
    long total = 0;
    for (const StepRecord& r : steps)
      if (r.step >= first && r.step <= last) total += r.solver_iterations;
    return total;
  }
};

namespace detail {
inline OptTrace run_loop(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                         std::int64_t n, int d, const TrainConfig& c, bool exact_gradients);
}  // namespace detail

/// train(X, y, config) -- proj/src/optimizer.cpp:175-177 -- on fp32 storage.
inline OptTrace train(b200::Device& dev, const std::vector<float>& X, const std::vector<float>& y,
                      std::int64_t n, int d, const TrainConfig& c) {
  return detail::run_loop(dev, X, y, n, d, c, false);
}

/// train(X, y, config) with the reference's exact signature and types
/// (Eigen::MatrixXd X, Eigen::VectorXd y), on b200::default_device().
template <class MatX, class VecY>
OptTrace train(const MatX& X, const VecY& y, const TrainConfig& c) {
  return detail::run_loop(b200::default_device(), b200::to_f32(X), b200::to_f32(y),
                          static_cast<std::int64_t>(X.rows()), static_cast<int>(X.cols()), c, false);
}
/// train_exact(X, y, config), the reference's signature.
template <class MatX, class VecY>
OptTrace train_exact(const MatX& X, const VecY& y, const TrainConfig& c) {
  return detail::run_loop(b200::default_device(), b200::to_f32(X), b200::to_f32(y),
                          static_cast<std::int64_t>(X.rows()), static_cast<int>(X.cols()), c, true);
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
  if (n < 1) throw std::invalid_argument("train: dataset is empty");
  if (static_cast<std::int64_t>(X.size()) != n * d)
    throw std::invalid_argument("build_kernel_matrices: input dimension mismatch");
  if (c.steps < 1) throw std::invalid_argument("TrainConfig: steps must be >= 1");
  if (c.num_probes < 1) throw std::invalid_argument("TrainConfig: num_probes must be >= 1");
  c.solver.validate();
  b200::check(wgp_set_data(dev.get(), X.data(), n, d));
  const int T = c.steps, p = d + 2, sp = c.num_probes + 1;
  std::vector<double> raw(T * p), con(T * p), grad(T * p), pcr(T * sp), wsd(T), sms(T), tms(T), wms(T);
  std::vector<float> sinit, ssol;
  if (c.record_solver_state) {
    sinit.resize(static_cast<size_t>(T) * n * sp);
    ssol.resize(static_cast<size_t>(T) * n * sp);
  }
  std::vector<int> it(T);
  std::vector<std::uint64_t> seeds(T);
  wgp_train_cfg cfg{c.steps, c.learning_rate, c.adam_beta1, c.adam_beta2, c.adam_eps, c.num_probes,
                    c.probe_distribution, static_cast<int>(c.mode), c.solver.c(), c.init_constrained,
                    c.seed, c.transform, c.estimator, c.rff_features, c.init_noise, c.init_signal,
                    c.warm_start_distance ? 1 : 0, exact_gradients ? 1 : 0, c.record_solver_state ? 1 : 0};
  wgp_trace tr{raw.data(), con.data(), grad.data(), it.data(), pcr.data(), wsd.data(), seeds.data(),
               sms.data(), tms.data(), nullptr, wms.data(),
               c.record_solver_state ? sinit.data() : nullptr, c.record_solver_state ? ssol.data() : nullptr};
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
    r.warm_distance_ms = wms[t];
    r.probe_seed = seeds[t];
    if (c.record_solver_state) {
      const size_t len = static_cast<size_t>(n) * sp;
      r.solver_init.assign(sinit.begin() + t * len, sinit.begin() + (t + 1) * len);
      r.solver_solutions.assign(ssol.begin() + t * len, ssol.begin() + (t + 1) * len);
    }
    out.steps.push_back(std::move(r));
  }
  return out;
}

}  // namespace warmgp
