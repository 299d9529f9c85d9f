// C++ adapter smoke test: the reference-shaped API (include/warmgp_b200.hpp)
// driving the B200 library, the way a warmgp maintainer would call it.
// Exit codes follow proj/tools/main.cpp:336-358 (3 = NumericalError).
#include <cmath>
#include <cstdio>
#include <random>

#include "warmgp_b200.hpp"

// Minimal stand-in for Eigen::MatrixXd / VectorXd (Eigen is not in this
// image): column-major doubles with rows(), cols(), data() and (r, c)
// construction -- the surface the adapter's fp64 entry points use.
struct MatrixXd {
  long r = 0, c = 0;
  std::vector<double> v;
  MatrixXd() = default;
  MatrixXd(long rows, long cols) : r(rows), c(cols), v(static_cast<size_t>(rows * cols)) {}
  long rows() const { return r; }
  long cols() const { return c; }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  double& operator()(long i, long j) { return v[static_cast<size_t>(i + j * r)]; }
  double operator()(long i, long j) const { return v[static_cast<size_t>(i + j * r)]; }
};

int main() {
  try {
    const int n = 600, d = 3, s = 4;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> normal(0.0, 1.0);
    std::vector<float> X(n * d), rhs(n * s);
    for (auto& v : X) v = static_cast<float>(normal(rng));
    for (auto& v : rhs) v = static_cast<float>(normal(rng));
    warmgp::b200::Device dev(0);
    warmgp::KernelOperator H(dev, X, n, d, {1.0, 0.8, 1.3, 1.1, 0.5});
    for (auto kind : {warmgp::SolverKind::Cg, warmgp::SolverKind::Ap, warmgp::SolverKind::Sgd}) {
      warmgp::SolverConfig cfg;
      cfg.kind = kind;
      cfg.tol_mean = cfg.tol_samples = 1e-3;
      cfg.block_size = 100;
      cfg.minibatch_size = n;
      cfg.learning_rate = 1.0;
      cfg.max_iterations = 100000;
      const warmgp::SolveState st = warmgp::solve(H, rhs, s, cfg);
      if (!st.all_converged()) return 1;
      // exact warm start -> zero passes (proj/tests/solvers_test.cpp:55-68)
      const warmgp::SolveState w = warmgp::solve(H, rhs, s, st.solutions, cfg);
      if (w.iterations_used != 0) return 1;
      std::printf("kind %d: %d iterations, residual[0] %.2e\n", static_cast<int>(kind), st.iterations_used,
                  st.per_column_relative_residual[0]);
    }
    warmgp::TrainConfig tc;
    tc.steps = 3;
    tc.num_probes = 4;
    std::vector<float> y(n);
    for (auto& v : y) v = static_cast<float>(normal(rng));
    const warmgp::OptTrace tr = warmgp::train(dev, X, y, n, d, tc);
    std::printf("train: %zu steps, noise %.4f\n", tr.steps.size(), tr.back().constrained_params[d + 1]);
    // exact path (proj/src/exact.cpp:25-50): the gradient matches central
    // differences of the exact MLL (proj/tests/kernel_test.cpp FD checks)
    const std::vector<double> raw0 = {0.1, -0.2, 0.3, 0.05, -0.4};
    const std::vector<double> g = warmgp::exact_gradient(dev, X, y, n, d, raw0);
    for (int k = 0; k < d + 2; ++k) {
      std::vector<double> rp = raw0, rm = raw0;
      const double h = 1e-5;
      rp[k] += h;
      rm[k] -= h;
      const double fd = (warmgp::exact_mll(dev, X, y, n, d, rp) - warmgp::exact_mll(dev, X, y, n, d, rm)) / (2 * h);
      if (std::fabs(fd - g[k]) > 1e-5 * (1.0 + std::fabs(g[k]))) {
        std::fprintf(stderr, "exact gradient %d: %.10g vs finite difference %.10g\n", k, g[k], fd);
        return 1;
      }
    }
    const warmgp::OptTrace te = warmgp::train_exact(dev, X, y, n, d, tc);
    std::printf("train_exact: %zu steps, noise %.4f\n", te.steps.size(), te.back().constrained_params[d + 1]);
    // non-finite inputs are std::invalid_argument (proj/src/solvers.cpp:58-67)
    rhs[0] = NAN;
    try {
      warmgp::solve(H, rhs, s, warmgp::SolverConfig{});
      return 1;
    } catch (const std::invalid_argument&) {
    }
    // the reference's own signatures on fp64 matrices (solvers.hpp:50-55,
    // optimizer.hpp:81): solve(H, rhs, init, config), train(X, y, config)
    MatrixXd Xd(n, d), Bd(n, s), yd(n, 1);
    for (long e = 0; e < n * d; ++e) Xd.v[e] = X[e];
    for (long e = 0; e < n * s; ++e) Bd.v[e] = normal(rng);
    for (long e = 0; e < n; ++e) yd.v[e] = y[e];
    warmgp::KernelOperator H64(dev, Xd, {1.0, 0.8, 1.3, 1.1, 0.5});
    warmgp::SolverConfig c64;
    c64.tol_mean = c64.tol_samples = 1e-6;
    c64.max_iterations = 5000;
    const warmgp::SolveStateT<MatrixXd> s64 = warmgp::solve(H64, Bd, c64);
    if (!s64.all_converged() || s64.solutions.rows() != n || s64.solutions.cols() != s) return 1;
    // the fp64 operator reproduces rhs from the fp64 solutions to the tolerance
    const MatrixXd HX = H64.apply(s64.solutions);
    for (int j = 0; j < s; ++j) {
      double num = 0, den = 0;
      for (long i = 0; i < n; ++i) {
        num += (Bd(i, j) - HX(i, j)) * (Bd(i, j) - HX(i, j));
        den += Bd(i, j) * Bd(i, j);
      }
      if (std::sqrt(num / den) > 1.01e-6) return 1;
    }
    const warmgp::SolveStateT<MatrixXd> w64 = warmgp::solve(H64, Bd, s64.solutions, c64);
    if (w64.iterations_used != 0) return 1;
    warmgp::TrainConfig rc;
    rc.steps = 4;
    rc.num_probes = 3;
    rc.record_solver_state = true;
    const warmgp::OptTrace tw = warmgp::train(Xd, yd, rc);
    // optimizer_test.cpp:113-124: warm init of step t = solutions of step t-1, zero at step 1
    for (float v : tw.steps[0].solver_init)
      if (v != 0.f) return 1;
    for (int t = 1; t < rc.steps; ++t)
      if (tw.steps[t].solver_init != tw.steps[t - 1].solver_solutions) return 1;
    rc.mode = warmgp::TrainMode::ColdStartFixedProbes;  // :130-134: cold init is zero every step
    const warmgp::OptTrace tc0 = warmgp::train(Xd, yd, rc);
    for (const auto& r : tc0.steps)
      for (float v : r.solver_init)
        if (v != 0.f) return 1;
    const warmgp::Hyperparameters fh = tw.final_hyperparameters(d);
    if (fh.input_dim() != d || fh.noise_scale() != tw.back().constrained_params[d + 1]) return 1;
    if (tw.total_solver_iterations() != tw.total_solver_iterations(1, rc.steps) ||
        tw.total_solver_iterations(2, 3) != tw.steps[1].solver_iterations + tw.steps[2].solver_iterations)
      return 1;
    std::printf("fp64 solve: %d iterations; train(X, y, config): noise %.4f, %ld iterations\n", s64.iterations_used,
                fh.noise_scale(), tw.total_solver_iterations());
    // shape errors are std::invalid_argument with the reference's messages
    try {
      warmgp::solve(H64, MatrixXd(n - 1, s), c64);
      return 1;
    } catch (const std::invalid_argument& e) {
      if (std::string(e.what()) != "solve: rhs row count mismatch") return 1;
    }
    std::printf("adapter ok\n");
    return 0;
  } catch (const warmgp::NumericalError& e) {
    std::fprintf(stderr, "numerical: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  }
}
