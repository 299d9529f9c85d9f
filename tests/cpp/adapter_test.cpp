// C++ adapter smoke test: the reference-shaped API (include/warmgp_b200.hpp)
// driving the B200 library, the way a warmgp maintainer would call it.
// Exit codes follow proj/tools/main.cpp:336-358 (3 = NumericalError).
#include <cmath>
#include <cstdio>
#include <random>

#include "warmgp_b200.hpp"

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
