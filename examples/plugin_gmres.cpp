// plugin_gmres.cpp -- the reference's generic plugin interface against the B200 library:
// gmres_right(n, apply_a, apply_pinv, b, cfg) with host callables (krylov.hpp:83-85), here the
// library's own operators behind make_apply_a / make_apply_pinv (host staging per call), compared
// with the device-resident gmres_right(op, plan, b, cfg); plus the AlphaCirculantPlan fields the
// reference exposes (alpha_circulant.hpp:52-67).
//   g++ -std=c++20 -O2 -Iinclude examples/plugin_gmres.cpp \
//       -Lpaper_2003_07020_b200 -lfracpint_b200 -Wl,-rpath,$PWD/paper_2003_07020_b200
// Prints: iterations_device iterations_generic rel_x_diff TRR_generic alpha scale_fwd[1]
//         scale_bwd[1]*scale_fwd[1] sigma[0] solve_count tau.n
#include <fracpint_b200.hpp>

#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

namespace fb = fracpint::b200;

int main() {
  const int h_inv = 256, n_time = 64;
  const double gamma = 1.5, kappa = 1.0, h = 1.0 / h_inv, dt = 1.0 / n_time;
  const int n_space = h_inv - 1;
  fb::TimeStencil stencil(n_time);
  fb::AllAtOnceOperator op(stencil, fb::RieszJacobian1D(gamma, kappa, h, n_space), dt);
  std::vector<double> u0(n_space), f(std::size_t(n_space) * n_time);
  for (int i = 0; i < n_space; ++i) {
    const double x = (i + 1) * h;
    u0[i] = x * x * (1 - x) * (1 - x);
  }
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (double& v : f) v = U(rng);
  const std::vector<double> b = fb::assemble_rhs(stencil, dt, f, u0);
  auto plan = fb::build_plan(fb::PreconditionerKind::generalized(), n_time, dt, op);
  fb::SolverConfig cfg;
  cfg.tol = 1e-10;
  auto dev = fb::gmres_right(op, plan, b, cfg);
  auto gen = fb::gmres_right(op.dim(), fb::make_apply_a(op), fb::make_apply_pinv(plan), b, cfg);
  double d2 = 0, x2 = 0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    d2 += (dev.x[i] - gen.x[i]) * (dev.x[i] - gen.x[i]);
    x2 += dev.x[i] * dev.x[i];
  }
  // a throwing callable aborts the solve with its own exception, as in the reference
  bool rethrown = false;
  try {
    fb::gmres_right(op.dim(), [](std::span<const double>, std::span<double>) { throw std::logic_error("boom"); },
                    fb::make_apply_pinv(plan), b, cfg);
  } catch (const std::logic_error&) {
    rethrown = true;
  }
  std::printf("%g %g %.3e %.3e %.17g %.17g %.17g %.17g %d %d %d\n", dev.report.iterations, gen.report.iterations,
              std::sqrt(d2 / x2), gen.report.true_relative_residual, plan.alpha, plan.scale_fwd[1],
              plan.scale_bwd[1] * plan.scale_fwd[1], plan.tau.sigma[0], plan.solve_count, plan.tau.n,
              rethrown ? 1 : 0);
  return (dev.report.converged && gen.report.converged && rethrown) ? 0 : 3;
}
