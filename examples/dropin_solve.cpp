// dropin_solve.cpp -- the reference's library-usage example (proj/README.md "Library usage")
// written against fracpint_b200.hpp: same names, same call sequence, GPU underneath.
//   g++ -std=c++20 -O2 -Iinclude examples/dropin_solve.cpp \
//       -Lpaper_2003_07020_b200 -lfracpint_b200 -Wl,-rpath,$PWD/paper_2003_07020_b200
// Prints one line: n_space n_time iterations TRR x_checksum
#include <fracpint_b200.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace fb = fracpint::b200;

int main(int argc, char** argv) {
  const int h_inv = argc > 1 ? std::atoi(argv[1]) : 256;
  const int n_time = argc > 2 ? std::atoi(argv[2]) : 64;
  const double gamma = 1.5, kappa = 1.0;
  const int n_space = h_inv - 1;
  const double h = 1.0 / h_inv, dt = 1.0 / n_time;

  fb::RieszJacobian1D jac(gamma, kappa, h, n_space);
  fb::TimeStencil stencil(n_time);
  fb::AllAtOnceOperator op(stencil, jac, dt);
  std::vector<double> u0(n_space), f(std::size_t(n_space) * n_time);
  for (int i = 0; i < n_space; ++i) {
    const double x = (i + 1) * h;
    u0[i] = x * x * (1 - x) * (1 - x);
  }
  std::mt19937_64 rng(20260819);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (double& v : f) v = U(rng);
  const std::vector<double> b = fb::assemble_rhs(stencil, dt, f, u0);

  auto plan = fb::build_plan(fb::PreconditionerKind::generalized(), n_time, dt, op);
  fb::SolverConfig cfg;
  cfg.tol = 1e-10;
  auto result = fb::gmres_right(op, plan, b, cfg);

  // the reference's plugin interface: the callables work with its generic GMRES too
  std::vector<double> ax(b.size());
  auto apply_a = fb::make_apply_a(op);
  apply_a(result.x, ax);
  double r2 = 0, b2 = 0, cs = 0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    r2 += (b[i] - ax[i]) * (b[i] - ax[i]);
    b2 += b[i] * b[i];
    cs += result.x[i] * double(1 + (i % 7));
  }
  std::printf("%d %d %g %.3e %.3e %.17g\n", n_space, n_time, result.report.iterations,
              result.report.true_relative_residual, std::sqrt(r2 / b2), cs);
  return result.report.converged ? 0 : 3;
}
