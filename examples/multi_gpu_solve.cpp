// multi_gpu_solve.cpp -- the all-at-once solve sharded over several GPUs of one process through the
// drop-in header (fracpint::b200::MultiDevice / ShardedOperator over fpc_multi_* / fpc_sharded_*):
// time-sharded Krylov vectors, peer-store transpositions around the frequency-sharded tau solves.
//   g++ -std=c++20 -O2 -Iinclude examples/multi_gpu_solve.cpp \
//       -Lpaper_2003_07020_b200 -lfracpint_b200 -Wl,-rpath,$PWD/paper_2003_07020_b200
//   ./a.out 0 1 2 3        (device list; a device may repeat: ./a.out 0 0 runs 2 ranks on GPU 0)
// Prints: ranks iterations_sharded iterations_single rel_x_diff TRR
#include <fracpint_b200.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace fb = fracpint::b200;

int main(int argc, char** argv) {
  std::vector<int> devices;
  for (int i = 1; i < argc; ++i) devices.push_back(std::atoi(argv[i]));
  if (devices.empty()) devices = {0};
  const int h_inv = 1024, n_time = 256, n_space = h_inv - 1;
  const double gamma = 1.5, h = 1.0 / h_inv, dt = 1.0 / n_time;
  fb::TimeStencil stencil(n_time);
  fb::RieszJacobian1D jac(gamma, 1.0, h, n_space);
  std::vector<double> u0(n_space), f(std::size_t(n_space) * n_time);
  for (int i = 0; i < n_space; ++i) {
    const double x = (i + 1) * h;
    u0[i] = x * x * (1 - x) * (1 - x);
  }
  std::mt19937_64 rng(20260819);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (double& v : f) v = U(rng);
  const std::vector<double> b = fb::assemble_rhs(stencil, dt, f, u0);
  fb::SolverConfig cfg;
  cfg.tol = 1e-10;
  cfg.restart = 20;

  fb::MultiDevice md(devices);
  fb::ShardedOperator<fb::RieszJacobian1D> sop(md, stencil, jac, dt);
  const auto rs = sop.gmres_right(b, cfg);

  fb::AllAtOnceOperator op(stencil, jac, dt);
  const auto plan = fb::build_plan(fb::PreconditionerKind::generalized(), n_time, dt, op);
  const auto r1 = fb::gmres_right(op, plan, b, cfg);
  double d2 = 0, x2 = 0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    d2 += (rs.x[i] - r1.x[i]) * (rs.x[i] - r1.x[i]);
    x2 += r1.x[i] * r1.x[i];
  }
  std::printf("%zu %g %g %.3e %.3e\n", devices.size(), rs.report.iterations, r1.report.iterations, std::sqrt(d2 / x2),
              rs.report.true_relative_residual);
  return rs.report.converged ? 0 : 3;
}
