// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/fracpint/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libfracpint_ref.so.  TEST / BASELINE INFRASTRUCTURE ONLY: it pins the C oracle
// (tests/test_oracle_pins.py), generates tests/golden fixtures (tests/golden/make_golden.py) and
// is the CPU reference arm of bench.py (--impl reference, cpu_baseline kind "reference").
// No reference source is copied: this file only calls the reference's public API
// (driver.hpp:49-92 orchestration pattern).
#include <fracpint/all_at_once.hpp>
#include <fracpint/driver.hpp>
#include <fracpint/problems.hpp>
#include <fracpint/alpha_circulant.hpp>
#include <fracpint/dst.hpp>
#include <fracpint/jacobian.hpp>
#include <fracpint/krylov.hpp>
#include <fracpint/parallel.hpp>
#include <fracpint/tau.hpp>
#include <fracpint/time_stencil.hpp>
#include <fracpint/toeplitz.hpp>
#include <fracpint/weights.hpp>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <complex>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

using fracpint::AllAtOnceOperator;
using fracpint::RieszJacobian1D;
using fracpint::RieszJacobian2D;

struct RefProblem {
  int nt = 0;
  double dt = 0.0;
  std::variant<AllAtOnceOperator<RieszJacobian1D>, AllAtOnceOperator<RieszJacobian2D>> op;
  std::optional<fracpint::AlphaCirculantPlan> plan;

  template <class J>
  RefProblem(int nt_, double dt_, J jac)
      : nt(nt_), dt(dt_), op(AllAtOnceOperator<J>(fracpint::TimeStencil(nt_), std::move(jac), dt_)) {}

  std::size_t dim() const {
    return std::visit([](const auto& o) { return o.dim(); }, op);
  }
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { fracpint::set_thread_count(n); }
int ref_threads() { return fracpint::thread_count(); }

void ref_fft_inplace(double* x, std::size_t n, int sign) {
  fracpint::fft_inplace(reinterpret_cast<std::complex<double>*>(x), n, sign);
}
int ref_dst1_real(const double* x, double* y, std::size_t n) {
  return guarded([&] { fracpint::dst1<double>({x, n}, {y, n}); });
}
int ref_dst1_complex(const double* x, double* y, std::size_t n) {
  using C = std::complex<double>;
  return guarded([&] {
    std::vector<C> in(reinterpret_cast<const C*>(x), reinterpret_cast<const C*>(x) + n);
    fracpint::dst1<C>(in, {reinterpret_cast<C*>(y), n});
  });
}
int ref_centred_weights(double gamma, int count, double* out) {
  return guarded([&] {
    auto fw = fracpint::centred_weights(gamma, count);
    std::copy(fw.weights.begin(), fw.weights.end(), out);
  });
}
int ref_toeplitz_matvec(const double* col, std::size_t n, const double* v, double* out) {
  return guarded([&] {
    fracpint::SymToeplitz t(std::vector<double>(col, col + n));
    t.matvec<double>({v, n}, {out, n});
  });
}
int ref_tau_spectrum(const double* col, std::size_t n, double* sigma) {
  return guarded([&] {
    auto tau = fracpint::tau_spectrum(fracpint::SymToeplitz(std::vector<double>(col, col + n)));
    std::copy(tau.sigma.begin(), tau.sigma.end(), sigma);
  });
}

void* ref_problem_1d(double gamma, double kappa, double h, int n, int nt, double dt) {
  RefProblem* p = nullptr;
  if (guarded([&] { p = new RefProblem(nt, dt, RieszJacobian1D(gamma, kappa, h, n)); })) return nullptr;
  return p;
}
void* ref_problem_2d(double gx, double gy, double kx, double ky, double h, int n, int nt,
                     double dt) {
  RefProblem* p = nullptr;
  if (guarded([&] { p = new RefProblem(nt, dt, RieszJacobian2D(gx, gy, kx, ky, h, n)); }))
    return nullptr;
  return p;
}
void ref_problem_free(void* p) { delete static_cast<RefProblem*>(p); }

int ref_matvec(void* hp, const double* v, double* out) {
  auto* p = static_cast<RefProblem*>(hp);
  const std::size_t n = p->dim();
  return guarded([&] { std::visit([&](const auto& o) { o.apply({v, n}, {out, n}); }, p->op); });
}

int ref_assemble_rhs(int nt, int ns, double dt, const double* f, const double* u0, double* b) {
  return guarded([&] {
    const std::size_t N = static_cast<std::size_t>(nt) * ns;
    auto r = fracpint::assemble_rhs(fracpint::TimeStencil(nt), dt, {f, N},
                                    {u0, static_cast<std::size_t>(ns)});
    std::copy(r.begin(), r.end(), b);
  });
}

// alpha <= 0 selects PreconditionerKind::generalized().
int ref_build_plan(void* hp, double alpha, double* min_margin, double* alpha_out) {
  auto* p = static_cast<RefProblem*>(hp);
  return guarded([&] {
    const auto kind = alpha <= 0.0 ? fracpint::PreconditionerKind::generalized()
                                   : fracpint::PreconditionerKind::with_alpha(alpha);
    std::visit([&](const auto& o) { p->plan = fracpint::build_plan(kind, p->nt, p->dt, o.jacobian()); },
               p->op);
    if (min_margin) *min_margin = p->plan->min_shift_margin;
    if (alpha_out) *alpha_out = p->plan->alpha;
  });
}

int ref_tau_sigma(void* hp, double* sigma) {
  auto* p = static_cast<RefProblem*>(hp);
  if (!p->plan) return 1;
  std::copy(p->plan->tau.sigma.begin(), p->plan->tau.sigma.end(), sigma);
  return 0;
}

int ref_pc_apply(void* hp, const double* v, double* out, int full_sweep) {
  auto* p = static_cast<RefProblem*>(hp);
  const std::size_t n = p->dim();
  return guarded([&] {
    if (!p->plan) throw std::invalid_argument("no plan");
    fracpint::apply_inverse(*p->plan, {v, n}, {out, n},
                            full_sweep ? fracpint::InnerSweep::full : fracpint::InnerSweep::half);
  });
}
int ref_pc_forward(void* hp, const double* v, double* out) {
  auto* p = static_cast<RefProblem*>(hp);
  const std::size_t n = p->dim();
  return guarded([&] {
    if (!p->plan) throw std::invalid_argument("no plan");
    fracpint::apply_forward(*p->plan, {v, n}, {out, n});
  });
}

// Manufactured benchmarks (problems.hpp:68-131) through the reference's run_problem
// (driver.hpp:84-112): dim 1 = example1(gx), dim 2 = example2(gx, gy).  strang != 0 selects
// PreconditionerKind::strang(), method 1 = bicgstab.  rhs_out (nt*ns) gets the assembled all-at-once
// right-hand side, exact_out (ns) the exact final state, final_out (ns) the computed one.
int ref_run_problem(int dim, double gx, double gy, int nt, int h_inv, int method, int strang,
                    double tol, int max_iter, double* iterations, int* converged, double* err_inf,
                    double* rhs_out, double* exact_out, double* final_out) {
  return guarded([&] {
    fracpint::RunConfig cfg;
    cfg.n_time = nt;
    cfg.h_inv = h_inv;
    cfg.kind = strang ? fracpint::PreconditionerKind::strang() : fracpint::PreconditionerKind::generalized();
    cfg.method = method == 1 ? fracpint::KrylovMethod::bicgstab : fracpint::KrylovMethod::gmres;
    cfg.solver.tol = tol;
    cfg.solver.max_iter = max_iter;
    fracpint::RunResult r;
    std::vector<double> u0, f, ex;
    double dt = 0.0;
    if (dim == 1) {
      const auto p = fracpint::example1(gx);
      fracpint::Grid1D g(p.a, p.b, h_inv);
      dt = p.t_final / nt;
      u0 = fracpint::sample_initial(p, g);
      f = fracpint::sample_source(p, g, dt, nt);
      ex = fracpint::sample_exact(p, g, p.t_final);
      r = fracpint::run_problem(p, cfg);
    } else {
      const auto p = fracpint::example2(gx, gy);
      fracpint::Grid2D g(p.ax, p.bx, p.ay, p.by, h_inv);
      dt = p.t_final / nt;
      u0 = fracpint::sample_initial(p, g);
      f = fracpint::sample_source(p, g, dt, nt);
      ex = fracpint::sample_exact(p, g, p.t_final);
      r = fracpint::run_problem(p, cfg);
    }
    *iterations = r.report.iterations;
    *converged = r.report.converged ? 1 : 0;
    *err_inf = r.err_inf;
    if (rhs_out) {
      auto b = fracpint::assemble_rhs(fracpint::TimeStencil(nt), dt, f, u0);
      std::copy(b.begin(), b.end(), rhs_out);
    }
    if (exact_out) std::copy(ex.begin(), ex.end(), exact_out);
    if (final_out) std::copy(r.final_state.begin(), r.final_state.end(), final_out);
  });
}

// bicgstab_left exactly as driver.hpp:68-71 wires it (KrylovMethod::bicgstab).
int ref_bicgstab(void* hp, const double* b, double* x, double tol, int max_iter, int* converged,
                 double* iterations, double* final_rel, double* true_rel, double* seconds,
                 double* history, int history_cap, int* history_len) {
  auto* p = static_cast<RefProblem*>(hp);
  const std::size_t n = p->dim();
  return guarded([&] {
    if (!p->plan) throw std::invalid_argument("no plan");
    fracpint::SolverConfig cfg;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    auto apply_pinv = [p](std::span<const double> in, std::span<double> out) {
      fracpint::apply_inverse(*p->plan, in, out);
    };
    fracpint::KrylovResult r = std::visit(
        [&](const auto& o) {
          auto apply_a = [&o](std::span<const double> in, std::span<double> out) { o.apply(in, out); };
          return fracpint::bicgstab_left(n, apply_a, apply_pinv, {b, n}, cfg);
        },
        p->op);
    std::copy(r.x.begin(), r.x.end(), x);
    *converged = r.report.converged ? 1 : 0;
    *iterations = r.report.iterations;
    *final_rel = r.report.final_relative_residual;
    *true_rel = r.report.true_relative_residual;
    *seconds = r.report.seconds;
    const int h = static_cast<int>(r.report.residual_history.size());
    *history_len = h;
    for (int i = 0; i < h && i < history_cap; ++i) history[i] = r.report.residual_history[i];
  });
}

// Unrestarted gmres_right exactly as driver.hpp:62-73 wires it.  Returns seconds =
// report.seconds (the reference's own timed span krylov.hpp:87-190).
int ref_gmres(void* hp, const double* b, double* x, double tol, int max_iter, int* converged,
              int* iterations, double* final_rel, double* true_rel, double* seconds,
              double* history, int history_cap, int* history_len) {
  auto* p = static_cast<RefProblem*>(hp);
  const std::size_t n = p->dim();
  return guarded([&] {
    if (!p->plan) throw std::invalid_argument("no plan");
    fracpint::SolverConfig cfg;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    auto apply_pinv = [p](std::span<const double> in, std::span<double> out) {
      fracpint::apply_inverse(*p->plan, in, out);
    };
    fracpint::KrylovResult r = std::visit(
        [&](const auto& o) {
          auto apply_a = [&o](std::span<const double> in, std::span<double> out) { o.apply(in, out); };
          return fracpint::gmres_right(n, apply_a, apply_pinv, {b, n}, cfg);
        },
        p->op);
    std::copy(r.x.begin(), r.x.end(), x);
    *converged = r.report.converged ? 1 : 0;
    *iterations = static_cast<int>(r.report.iterations);
    *final_rel = r.report.final_relative_residual;
    *true_rel = r.report.true_relative_residual;
    *seconds = r.report.seconds;
    const int h = static_cast<int>(r.report.residual_history.size());
    *history_len = h;
    for (int i = 0; i < h && i < history_cap; ++i) history[i] = r.report.residual_history[i];
  });
}

// GMRES(m) restart emulation (the reference has no restart) on top of the
// reference's own unrestarted gmres_right, exactly as driver.hpp:62-73 wires it:
//   r = b; x = 0; loop { d = gmres_right(r, tol*||b||/||r||, min(m, budget)); x += d.x;
//                        stop if d converged or the budget is spent; r = b - A x }.
// iterations = the sum of the inner counts; true_rel = ||b - A x|| / ||b|| (krylov.hpp:64-75);
// seconds = wall time of the whole loop.
int ref_gmres_restart(void* hp, const double* b, double* x, double tol, int max_iter, int restart,
                      int* converged, int* iterations, int* restarts, double* true_rel, double* seconds) {
  auto* p = static_cast<RefProblem*>(hp);
  const std::size_t n = p->dim();
  return guarded([&] {
    if (!p->plan) throw std::invalid_argument("no plan");
    const auto t0 = std::chrono::steady_clock::now();
    auto apply_pinv = [p](std::span<const double> in, std::span<double> out) {
      fracpint::apply_inverse(*p->plan, in, out);
    };
    auto apply_a = [p](std::span<const double> in, std::span<double> out) {
      std::visit([&](const auto& o) { o.apply(in, out); }, p->op);
    };
    auto nrm = [n](const std::vector<double>& v) {
      double s = 0.0;
      for (std::size_t i = 0; i < n; ++i) s += v[i] * v[i];
      return std::sqrt(s);
    };
    std::vector<double> bb(b, b + n), r(bb), xx(n, 0.0), ax(n);
    const double norm_b = nrm(bb);
    int budget = max_iter, its = 0, cycles = 0;
    bool conv = norm_b == 0.0;
    double norm_r = norm_b;
    while (!conv && budget > 0) {
      fracpint::SolverConfig cfg;
      cfg.tol = tol * norm_b / norm_r;
      cfg.max_iter = restart > 0 ? std::min(restart, budget) : budget;
      fracpint::KrylovResult d = fracpint::gmres_right(n, apply_a, apply_pinv, {r.data(), n}, cfg);
      for (std::size_t i = 0; i < n; ++i) xx[i] += d.x[i];
      const int k = static_cast<int>(d.report.iterations);
      its += k;
      budget -= k;
      ++cycles;
      if (d.report.converged) {
        conv = true;
        break;
      }
      if (k == 0) break;
      apply_a({xx.data(), n}, {ax.data(), n});
      for (std::size_t i = 0; i < n; ++i) r[i] = bb[i] - ax[i];
      norm_r = nrm(r);
    }
    apply_a({xx.data(), n}, {ax.data(), n});
    for (std::size_t i = 0; i < n; ++i) ax[i] = bb[i] - ax[i];
    *true_rel = norm_b > 0.0 ? nrm(ax) / norm_b : 0.0;
    std::copy(xx.begin(), xx.end(), x);
    *converged = conv ? 1 : 0;
    *iterations = its;
    *restarts = cycles > 0 ? cycles - 1 : 0;
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// The reference's own generic gmres_right (krylov.hpp:83-192) driving arbitrary C callbacks
// (the plugin interface krylov.hpp:83-85): out = op(in), return 0 on success.  Used to drive the
// B200 library's fpc_matvec / fpc_pc_apply from the unmodified reference Krylov layer.
typedef int (*ref_apply_fn)(const double* in, double* out, std::size_t n, void* user);
int ref_gmres_callbacks(std::size_t n, ref_apply_fn a, void* ua, ref_apply_fn pinv, void* up, const double* b,
                        double* x, double tol, int max_iter, int* converged, int* iterations, double* true_rel,
                        double* history, int history_cap, int* history_len) {
  return guarded([&] {
    fracpint::SolverConfig cfg;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    auto apply_a = [&](std::span<const double> in, std::span<double> out) {
      if (a(in.data(), out.data(), in.size(), ua) != 0) throw std::runtime_error("apply_a callback failed");
    };
    auto apply_pinv = [&](std::span<const double> in, std::span<double> out) {
      if (pinv(in.data(), out.data(), in.size(), up) != 0) throw std::runtime_error("apply_pinv callback failed");
    };
    fracpint::KrylovResult r = fracpint::gmres_right(n, apply_a, apply_pinv, {b, n}, cfg);
    std::copy(r.x.begin(), r.x.end(), x);
    *converged = r.report.converged ? 1 : 0;
    *iterations = static_cast<int>(r.report.iterations);
    *true_rel = r.report.true_relative_residual;
    const int h = static_cast<int>(r.report.residual_history.size());
    *history_len = h;
    for (int i = 0; i < h && i < history_cap; ++i) history[i] = r.report.residual_history[i];
  });
}

}  // extern "C"
