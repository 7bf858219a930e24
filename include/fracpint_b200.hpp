// fracpint_b200.hpp -- C++20 drop-in for the reference's solver API (namespace fracpint,
// /root/reference/proj/include/fracpint/*.hpp) over the C-ABI of libfracpint_b200.so.
//
// Same names, argument meaning and exceptions as the reference, in namespace fracpint::b200:
//   TimeStencil                      time_stencil.hpp:16-26
//   RieszJacobian1D / RieszJacobian2D jacobian.hpp:19-105 (parameters; spectra built by the library)
//   AllAtOnceOperator<J>             all_at_once.hpp:18-61   (apply = fpc_matvec)
//   assemble_rhs                     all_at_once.hpp:66-80
//   PreconditionerKind, InnerSweep   alpha_circulant.hpp:23-42, 128
//   AlphaCirculantPlan, build_plan   alpha_circulant.hpp:52-126 (fpc_plan_create)
//   apply_inverse / apply_forward    alpha_circulant.hpp:206-215 (fpc_pc_apply / fpc_pc_forward)
//   SolverConfig/SolveReport/KrylovResult, gmres_right   krylov.hpp:25-42, 83-192 (fpc_gmres)
//   gmres_right(n, apply_a, apply_pinv, b, cfg) for any host callables  krylov.hpp:83-85
//                                    (fpc_gmres_callbacks: basis on the device)
//   TauOperator                      tau.hpp:20-26 (AlphaCirculantPlan::tau)
//   MultiDevice / ShardedOperator    one process over 1..8 GPUs (fpc_multi_*, fpc_sharded_*)
// plus SolverConfig::restart (GMRES(m); 0 = the reference's unrestarted GMRES).
//
// Two ways to use it:
//   * the device-resident solve: gmres_right(op, plan, b, cfg) -- the whole iteration in HBM;
//   * the reference's own plugin interface: make_apply_a(op) / make_apply_pinv(plan) return the
//     void(std::span<const double>, std::span<double>) callables the reference's generic
//     fracpint::gmres_right(n, apply_a, apply_pinv, b, cfg) takes (krylov.hpp:83-85), each call
//     one host<->device round trip through the C-ABI.
#pragma once

#include <fracpint_b200.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <exception>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace fracpint::b200 {

namespace detail {
inline void check(int rc) {
  if (rc == FPC_OK) return;
  const std::string msg = fpc_last_error();
  if (rc == FPC_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);  // runtime_error, CUDA failure, unsupported size
}
}  // namespace detail

class Context {
 public:
  explicit Context(int device = 0) {
    fpc_context_t h = nullptr;
    detail::check(fpc_context_create(device, &h));
    h_.reset(h, [](fpc_context_t c) { fpc_context_destroy(c); });
  }
  static Context& default_context() {
    static Context ctx(0);
    return ctx;
  }
  fpc_context_t handle() const { return h_.get(); }
  void synchronize() const { detail::check(fpc_synchronize(h_.get())); }

 private:
  std::shared_ptr<fpc_context_s> h_;
};

struct TimeStencil {
  static constexpr double r0 = 1.5, r1 = -2.0, r2 = 0.5;
  int n_time = 0;
  explicit TimeStencil(int nt) : n_time(nt) {
    if (nt < 3) throw std::invalid_argument("TimeStencil: need at least 3 time levels");
  }
};

struct RieszJacobian1D {
  double gamma, kappa, h;
  int n;
  RieszJacobian1D(double gamma_, double kappa_, double h_, int n_space)
      : gamma(gamma_), kappa(kappa_), h(h_), n(n_space) {
    if (!(kappa > 0.0)) throw std::invalid_argument("RieszJacobian1D: kappa must be positive");
    if (!(h > 0.0)) throw std::invalid_argument("RieszJacobian1D: h must be positive");
    if (n_space < 1) throw std::invalid_argument("RieszJacobian1D: n_space must be at least 1");
  }
  int dim() const { return n; }
};

struct RieszJacobian2D {
  double gamma_x, gamma_y, kappa_x, kappa_y, h;
  int n;
  RieszJacobian2D(double gx, double gy, double kx, double ky, double h_, int n_per_dim)
      : gamma_x(gx), gamma_y(gy), kappa_x(kx), kappa_y(ky), h(h_), n(n_per_dim) {
    if (!(kx > 0.0) || !(ky > 0.0))
      throw std::invalid_argument("RieszJacobian2D: diffusion coefficients must be positive");
    if (!(h > 0.0)) throw std::invalid_argument("RieszJacobian2D: h must be positive");
    if (n_per_dim < 1) throw std::invalid_argument("RieszJacobian2D: n_per_dim must be at least 1");
  }
  int dim() const { return n * n; }
  int n_per_dim() const { return n; }
};

template <class Jacobian>
class AllAtOnceOperator {
 public:
  AllAtOnceOperator(TimeStencil stencil, Jacobian jac, double dt,
                    Context& ctx = Context::default_context())
      : stencil_(stencil), jac_(jac), dt_(dt), ctx_(ctx) {
    if (!(dt > 0.0)) throw std::invalid_argument("AllAtOnceOperator: dt must be positive");
    fpc_problem_t h = nullptr;
    if constexpr (std::is_same_v<Jacobian, RieszJacobian1D>)
      detail::check(fpc_problem_create_1d(ctx.handle(), jac.gamma, jac.kappa, jac.h, jac.n,
                                          stencil.n_time, dt, &h));
    else
      detail::check(fpc_problem_create_2d(ctx.handle(), jac.gamma_x, jac.gamma_y, jac.kappa_x,
                                          jac.kappa_y, jac.h, jac.n, stencil.n_time, dt, &h));
    h_.reset(h, [](fpc_problem_t p) { fpc_problem_destroy(p); });
  }
  int n_time() const { return stencil_.n_time; }
  int n_space() const { return jac_.dim(); }
  std::size_t dim() const { return std::size_t(n_time()) * std::size_t(n_space()); }
  double dt() const { return dt_; }
  const TimeStencil& stencil() const { return stencil_; }
  const Jacobian& jacobian() const { return jac_; }
  fpc_problem_t handle() const { return h_.get(); }

  // host spans (all_at_once.hpp:33)
  void apply(std::span<const double> v, std::span<double> out) const {
    if (v.size() != dim() || out.size() != dim())
      throw std::invalid_argument("AllAtOnceOperator::apply: size mismatch");
    detail::check(fpc_matvec(h_.get(), v.data(), out.data(), FPC_HOST));
  }
  // device pointers, stream-ordered on the context stream
  void apply_device(const double* v, double* out) const {
    detail::check(fpc_matvec(h_.get(), v, out, FPC_DEVICE));
  }

 private:
  TimeStencil stencil_;
  Jacobian jac_;
  double dt_;
  Context& ctx_;
  std::shared_ptr<fpc_problem_s> h_;
};

inline std::vector<double> assemble_rhs(const TimeStencil& st, double dt, std::span<const double> f,
                                        std::span<const double> u0) {
  std::vector<double> b(f.size());
  if (f.size() != std::size_t(st.n_time) * u0.size())
    throw std::invalid_argument("assemble_rhs: size mismatch");
  detail::check(fpc_assemble_rhs(st.n_time, int(u0.size()), dt, f.data(), u0.data(), b.data()));
  return b;
}

class PreconditionerKind {
 public:
  static PreconditionerKind generalized() { return PreconditionerKind(true, 0.0); }
  static PreconditionerKind strang() { return PreconditionerKind(false, 1.0); }
  static PreconditionerKind with_alpha(double a) { return PreconditionerKind(false, a); }
  double alpha_for(double dt) const {
    const double a = auto_ ? std::min(0.5, 0.5 * dt) : alpha_;
    if (!(a > 0.0) || a > 1.0) throw std::invalid_argument("PreconditionerKind: alpha must lie in (0, 1]");
    return a;
  }
  bool is_auto() const { return auto_; }

 private:
  PreconditionerKind(bool a, double al) : auto_(a), alpha_(al) {}
  bool auto_;
  double alpha_;
};

enum class InnerSweep { half = FPC_SWEEP_HALF, full = FPC_SWEEP_FULL };

// TauOperator (tau.hpp:20-26): the spectrum of tau(A); 2D: sigma[ix*ny + iy], nx = ny = n.
struct TauOperator {
  int n = 0;
  std::vector<double> sigma;
  int nx = 0;
  int ny = 0;
  bool two_dim() const { return nx > 0; }
};

// AlphaCirculantPlan (alpha_circulant.hpp:52-67): the reference's fields, filled from the
// library's plan (the device-resident factors live behind `h`).
struct AlphaCirculantPlan {
  int n_time = 0;
  int n_space = 0;
  double dt = 0.0;
  double alpha = 0.0;
  std::vector<std::complex<double>> lambda;  // eigenvalues of C_alpha
  std::vector<double> scale_fwd;             // alpha^{+k/N_t}
  std::vector<double> scale_bwd;             // alpha^{-k/N_t}
  int solve_count = 0;                       // floor(N_t/2)+1
  TauOperator tau;                           // spectrum of tau(A)
  double min_shift_margin = 0.0;
  std::vector<std::string> warnings;
  std::shared_ptr<fpc_plan_s> h;
  int mirror_index(int n) const { return n_time - n + 2; }
  fpc_plan_t handle() const { return h.get(); }
};

template <class Jacobian>
AlphaCirculantPlan build_plan(const PreconditionerKind& kind, int n_time, double dt,
                              const AllAtOnceOperator<Jacobian>& op) {
  if (n_time < 3) throw std::invalid_argument("build_plan: need at least 3 time levels");
  if (!(dt > 0.0)) throw std::invalid_argument("build_plan: dt must be positive");
  AlphaCirculantPlan plan;
  fpc_plan_t h = nullptr;
  detail::check(fpc_plan_create(op.handle(), kind.alpha_for(dt), &h));
  plan.h.reset(h, [](fpc_plan_t p) { fpc_plan_destroy(p); });
  int nw = 0;
  detail::check(fpc_plan_info(h, &plan.alpha, &plan.min_shift_margin, &plan.solve_count, &nw));
  plan.n_time = n_time;
  plan.n_space = op.n_space();
  plan.dt = dt;
  plan.lambda.resize(std::size_t(n_time));
  detail::check(fpc_plan_lambda(h, reinterpret_cast<double*>(plan.lambda.data())));
  plan.scale_fwd.resize(std::size_t(n_time));
  plan.scale_bwd.resize(std::size_t(n_time));
  detail::check(fpc_plan_scales(h, plan.scale_fwd.data(), plan.scale_bwd.data()));
  plan.tau.n = op.n_space();
  plan.tau.sigma.resize(std::size_t(op.n_space()));
  detail::check(fpc_problem_tau_sigma(op.handle(), plan.tau.sigma.data()));
  if constexpr (std::is_same_v<Jacobian, RieszJacobian2D>) plan.tau.nx = plan.tau.ny = op.jacobian().n;
  if (nw)
    plan.warnings.push_back(
        "alpha below 1e-8: the diagonalization scalings span a wide dynamic range and may amplify "
        "roundoff");
  return plan;
}

inline void apply_inverse(const AlphaCirculantPlan& plan, std::span<const double> v,
                          std::span<double> out, InnerSweep sweep = InnerSweep::half) {
  detail::check(fpc_pc_apply(plan.handle(), v.data(), out.data(), int(sweep), FPC_HOST));
}

inline void apply_forward(const AlphaCirculantPlan& plan, std::span<const double> v,
                          std::span<double> out) {
  detail::check(fpc_pc_forward(plan.handle(), v.data(), out.data(), FPC_HOST));
}

struct SolverConfig {
  double tol = 1e-9;
  int max_iter = 200;
  int restart = 0;
};

struct SolveReport {
  bool converged = false;
  double iterations = 0.0;
  std::vector<double> residual_history;
  double final_relative_residual = 0.0;
  double true_relative_residual = 0.0;
  double seconds = 0.0;
  int restarts = 0;
};

struct KrylovResult {
  std::vector<double> x;
  SolveReport report;
};

namespace detail {
inline void fill_report(SolveReport& out, const fpc_report& rep, const std::vector<double>& hist) {
  out.converged = rep.converged != 0;
  out.iterations = rep.iterations_exact;
  out.residual_history.assign(hist.begin(),
                              hist.begin() + std::min<std::size_t>(rep.history_len, hist.size()));
  out.final_relative_residual = rep.final_relative_residual;
  out.true_relative_residual = rep.true_relative_residual;
  out.seconds = rep.seconds;
  out.restarts = rep.restarts;
}
}  // namespace detail

// device-resident right-preconditioned GMRES (krylov.hpp:83-192), x0 = 0
template <class Jacobian>
KrylovResult gmres_right(const AllAtOnceOperator<Jacobian>& op, const AlphaCirculantPlan& plan,
                         std::span<const double> b, const SolverConfig& cfg = {}) {
  if (b.size() != op.dim()) throw std::invalid_argument("gmres_right: size mismatch");
  KrylovResult r;
  r.x.assign(op.dim(), 0.0);
  fpc_solver_config c{cfg.tol, cfg.max_iter, cfg.restart, FPC_SWEEP_HALF};
  fpc_report rep{};
  std::vector<double> hist(std::size_t(std::max(cfg.max_iter, 1)) + 1);
  detail::check(fpc_gmres(plan.handle(), b.data(), r.x.data(), &c, &rep, hist.data(),
                          int(hist.size()), FPC_HOST));
  detail::fill_report(r.report, rep, hist);
  return r;
}

// device-resident left-preconditioned BiCGSTAB (krylov.hpp:204-280), x0 = 0
template <class Jacobian>
KrylovResult bicgstab_left(const AllAtOnceOperator<Jacobian>& op, const AlphaCirculantPlan& plan,
                           std::span<const double> b, const SolverConfig& cfg = {}) {
  if (b.size() != op.dim()) throw std::invalid_argument("bicgstab_left: size mismatch");
  KrylovResult r;
  r.x.assign(op.dim(), 0.0);
  fpc_solver_config c{cfg.tol, cfg.max_iter, 0, FPC_SWEEP_HALF};
  fpc_report rep{};
  std::vector<double> hist(2 * std::size_t(std::max(cfg.max_iter, 1)) + 2);
  detail::check(fpc_bicgstab(plan.handle(), b.data(), r.x.data(), &c, &rep, hist.data(),
                             int(hist.size()), FPC_HOST));
  detail::fill_report(r.report, rep, hist);
  return r;
}

// gmres_right(n, apply_a, apply_pinv, b, cfg) for ANY host callables with the reference's plugin
// signature void(std::span<const double>, std::span<double>) (krylov.hpp:83-85): the reference's
// iteration with the Krylov basis on the context's device (fpc_gmres_callbacks).  An exception
// thrown by a callable aborts the solve and is rethrown here, as in the reference.
namespace detail {
template <class F>
struct CallableSlot {
  F* f;
  std::exception_ptr err;
  static int call(const double* in, double* out, std::size_t n, void* user) {
    auto* self = static_cast<CallableSlot*>(user);
    try {
      (*self->f)(std::span<const double>(in, n), std::span<double>(out, n));
      return 0;
    } catch (...) {
      self->err = std::current_exception();
      return 1;
    }
  }
};
}  // namespace detail

template <class OpA, class OpP>
KrylovResult gmres_right(std::size_t n, OpA&& apply_a, OpP&& apply_pinv, std::span<const double> b,
                         const SolverConfig& cfg = {}, Context& ctx = Context::default_context()) {
  if (b.size() != n) throw std::invalid_argument("gmres_right: size mismatch");
  using A = std::remove_reference_t<OpA>;
  using P = std::remove_reference_t<OpP>;
  detail::CallableSlot<A> sa{&apply_a, nullptr};
  detail::CallableSlot<P> sp{&apply_pinv, nullptr};
  KrylovResult r;
  r.x.assign(n, 0.0);
  fpc_solver_config c{cfg.tol, cfg.max_iter, cfg.restart, FPC_SWEEP_HALF};
  fpc_report rep{};
  std::vector<double> hist(std::size_t(std::max(cfg.max_iter, 1)) + 1);
  const int rc = fpc_gmres_callbacks(ctx.handle(), n, &detail::CallableSlot<A>::call, &sa,
                                     &detail::CallableSlot<P>::call, &sp, b.data(), r.x.data(), &c, &rep,
                                     hist.data(), int(hist.size()));
  if (sa.err) std::rethrow_exception(sa.err);
  if (sp.err) std::rethrow_exception(sp.err);
  detail::check(rc);
  detail::fill_report(r.report, rep, hist);
  return r;
}

// ---- one process, 1..8 devices (fpc_multi_* / fpc_sharded_*): the frequency-sharded solve of a C++
// caller of solve_all_at_once (driver.hpp:49-92) on several GPUs.  A device may repeat.
class MultiDevice {
 public:
  explicit MultiDevice(const std::vector<int>& devices) {
    fpc_multi_t h = nullptr;
    detail::check(fpc_multi_create(devices.data(), int(devices.size()), &h));
    h_.reset(h, [](fpc_multi_t m) { fpc_multi_destroy(m); });
  }
  fpc_multi_t handle() const { return h_.get(); }

 private:
  std::shared_ptr<fpc_multi_s> h_;
};

template <class Jacobian>
class ShardedOperator {
 public:
  ShardedOperator(MultiDevice& md, TimeStencil stencil, Jacobian jac, double dt,
                  const PreconditionerKind& kind = PreconditionerKind::generalized())
      : md_(md), nt_(stencil.n_time), ns_(jac.dim()) {
    fpc_sharded_t h = nullptr;
    if constexpr (std::is_same_v<Jacobian, RieszJacobian1D>)
      detail::check(fpc_sharded_create_1d(md.handle(), jac.gamma, jac.kappa, jac.h, jac.n, nt_, dt,
                                          kind.alpha_for(dt), &h));
    else
      detail::check(fpc_sharded_create_2d(md.handle(), jac.gamma_x, jac.gamma_y, jac.kappa_x, jac.kappa_y, jac.h,
                                          jac.n, nt_, dt, kind.alpha_for(dt), &h));
    h_.reset(h, [](fpc_sharded_t p) { fpc_sharded_destroy(p); });
  }
  std::size_t dim() const { return std::size_t(nt_) * std::size_t(ns_); }
  void apply(std::span<const double> v, std::span<double> out) const {
    detail::check(fpc_sharded_matvec(h_.get(), v.data(), out.data()));
  }
  void apply_inverse(std::span<const double> v, std::span<double> out) const {
    detail::check(fpc_sharded_pc_apply(h_.get(), v.data(), out.data()));
  }
  KrylovResult gmres_right(std::span<const double> b, const SolverConfig& cfg = {}) const {
    if (b.size() != dim()) throw std::invalid_argument("gmres_right: size mismatch");
    KrylovResult r;
    r.x.assign(dim(), 0.0);
    fpc_solver_config c{cfg.tol, cfg.max_iter, cfg.restart, FPC_SWEEP_HALF};
    fpc_report rep{};
    std::vector<double> hist(std::size_t(std::max(cfg.max_iter, 1)) + 1);
    detail::check(fpc_sharded_gmres(h_.get(), b.data(), r.x.data(), &c, &rep, hist.data(), int(hist.size())));
    detail::fill_report(r.report, rep, hist);
    return r;
  }

 private:
  MultiDevice& md_;
  int nt_, ns_;
  std::shared_ptr<fpc_sharded_s> h_;
};

// Callables for the reference's generic gmres_right(n, apply_a, apply_pinv, b, cfg)
template <class Jacobian>
auto make_apply_a(const AllAtOnceOperator<Jacobian>& op) {
  return [&op](std::span<const double> in, std::span<double> out) { op.apply(in, out); };
}
inline auto make_apply_pinv(const AlphaCirculantPlan& plan, InnerSweep sweep = InnerSweep::half) {
  return [&plan, sweep](std::span<const double> in, std::span<double> out) {
    apply_inverse(plan, in, out, sweep);
  };
}

}  // namespace fracpint::b200
