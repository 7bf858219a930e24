"""Python mirror of the reference's C++ solver API (namespace fracpint), backed by the B200
C-ABI (libfracpint_b200.so).  Names, argument meaning and error behaviour follow the reference:

  TimeStencil            time_stencil.hpp:16-26
  RieszJacobian1D/2D     jacobian.hpp:19-105
  AllAtOnceOperator      all_at_once.hpp:18-61
  assemble_rhs           all_at_once.hpp:66-80
  PreconditionerKind     alpha_circulant.hpp:23-42
  AlphaCirculantPlan     alpha_circulant.hpp:52-67
  build_plan             alpha_circulant.hpp:83-126
  InnerSweep             alpha_circulant.hpp:128
  apply_inverse/forward  alpha_circulant.hpp:206-215
  SolverConfig/SolveReport/KrylovResult/gmres_right   krylov.hpp:25-42, 83-192

Arrays: numpy float64 (host; copied to the GPU and back) or torch CUDA float64 tensors (device
resident, stream-ordered on the context stream).  std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError; sizes the kernels do not cover raise NotImplementedError.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _native as N


# ---------------------------------------------------------------------------------- context
class Context:
    """One device + one CUDA stream (fpc_context_t)."""

    _default: dict = {}

    def __init__(self, device: int = 0, stream=None):
        self.lib = N.load()
        h = C.c_void_p()
        N.check(self.lib.fpc_context_create(int(device), C.byref(h)))
        self.h = h
        self.device = int(device)
        if stream is not None:
            self.set_stream(stream)

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    def set_stream(self, stream) -> None:
        """Use an external cudaStream_t (int handle or torch.cuda.Stream)."""
        handle = getattr(stream, "cuda_stream", stream)
        N.check(self.lib.fpc_context_set_stream(self.h, C.c_void_p(int(handle))))

    @property
    def stream_handle(self) -> int:
        return int(self.lib.fpc_context_stream(self.h) or 0)

    def synchronize(self) -> None:
        N.check(self.lib.fpc_synchronize(self.h))

    def __del__(self):
        try:
            if self.h:
                self.lib.fpc_context_destroy(self.h)
        except Exception:
            pass


def kernel_launches() -> int:
    return int(N.load().fpc_kernel_launches())


class KernelProfile:
    """Live per-kernel device time (CUDA events around every launch of this library)."""

    def __enter__(self):
        self.lib = N.load()
        self.lib.fpc_profile_start()
        return self

    def __exit__(self, *exc):
        n = self.lib.fpc_profile_stop()
        self.table = {}
        for i in range(n):
            name = C.create_string_buffer(64)
            ms, cnt = C.c_double(), C.c_longlong()
            N.check(self.lib.fpc_profile_entry(i, name, 64, C.byref(ms), C.byref(cnt)))
            if cnt.value:
                self.table[name.value.decode()] = (ms.value, cnt.value)
        return False


# ---------------------------------------------------------------------------------- arrays
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _host_in(x, n: int) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.size != n:
        raise ValueError(f"size mismatch: expected {n}, got {a.size}")
    return a


def _dev_in(x, n: int):
    if x.dtype.__str__() != "torch.float64" or not x.is_cuda:
        raise ValueError("device arrays must be CUDA float64 tensors")
    if x.numel() != n:
        raise ValueError(f"size mismatch: expected {n}, got {x.numel()}")
    if not x.is_contiguous():
        raise ValueError("device arrays must be contiguous")
    return x


class _TorchOrder:
    """Device-tensor calls run on the library context's stream; order them after the work torch
    has queued on its current stream (the inputs' producers) and make torch's stream wait for the
    call (the outputs' consumers).  Two events, no host synchronisation; nothing when the context
    already runs on torch's current stream."""

    def __init__(self, ctx):
        self.ctx = ctx

    def __enter__(self):
        import torch
        self.cur = torch.cuda.current_stream()
        self.same = int(self.cur.cuda_stream) == int(self.ctx.stream_handle)
        if not self.same:
            self.lib_stream = torch.cuda.ExternalStream(self.ctx.stream_handle)
            ev = torch.cuda.Event()
            ev.record(self.cur)
            self.lib_stream.wait_event(ev)
        return self

    def __exit__(self, *exc):
        if not self.same:
            import torch
            ev = torch.cuda.Event()
            ev.record(self.lib_stream)
            self.cur.wait_event(ev)
        return False


def _call_vec(fn, handle, n, v, out, *extra, ctx=None):
    """Run fn(handle, in, out, *extra, where) for numpy or torch-CUDA arguments."""
    if _is_torch(v):
        import torch
        vin = _dev_in(v, n)
        if out is None:
            out = torch.empty_like(vin)
        _dev_in(out, n)
        if ctx is None:
            N.check(fn(handle, C.c_void_p(vin.data_ptr()), C.c_void_p(out.data_ptr()), *extra, N.FPC_DEVICE))
        else:
            with _TorchOrder(ctx):
                N.check(fn(handle, C.c_void_p(vin.data_ptr()), C.c_void_p(out.data_ptr()), *extra, N.FPC_DEVICE))
        return out
    vin = _host_in(v, n)
    res = np.empty(n) if out is None else out
    if not (isinstance(res, np.ndarray) and res.dtype == np.float64 and res.flags.c_contiguous and res.size == n):
        raise ValueError("out must be a contiguous float64 numpy array of the operator size")
    N.check(fn(handle, C.c_void_p(vin.ctypes.data), C.c_void_p(res.ctypes.data), *extra, N.FPC_HOST))
    return res


# ---------------------------------------------------------------------------------- operator
class TimeStencil:
    """BDF2 stencil with backward-Euler start (time_stencil.hpp:16-26)."""
    r0, r1, r2 = 1.5, -2.0, 0.5

    def __init__(self, n_time: int):
        if n_time < 3:
            raise ValueError("TimeStencil: need at least 3 time levels")
        self.n_time = int(n_time)


def centred_weights(gamma: float, count: int) -> np.ndarray:
    """weights.hpp:21-35, computed by the library's host setup (fpc_centred_weights)."""
    out = np.empty(max(int(count), 1))
    N.check(N.load().fpc_centred_weights(float(gamma), int(count), out.ctypes.data))
    return out[:count]


def tau_spectrum(column) -> np.ndarray:
    """tau.hpp:40-55: eigenvalues of the tau approximation of the symmetric Toeplitz matrix with
    this first column (library host setup, fpc_tau_spectrum)."""
    col = np.ascontiguousarray(column, dtype=np.float64)
    out = np.empty(max(col.size, 1))
    N.check(N.load().fpc_tau_spectrum(col.ctypes.data, int(col.size), out.ctypes.data))
    return out[:col.size]


def circulant_eigenvalues(column) -> np.ndarray:
    """toeplitz.hpp:23-35: real parts of the circulant embedding's spectrum, k = 0..L/2,
    L = next_pow2(2n) (fpc_circulant_eigenvalues)."""
    col = np.ascontiguousarray(column, dtype=np.float64)
    L = 1
    while L < 2 * col.size:
        L <<= 1
    out = np.empty(L // 2 + 1)
    N.check(N.load().fpc_circulant_eigenvalues(col.ctypes.data, int(col.size), out.ctypes.data))
    return out


def alpha_circulant_eigenvalues(alpha: float, n_time: int) -> np.ndarray:
    """alpha_circulant.hpp:71-81 (fpc_alpha_circulant_eigenvalues): complex128[n_time]."""
    out = np.empty(int(n_time), dtype=np.complex128)
    N.check(N.load().fpc_alpha_circulant_eigenvalues(float(alpha), int(n_time), out.ctypes.data))
    return out


class RieszJacobian1D:
    """A = -(kappa/h^gamma) T(w) (jacobian.hpp:19-51); realised on the device by the operator."""

    def __init__(self, gamma: float, kappa: float, h: float, n_space: int):
        if not (kappa > 0.0):
            raise ValueError("RieszJacobian1D: kappa must be positive")
        if not (h > 0.0):
            raise ValueError("RieszJacobian1D: h must be positive")
        if n_space < 1:
            raise ValueError("RieszJacobian1D: n_space must be at least 1")
        centred_weights(gamma, 1)
        self.gamma, self.kappa, self.h, self.n = float(gamma), float(kappa), float(h), int(n_space)

    def dim(self) -> int:
        return self.n

    def first_column(self) -> np.ndarray:
        return -self.kappa / self.h ** self.gamma * centred_weights(self.gamma, self.n)


class RieszJacobian2D:
    """A = -sx (Tx (x) I) - sy (I (x) Ty), lattice p = ix*n + iy (jacobian.hpp:56-105)."""

    def __init__(self, gamma_x, gamma_y, kappa_x, kappa_y, h, n_per_dim):
        if not (kappa_x > 0.0) or not (kappa_y > 0.0):
            raise ValueError("RieszJacobian2D: diffusion coefficients must be positive")
        if not (h > 0.0):
            raise ValueError("RieszJacobian2D: h must be positive")
        if n_per_dim < 1:
            raise ValueError("RieszJacobian2D: n_per_dim must be at least 1")
        centred_weights(gamma_x, 1)
        centred_weights(gamma_y, 1)
        self.gamma_x, self.gamma_y = float(gamma_x), float(gamma_y)
        self.kappa_x, self.kappa_y = float(kappa_x), float(kappa_y)
        self.h, self.n = float(h), int(n_per_dim)

    def dim(self) -> int:
        return self.n * self.n

    def n_per_dim(self) -> int:
        return self.n


class AllAtOnceOperator:
    """M = C (x) I_s - dt I_t (x) A over time-major vectors (all_at_once.hpp:18-61)."""

    def __init__(self, stencil: TimeStencil, jac, dt: float, context: Context | None = None):
        if not (dt > 0.0):
            raise ValueError("AllAtOnceOperator: dt must be positive")
        self.stencil, self.jac, self._dt = stencil, jac, float(dt)
        self.ctx = context or Context.default()
        self.lib = self.ctx.lib
        h = C.c_void_p()
        if isinstance(jac, RieszJacobian1D):
            rc = self.lib.fpc_problem_create_1d(self.ctx.h, jac.gamma, jac.kappa, jac.h, jac.n,
                                                stencil.n_time, self._dt, C.byref(h))
        elif isinstance(jac, RieszJacobian2D):
            rc = self.lib.fpc_problem_create_2d(self.ctx.h, jac.gamma_x, jac.gamma_y, jac.kappa_x,
                                                jac.kappa_y, jac.h, jac.n, stencil.n_time, self._dt,
                                                C.byref(h))
        else:
            raise TypeError("jacobian must be RieszJacobian1D or RieszJacobian2D")
        N.check(rc)
        self.h = h

    def n_time(self) -> int:
        return self.stencil.n_time

    def n_space(self) -> int:
        return self.jac.dim()

    def dim(self) -> int:
        return self.n_time() * self.n_space()

    def dt(self) -> float:
        return self._dt

    def jacobian(self):
        return self.jac

    def tau_sigma(self) -> np.ndarray:
        s = np.empty(self.n_space())
        N.check(self.lib.fpc_problem_tau_sigma(self.h, C.c_void_p(s.ctypes.data)))
        return s

    def apply(self, v, out=None):
        return _call_vec(self.lib.fpc_matvec, self.h, self.dim(), v, out, ctx=self.ctx)

    def __del__(self):
        try:
            if self.h:
                self.lib.fpc_problem_destroy(self.h)
        except Exception:
            pass


def assemble_rhs(stencil: TimeStencil, dt: float, f_flat, u0) -> np.ndarray:
    """all_at_once.hpp:66-80 (host setup)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    f = np.ascontiguousarray(f_flat, dtype=np.float64)
    ns, nt = u0.size, stencil.n_time
    if f.size != nt * ns:
        raise ValueError("assemble_rhs: size mismatch")
    b = np.empty(nt * ns)
    N.check(N.load().fpc_assemble_rhs(nt, ns, float(dt), C.c_void_p(f.ctypes.data),
                                      C.c_void_p(u0.ctypes.data), C.c_void_p(b.ctypes.data)))
    return b


# ---------------------------------------------------------------------------------- plan
class PreconditionerKind:
    """alpha_circulant.hpp:23-42."""

    def __init__(self, auto_policy: bool, alpha: float):
        self._auto, self._alpha = auto_policy, float(alpha)

    @staticmethod
    def generalized() -> "PreconditionerKind":
        return PreconditionerKind(True, 0.0)

    @staticmethod
    def strang() -> "PreconditionerKind":
        return PreconditionerKind(False, 1.0)

    @staticmethod
    def with_alpha(alpha: float) -> "PreconditionerKind":
        return PreconditionerKind(False, alpha)

    def alpha_for(self, dt: float) -> float:
        a = min(0.5, 0.5 * dt) if self._auto else self._alpha
        if not (a > 0.0) or a > 1.0:
            raise ValueError("PreconditionerKind: alpha must lie in (0, 1]")
        return a

    def is_auto(self) -> bool:
        return self._auto


class Ordering(IntEnum):
    """Factor ordering of the half-sweep preconditioner apply.  `reference`: time FFT, tau solves
    per retained frequency, inverse time FFT (alpha_circulant.hpp:137-199).  `commuted`: DST per
    time level, per-mode time solve, DST per time level (same operator up to
    rounding, 1D only)."""
    reference = N.FPC_ORDER_REFERENCE
    commuted = N.FPC_ORDER_COMMUTED


class InnerSweep(IntEnum):
    half = N.FPC_SWEEP_HALF
    full = N.FPC_SWEEP_FULL


class AlphaCirculantPlan:
    """Device-resident factorised preconditioner P = C_alpha (x) I - dt I (x) tau(A)."""

    def __init__(self, op: AllAtOnceOperator, alpha: float):
        self.op = op
        self.lib = op.lib
        h = C.c_void_p()
        N.check(self.lib.fpc_plan_create(op.h, float(alpha), C.byref(h)))
        self.h = h
        a, m, sc, nw = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        N.check(self.lib.fpc_plan_info(h, C.byref(a), C.byref(m), C.byref(sc), C.byref(nw)))
        self.alpha, self.min_shift_margin, self.solve_count = a.value, m.value, sc.value
        self.n_time, self.n_space, self.dt = op.n_time(), op.n_space(), op.dt()
        self.warnings = (["alpha below 1e-8: the diagonalization scalings span a wide dynamic range "
                          "and may amplify roundoff"] if nw.value else [])
        lam = np.empty(self.n_time, dtype=np.complex128)
        N.check(self.lib.fpc_plan_lambda(h, C.c_void_p(lam.ctypes.data)))
        self.lambda_ = lam
        k = np.arange(self.n_time) / self.n_time
        self.scale_fwd = self.alpha ** k
        self.scale_bwd = self.alpha ** (-k)
        self.ordering = Ordering.reference

    def set_ordering(self, ordering: "Ordering") -> None:
        N.check(self.lib.fpc_plan_set_ordering(self.h, int(ordering)))
        self.ordering = Ordering(ordering)

    def mirror_index(self, n: int) -> int:
        return self.n_time - n + 2

    def __del__(self):
        try:
            if self.h:
                self.lib.fpc_plan_destroy(self.h)
        except Exception:
            pass


def build_plan(kind: PreconditionerKind, n_time: int, dt: float, op,
               ordering: Ordering = Ordering.reference) -> AlphaCirculantPlan:
    """alpha_circulant.hpp:83-126.  `op` is the AllAtOnceOperator whose Jacobian the reference
    passes (the device plan shares its spectra)."""
    if n_time < 3:
        raise ValueError("build_plan: need at least 3 time levels")
    if not (dt > 0.0):
        raise ValueError("build_plan: dt must be positive")
    if not isinstance(op, AllAtOnceOperator):
        raise TypeError("build_plan: pass the AllAtOnceOperator (device operator)")
    if op.n_time() != n_time or abs(op.dt() - dt) > 0.0:
        raise ValueError("build_plan: n_time/dt must match the operator")
    plan = AlphaCirculantPlan(op, kind.alpha_for(dt))
    if ordering != Ordering.reference:
        plan.set_ordering(ordering)
    return plan


def apply_inverse(plan: AlphaCirculantPlan, v, out=None, sweep: InnerSweep = InnerSweep.half):
    """out = P^{-1} v (alpha_circulant.hpp:206-209)."""
    n = plan.n_time * plan.n_space
    return _call_vec(plan.lib.fpc_pc_apply, plan.h, n, v, out, int(sweep), ctx=plan.op.ctx)


def apply_forward(plan: AlphaCirculantPlan, v, out=None):
    """out = P v (alpha_circulant.hpp:212-215)."""
    n = plan.n_time * plan.n_space
    return _call_vec(plan.lib.fpc_pc_forward, plan.h, n, v, out, ctx=plan.op.ctx)


# ---------------------------------------------------------------------------------- Krylov
@dataclass
class SolverConfig:
    tol: float = 1e-9
    max_iter: int = 200
    restart: int = 0  # 0 = unrestarted (the reference); m > 0 = GMRES(m)
    sweep: InnerSweep = InnerSweep.half


@dataclass
class SolveReport:
    converged: bool = False
    iterations: float = 0.0
    residual_history: list = field(default_factory=list)
    final_relative_residual: float = 0.0
    true_relative_residual: float = 0.0
    seconds: float = 0.0
    restarts: int = 0
    reorthogonalizations: int = 0


@dataclass
class KrylovResult:
    x: object
    report: SolveReport


def _krylov(fn, name, op, plan, b, cfg, out):
    if not isinstance(op, AllAtOnceOperator) or not isinstance(plan, AlphaCirculantPlan):
        raise TypeError(f"{name}(op, plan, b, cfg): device operator and plan required")
    if plan.op.h.value != op.h.value:
        raise ValueError(f"{name}: the plan was built for a different operator")
    cfg = cfg or SolverConfig()
    n = op.dim()
    c = N.SolverConfigC(float(cfg.tol), int(cfg.max_iter), int(cfg.restart), int(cfg.sweep))
    rep = N.ReportC()
    cap = 2 * max(int(cfg.max_iter), 1) + 2
    hist = np.zeros(cap)
    if _is_torch(b):
        import torch
        bin_ = _dev_in(b, n)
        x = torch.empty_like(bin_) if out is None else _dev_in(out, n)
        with _TorchOrder(op.ctx):
            N.check(fn(plan.h, C.c_void_p(bin_.data_ptr()), C.c_void_p(x.data_ptr()), C.byref(c),
                       C.byref(rep), C.c_void_p(hist.ctypes.data), cap, N.FPC_DEVICE))
    else:
        bin_ = _host_in(b, n)
        x = np.empty(n) if out is None else out
        if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.size == n
                and x.flags.c_contiguous and x.flags.writeable):
            raise ValueError(f"{name}: out must be a writable contiguous float64 array of size {n}")
        N.check(fn(plan.h, C.c_void_p(bin_.ctypes.data), C.c_void_p(x.ctypes.data), C.byref(c),
                   C.byref(rep), C.c_void_p(hist.ctypes.data), cap, N.FPC_HOST))
    r = SolveReport(bool(rep.converged), float(rep.iterations_exact), list(hist[:min(rep.history_len, cap)]),
                    rep.final_relative_residual, rep.true_relative_residual, rep.seconds, rep.restarts,
                    rep.reorthogonalizations)
    return KrylovResult(x, r)


def gmres_right(op: AllAtOnceOperator, plan: AlphaCirculantPlan, b, cfg: SolverConfig | None = None,
                out=None) -> KrylovResult:
    """Right-preconditioned GMRES on the device (krylov.hpp:83-192), x0 = 0.

    This is the non-generic overload of the reference's gmres_right(n, apply_a, apply_pinv, b, cfg):
    the operator and the plan are the device objects, so the whole iteration stays in HBM."""
    return _krylov(plan.lib.fpc_gmres if isinstance(plan, AlphaCirculantPlan) else None, "gmres_right",
                   op, plan, b, cfg, out)


def gmres_right_callables(n: int, apply_a, apply_pinv, b, cfg: SolverConfig | None = None,
                          ctx: "Context | None" = None) -> KrylovResult:
    """The reference's generic gmres_right(n, apply_a, apply_pinv, b, cfg) (krylov.hpp:83-85) for any
    host callables apply(v: np.ndarray, out: np.ndarray) -> None; the Krylov basis and the
    Gram-Schmidt run on the device (fpc_gmres_callbacks).  A callable's exception is re-raised."""
    ctx = ctx or Context.default()
    cfg = cfg or SolverConfig()
    bh = _host_in(b, n)
    x = np.empty(n)
    errors = []

    def wrap(fn):
        def cb(pin, pout, nn, _user):
            try:
                a = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_double)), shape=(nn,))
                o = np.ctypeslib.as_array(C.cast(pout, C.POINTER(C.c_double)), shape=(nn,))
                fn(a, o)
                return 0
            except BaseException as e:  # noqa: BLE001 -- surfaced below
                errors.append(e)
                return 1
        return N.APPLY_FN(cb)

    ca, cp = wrap(apply_a), wrap(apply_pinv)
    c = N.SolverConfigC(float(cfg.tol), int(cfg.max_iter), int(cfg.restart), int(cfg.sweep))
    rep = N.ReportC()
    cap = max(int(cfg.max_iter), 1) + 1
    hist = np.zeros(cap)
    lib = N.load()
    rc = lib.fpc_gmres_callbacks(ctx.h, n, ca, None, cp, None, C.c_void_p(bh.ctypes.data), C.c_void_p(x.ctypes.data),
                                 C.byref(c), C.byref(rep), C.c_void_p(hist.ctypes.data), cap)
    if errors:
        raise errors[0]
    N.check(rc)
    r = SolveReport(bool(rep.converged), float(rep.iterations_exact), list(hist[:min(rep.history_len, cap)]),
                    rep.final_relative_residual, rep.true_relative_residual, rep.seconds, rep.restarts,
                    rep.reorthogonalizations)
    return KrylovResult(x, r)


def bicgstab_left(op: AllAtOnceOperator, plan: AlphaCirculantPlan, b, cfg: SolverConfig | None = None,
                  out=None) -> KrylovResult:
    """Left-preconditioned BiCGSTAB on the device (krylov.hpp:204-280), x0 = 0: the recurrence on
    P^{-1}-preconditioned vectors, convergence tested on the true residual carried alongside;
    `report.iterations` counts a half-step convergence as k + 0.5 like the reference.
    `cfg.restart` is ignored."""
    return _krylov(plan.lib.fpc_bicgstab if isinstance(plan, AlphaCirculantPlan) else None, "bicgstab_left",
                   op, plan, b, cfg, out)
