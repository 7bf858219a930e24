"""ctypes front end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Two back ends with the same Python surface:

* ``Oracle``    -> oracle/_build/liboracle.so, the C restatement (oracle/fracpint_oracle.c);
* ``Reference`` -> oracle/_ref/libfracpint_ref.so, the unmodified reference headers
  (/root/reference/proj/include/fracpint) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import
this module, and only as the checker or the CPU baseline -- never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfracpint_ref.so")

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def build(quiet: bool = True) -> None:
    """Build oracle/_build (always) and oracle/_ref (when /root/reference is present)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(ValueError):
    pass


@dataclass
class SolveReport:
    converged: bool
    iterations: int
    final_relative_residual: float
    true_relative_residual: float
    residual_history: list = field(default_factory=list)
    seconds: float = 0.0
    restarts: int = 0


class _ORep(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("restarts", C.c_int),
                ("final_relative_residual", C.c_double), ("true_relative_residual", C.c_double),
                ("history_len", C.c_int)]


_lib_cache: dict = {}

# int (*)(const double* in, double* out, size_t n, void* user)
REF_APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def _load(path: str, kind: str):
    if path in _lib_cache:
        return _lib_cache[path]
    if not os.path.exists(path):
        raise FileNotFoundError(f"{kind} library missing: {path} (run `make -C oracle`)")
    lib = C.CDLL(path)
    if kind == "oracle":
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_problem_1d.restype = C.c_void_p
        lib.orc_problem_1d.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double]
        lib.orc_problem_2d.restype = C.c_void_p
        lib.orc_problem_2d.argtypes = [C.c_double] * 5 + [C.c_int, C.c_int, C.c_double]
        lib.orc_problem_free.argtypes = [C.c_void_p]
        lib.orc_problem_dim.restype = C.c_size_t
        lib.orc_problem_dim.argtypes = [C.c_void_p]
        for fn in ("orc_matvec", "orc_pc_forward"):
            getattr(lib, fn).argtypes = [C.c_void_p, _dp, _dp]
        lib.orc_jacobian_apply.argtypes = [C.c_void_p, _dp, _dp]
        lib.orc_pc_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        lib.orc_build_plan.argtypes = [C.c_void_p, C.c_double]
        lib.orc_plan_alpha.restype = C.c_double
        lib.orc_plan_alpha.argtypes = [C.c_void_p]
        lib.orc_plan_min_shift_margin.restype = C.c_double
        lib.orc_plan_min_shift_margin.argtypes = [C.c_void_p]
        lib.orc_plan_n_warnings.argtypes = [C.c_void_p]
        lib.orc_plan_lambda.argtypes = [C.c_void_p, _dp]
        lib.orc_tau_sigma.argtypes = [C.c_void_p, _dp]
        lib.orc_jacobian_column.argtypes = [C.c_void_p, C.c_int, _dp]
        lib.orc_gmres.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(_ORep), _dp, C.c_int]
        lib.orc_bicgstab.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.c_int, _dp,
                                     C.POINTER(_ORep), _dp, C.c_int]
        lib.orc_fft_inplace.argtypes = [_dp, C.c_size_t, C.c_int]
        lib.orc_dst1_real.argtypes = [_dp, _dp, C.c_size_t]
        lib.orc_dst1_complex.argtypes = [_dp, _dp, C.c_size_t]
        lib.orc_centred_weights.argtypes = [C.c_double, C.c_int, _dp]
        lib.orc_toeplitz_matvec.argtypes = [_dp, C.c_size_t, _dp, _dp]
        lib.orc_tau_spectrum.argtypes = [_dp, C.c_size_t, _dp]
        lib.orc_tau_solve_shifted.argtypes = [_dp, C.c_int, C.c_int, C.c_size_t, C.c_double,
                                              C.c_double, C.c_double, _dp, _dp]
        lib.orc_alpha_circulant_eigenvalues.argtypes = [C.c_double, C.c_int, _dp]
        lib.orc_assemble_rhs.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp, _dp]
    else:
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_set_threads.argtypes = [C.c_int]
        lib.ref_problem_1d.restype = C.c_void_p
        lib.ref_problem_1d.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double]
        lib.ref_problem_2d.restype = C.c_void_p
        lib.ref_problem_2d.argtypes = [C.c_double] * 5 + [C.c_int, C.c_int, C.c_double]
        lib.ref_problem_free.argtypes = [C.c_void_p]
        lib.ref_matvec.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_pc_forward.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_pc_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        lib.ref_build_plan.argtypes = [C.c_void_p, C.c_double, _dp, _dp]
        lib.ref_tau_sigma.argtypes = [C.c_void_p, _dp]
        lib.ref_gmres.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), _dp, _dp, _dp, _dp, C.c_int, C.POINTER(C.c_int)]
        lib.ref_gmres_callbacks.argtypes = [C.c_size_t, REF_APPLY_FN, C.c_void_p, REF_APPLY_FN, C.c_void_p, _dp, _dp,
                                            C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, _dp,
                                            C.c_int, C.POINTER(C.c_int)]
        lib.ref_gmres_restart.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_int),
                                          C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, _dp]
        lib.ref_bicgstab.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int),
                                     _dp, _dp, _dp, _dp, _dp, C.c_int, C.POINTER(C.c_int)]
        lib.ref_run_problem.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_int, _dp, C.POINTER(C.c_int), _dp, _dp, _dp, _dp]
        lib.ref_fft_inplace.argtypes = [_dp, C.c_size_t, C.c_int]
        lib.ref_dst1_real.argtypes = [_dp, _dp, C.c_size_t]
        lib.ref_dst1_complex.argtypes = [_dp, _dp, C.c_size_t]
        lib.ref_centred_weights.argtypes = [C.c_double, C.c_int, _dp]
        lib.ref_toeplitz_matvec.argtypes = [_dp, C.c_size_t, _dp, _dp]
        lib.ref_tau_spectrum.argtypes = [_dp, C.c_size_t, _dp]
        lib.ref_assemble_rhs.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp, _dp]
    _lib_cache[path] = lib
    return lib


def _raise(code: int, msg: bytes):
    text = msg.decode() if msg else ""
    if code == 1:
        raise OracleInvalidArgument(text)
    raise OracleError(text)


class _Backend:
    prefix = ""

    def __init__(self):
        self.lib = _load(self.path, self.kind)

    def _chk(self, rc):
        if rc != 0:
            _raise(rc, getattr(self.lib, self.prefix + "last_error")())

    # ---- transforms / setup -------------------------------------------------------------
    def fft(self, x: np.ndarray, sign: int) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.complex128).copy()
        getattr(self.lib, self.prefix + "fft_inplace")(y.view(np.float64).ctypes.data_as(_dp), y.size, sign)
        return y

    def dst1(self, x: np.ndarray) -> np.ndarray:
        if np.iscomplexobj(x):
            xi = np.ascontiguousarray(x, dtype=np.complex128)
            y = np.empty_like(xi)
            self._chk(getattr(self.lib, self.prefix + "dst1_complex")(
                _ptr(xi.view(np.float64)), _ptr(y.view(np.float64)), xi.size))
            return y
        xi = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(xi)
        self._chk(getattr(self.lib, self.prefix + "dst1_real")(_ptr(xi), _ptr(y), xi.size))
        return y

    def centred_weights(self, gamma: float, count: int) -> np.ndarray:
        w = np.empty(max(count, 1))
        self._chk(getattr(self.lib, self.prefix + "centred_weights")(gamma, count, _ptr(w)))
        return w

    def toeplitz_matvec(self, col, v):
        col = np.ascontiguousarray(col, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self._chk(getattr(self.lib, self.prefix + "toeplitz_matvec")(_ptr(col), col.size, _ptr(v), _ptr(out)))
        return out

    def tau_spectrum(self, col):
        col = np.ascontiguousarray(col, dtype=np.float64)
        s = np.empty_like(col)
        self._chk(getattr(self.lib, self.prefix + "tau_spectrum")(_ptr(col), col.size, _ptr(s)))
        return s

    def assemble_rhs(self, nt, ns, dt, f, u0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        b = np.empty(nt * ns)
        self._chk(getattr(self.lib, self.prefix + "assemble_rhs")(nt, ns, dt, _ptr(f), _ptr(u0), _ptr(b)))
        return b


class _ProblemBase:
    def __init__(self, backend, handle, nt, ns):
        self.be, self.h, self.nt, self.ns = backend, handle, nt, ns
        self.n = nt * ns

    def __del__(self):
        try:
            getattr(self.be.lib, self.be.prefix + "problem_free")(self.h)
        except Exception:
            pass

    def matvec(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self.be._chk(getattr(self.be.lib, self.be.prefix + "matvec")(self.h, _ptr(v), _ptr(out)))
        return out

    def pc_apply(self, v, full_sweep=False):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self.be._chk(getattr(self.be.lib, self.be.prefix + "pc_apply")(self.h, _ptr(v), _ptr(out), int(full_sweep)))
        return out

    def pc_forward(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self.be._chk(getattr(self.be.lib, self.be.prefix + "pc_forward")(self.h, _ptr(v), _ptr(out)))
        return out


class Oracle(_Backend):
    """The C restatement (oracle/fracpint_oracle.c)."""
    path, kind, prefix = ORACLE_SO, "oracle", "orc_"

    def problem_1d(self, gamma, kappa, h, n, nt, dt):
        hd = self.lib.orc_problem_1d(gamma, kappa, h, n, nt, dt)
        if not hd:
            _raise(1, self.lib.orc_last_error())
        p = OracleProblem(self, hd, nt, n)
        p.npd = n
        return p

    def problem_2d(self, gx, gy, kx, ky, h, n, nt, dt):
        hd = self.lib.orc_problem_2d(gx, gy, kx, ky, h, n, nt, dt)
        if not hd:
            _raise(1, self.lib.orc_last_error())
        p = OracleProblem(self, hd, nt, n * n)
        p.npd = n
        return p

    def tau_solve_shifted(self, sigma, nx, ny, shift, dt, rhs):
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        out = np.empty_like(rhs)
        self._chk(self.lib.orc_tau_solve_shifted(_ptr(sigma), nx, ny, rhs.size, shift.real, shift.imag, dt,
                                                 _ptr(rhs.view(np.float64)), _ptr(out.view(np.float64))))
        return out

    def alpha_circulant_eigenvalues(self, alpha, nt):
        lam = np.empty(nt, dtype=np.complex128)
        self.lib.orc_alpha_circulant_eigenvalues(alpha, nt, _ptr(lam.view(np.float64)))
        return lam


class OracleProblem(_ProblemBase):
    def jacobian_apply(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self.be._chk(self.be.lib.orc_jacobian_apply(self.h, _ptr(v), _ptr(out)))
        return out

    def build_plan(self, alpha: float = 0.0):
        self.be._chk(self.be.lib.orc_build_plan(self.h, alpha))
        return self

    @property
    def alpha(self):
        return self.be.lib.orc_plan_alpha(self.h)

    @property
    def min_shift_margin(self):
        return self.be.lib.orc_plan_min_shift_margin(self.h)

    @property
    def n_warnings(self):
        return self.be.lib.orc_plan_n_warnings(self.h)

    def lam(self):
        out = np.empty(self.nt, dtype=np.complex128)
        self.be._chk(self.be.lib.orc_plan_lambda(self.h, _ptr(out.view(np.float64))))
        return out

    def sigma(self):
        s = np.empty(self.ns)
        self.be._chk(self.be.lib.orc_tau_sigma(self.h, _ptr(s)))
        return s

    def column(self, axis=0):
        c = np.empty(self.npd)
        self.be._chk(self.be.lib.orc_jacobian_column(self.h, axis, _ptr(c)))
        return c

    def gmres(self, b, tol=1e-9, max_iter=200, restart=0, full_sweep=False):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        rep = _ORep()
        cap = max(max_iter, 1) + 1
        hist = np.zeros(cap)
        self.be._chk(self.be.lib.orc_gmres(self.h, _ptr(b), _ptr(x), tol, max_iter, restart,
                                           int(full_sweep), C.byref(rep), _ptr(hist), cap))
        return x, SolveReport(bool(rep.converged), rep.iterations, rep.final_relative_residual,
                              rep.true_relative_residual, list(hist[:min(rep.history_len, cap)]),
                              0.0, rep.restarts)

    def bicgstab(self, b, tol=1e-9, max_iter=200, full_sweep=False):
        """bicgstab_left (krylov.hpp:204-280); report.iterations is the reference's float count."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        rep = _ORep()
        it = np.zeros(1)
        cap = 2 * max(max_iter, 1) + 2
        hist = np.zeros(cap)
        self.be._chk(self.be.lib.orc_bicgstab(self.h, _ptr(b), _ptr(x), tol, max_iter, int(full_sweep), _ptr(it),
                                              C.byref(rep), _ptr(hist), cap))
        return x, SolveReport(bool(rep.converged), float(it[0]), rep.final_relative_residual,
                              rep.true_relative_residual, list(hist[:min(rep.history_len, cap)]))


class Reference(_Backend):
    """The unmodified reference, compiled from /root/reference headers (oracle/_ref)."""
    path, kind, prefix = REF_SO, "ref", "ref_"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def set_threads(self, n: int):
        self.lib.ref_set_threads(int(n))

    def run_problem(self, dim, gx, gy, nt, h_inv, method="gmres", strang=False, tol=1e-9, max_iter=200):
        """run_problem(example1(gx) | example2(gx, gy), RunConfig) (driver.hpp:84-112).
        Returns dict(iterations, converged, err_inf, rhs, exact, final)."""
        n = h_inv - 1
        ns = n if dim == 1 else n * n
        it, err = np.zeros(1), np.zeros(1)
        conv = C.c_int()
        rhs, ex, fin = np.zeros(nt * ns), np.zeros(ns), np.zeros(ns)
        self._chk(self.lib.ref_run_problem(dim, gx, gy, nt, h_inv, 1 if method == "bicgstab" else 0, int(strang),
                                           tol, max_iter, _ptr(it), C.byref(conv), _ptr(err), _ptr(rhs), _ptr(ex),
                                           _ptr(fin)))
        return {"iterations": float(it[0]), "converged": bool(conv.value), "err_inf": float(err[0]),
                "rhs": rhs, "exact": ex, "final": fin}

    def gmres_callables(self, n, apply_a, apply_pinv, b, tol=1e-9, max_iter=200):
        """The reference's own gmres_right (krylov.hpp:83-192) driving Python callables
        apply(v, out) (e.g. the B200 library's operators).  Returns (x, dict(...))."""
        errors = []

        def wrap(fn):
            def cb(pin, pout, nn, _u):
                try:
                    a = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_double)), shape=(nn,))
                    o = np.ctypeslib.as_array(C.cast(pout, C.POINTER(C.c_double)), shape=(nn,))
                    fn(a, o)
                    return 0
                except BaseException as e:  # noqa: BLE001
                    errors.append(e)
                    return 1
            return REF_APPLY_FN(cb)

        ca, cp = wrap(apply_a), wrap(apply_pinv)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        conv, it, hl = C.c_int(), C.c_int(), C.c_int()
        tr = np.zeros(1)
        hist = np.zeros(max_iter + 1)
        rc = self.lib.ref_gmres_callbacks(n, ca, None, cp, None, _ptr(b), _ptr(x), tol, max_iter, C.byref(conv),
                                          C.byref(it), _ptr(tr), _ptr(hist), max_iter + 1, C.byref(hl))
        if errors:
            raise errors[0]
        self._chk(rc)
        return x, {"converged": bool(conv.value), "iterations": it.value, "true_relative_residual": float(tr[0]),
                   "residual_history": list(hist[:min(hl.value, max_iter + 1)])}

    def problem_1d(self, gamma, kappa, h, n, nt, dt):
        hd = self.lib.ref_problem_1d(gamma, kappa, h, n, nt, dt)
        if not hd:
            _raise(1, self.lib.ref_last_error())
        return RefProblem(self, hd, nt, n)

    def problem_2d(self, gx, gy, kx, ky, h, n, nt, dt):
        hd = self.lib.ref_problem_2d(gx, gy, kx, ky, h, n, nt, dt)
        if not hd:
            _raise(1, self.lib.ref_last_error())
        return RefProblem(self, hd, nt, n * n)


class RefProblem(_ProblemBase):
    def build_plan(self, alpha: float = 0.0):
        mm = np.zeros(1)
        al = np.zeros(1)
        self.be._chk(self.be.lib.ref_build_plan(self.h, alpha, _ptr(mm), _ptr(al)))
        self.min_shift_margin = float(mm[0])
        self.alpha = float(al[0])
        return self

    def sigma(self):
        s = np.empty(self.ns)
        self.be._chk(self.be.lib.ref_tau_sigma(self.h, _ptr(s)))
        return s

    def gmres(self, b, tol=1e-9, max_iter=200):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        conv, it, hl = C.c_int(), C.c_int(), C.c_int()
        fr, tr, sec = np.zeros(1), np.zeros(1), np.zeros(1)
        cap = max_iter + 1
        hist = np.zeros(cap)
        self.be._chk(self.be.lib.ref_gmres(self.h, _ptr(b), _ptr(x), tol, max_iter, C.byref(conv), C.byref(it),
                                           _ptr(fr), _ptr(tr), _ptr(sec), _ptr(hist), cap, C.byref(hl)))
        return x, SolveReport(bool(conv.value), it.value, float(fr[0]), float(tr[0]),
                              list(hist[:min(hl.value, cap)]), float(sec[0]))

    def gmres_restarted(self, b, tol=1e-9, max_iter=200, restart=0):
        """GMRES(m) emulated on the reference's own gmres_right (ref_shim.cpp).
        Returns (x, dict(converged, iterations, restarts, true_relative_residual, seconds))."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        conv, it, rs = C.c_int(), C.c_int(), C.c_int()
        tr, sec = np.zeros(1), np.zeros(1)
        self.be._chk(self.be.lib.ref_gmres_restart(self.h, _ptr(b), _ptr(x), tol, max_iter, restart, C.byref(conv),
                                                   C.byref(it), C.byref(rs), _ptr(tr), _ptr(sec)))
        return x, {"converged": bool(conv.value), "iterations": it.value, "restarts": rs.value,
                   "true_relative_residual": float(tr[0]), "seconds": float(sec[0])}

    def bicgstab(self, b, tol=1e-9, max_iter=200):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        conv, hl = C.c_int(), C.c_int()
        it, fr, tr, sec = np.zeros(1), np.zeros(1), np.zeros(1), np.zeros(1)
        cap = 2 * max_iter + 2
        hist = np.zeros(cap)
        self.be._chk(self.be.lib.ref_bicgstab(self.h, _ptr(b), _ptr(x), tol, max_iter, C.byref(conv), _ptr(it),
                                              _ptr(fr), _ptr(tr), _ptr(sec), _ptr(hist), cap, C.byref(hl)))
        return x, SolveReport(bool(conv.value), float(it[0]), float(fr[0]), float(tr[0]),
                              list(hist[:min(hl.value, cap)]), float(sec[0]))
