"""Single-process multi-device solve through the C-ABI (fpc_multi_* / fpc_sharded_*).

SURVEY §8(b) asks for a context over 1..8 devices behind the drop-in boundary; §8(e) for the
frequency-sharded solve.  `MultiDevice([0, 1, ..., 7])` is that context (one stream per rank, peer
access enabled); `ShardedProblem` is the all-at-once operator + BC plan sharded over it, with
matvec / apply_inverse / gmres_right on host vectors of the whole problem (time-major).  A device
index may repeat ([0, 0, 0, 0]): the G-rank schedule then runs on one GPU (no kernel waits on
another rank), which is how the GPU tests cover G = 2 and 4 on a one-GPU box.  The multi-process
(torchrun, one rank per GPU) route is distributed.py's ShardedSolver.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .solver import (KrylovResult, PreconditionerKind, RieszJacobian1D, RieszJacobian2D, SolveReport,
                     SolverConfig, TimeStencil, _host_in)


class MultiDevice:
    def __init__(self, devices):
        self.lib = N.load()
        self.devices = [int(d) for d in devices]
        arr = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        N.check(self.lib.fpc_multi_create(arr, len(self.devices), C.byref(h)))
        self.h = h

    @property
    def n_ranks(self) -> int:
        return len(self.devices)

    def __del__(self):
        try:
            if self.h:
                self.lib.fpc_multi_destroy(self.h)
        except Exception:  # noqa: BLE001
            pass


class ShardedProblem:
    """AllAtOnceOperator(TimeStencil(nt), jac, dt) + build_plan(kind, nt, dt, op), time-sharded over
    the ranks of `multi` (fpc_sharded_create_1d/2d)."""

    def __init__(self, multi: MultiDevice, stencil: TimeStencil, jac, dt: float,
                 kind: PreconditionerKind | None = None):
        self.multi, self.lib = multi, multi.lib
        self.nt = stencil.n_time
        self.ns = jac.dim()
        alpha = (kind or PreconditionerKind.generalized()).alpha_for(dt)
        h = C.c_void_p()
        if isinstance(jac, RieszJacobian1D):
            N.check(self.lib.fpc_sharded_create_1d(multi.h, jac.gamma, jac.kappa, jac.h, jac.n, self.nt, float(dt),
                                                   alpha, C.byref(h)))
        elif isinstance(jac, RieszJacobian2D):
            N.check(self.lib.fpc_sharded_create_2d(multi.h, jac.gamma_x, jac.gamma_y, jac.kappa_x, jac.kappa_y, jac.h,
                                                   jac.n, self.nt, float(dt), alpha, C.byref(h)))
        else:
            raise TypeError("ShardedProblem: RieszJacobian1D or RieszJacobian2D expected")
        self.h = h

    def dim(self) -> int:
        return self.nt * self.ns

    def _vec(self, fn, v):
        vin = _host_in(v, self.dim())
        out = np.empty(self.dim())
        N.check(fn(self.h, C.c_void_p(vin.ctypes.data), C.c_void_p(out.ctypes.data)))
        return out

    def matvec(self, v):
        """AllAtOnceOperator::apply (all_at_once.hpp:33-55) on the sharded layout."""
        return self._vec(self.lib.fpc_sharded_matvec, v)

    def apply_inverse(self, v):
        """apply_inverse (alpha_circulant.hpp:206-209), reference ordering, peer-store exchanges."""
        return self._vec(self.lib.fpc_sharded_pc_apply, v)

    def gmres_right(self, b, cfg: SolverConfig | None = None) -> KrylovResult:
        """gmres_right (krylov.hpp:83-192) on the sharded operator, x0 = 0; GMRES(m) by cfg.restart."""
        cfg = cfg or SolverConfig()
        bh = _host_in(b, self.dim())
        x = np.empty(self.dim())
        c = N.SolverConfigC(float(cfg.tol), int(cfg.max_iter), int(cfg.restart), 0)
        rep = N.ReportC()
        cap = max(int(cfg.max_iter), 1) + 1
        hist = np.zeros(cap)
        N.check(self.lib.fpc_sharded_gmres(self.h, C.c_void_p(bh.ctypes.data), C.c_void_p(x.ctypes.data), C.byref(c),
                                           C.byref(rep), C.c_void_p(hist.ctypes.data), cap))
        r = SolveReport(bool(rep.converged), float(rep.iterations_exact), list(hist[:min(rep.history_len, cap)]),
                        rep.final_relative_residual, rep.true_relative_residual, rep.seconds, rep.restarts,
                        rep.reorthogonalizations)
        return KrylovResult(x, r)

    def __del__(self):
        try:
            if self.h:
                self.lib.fpc_sharded_destroy(self.h)
        except Exception:  # noqa: BLE001
            pass
