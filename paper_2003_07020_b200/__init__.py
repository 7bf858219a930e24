"""paper_2003_07020_b200 -- B200-native preconditioned Krylov solve for the all-at-once BDF2
Riesz fractional diffusion system (arXiv 2003.07020), drop-in for the reference's `fracpint`
solver API.  The compute lives in libfracpint_b200.so (hand-written sm_100a CUDA behind the C-ABI
include/fracpint_b200.h); this package is the Python mirror of the reference interface.
"""
from .solver import (AllAtOnceOperator, AlphaCirculantPlan, Context, InnerSweep, KrylovResult, Ordering,
                     PreconditionerKind, RieszJacobian1D, RieszJacobian2D, SolveReport, SolverConfig,
                     TimeStencil, apply_forward, apply_inverse, assemble_rhs, bicgstab_left, build_plan,
                     centred_weights, tau_spectrum, circulant_eigenvalues, alpha_circulant_eigenvalues,
                     gmres_right, gmres_right_callables, kernel_launches, KernelProfile)
from .multi import MultiDevice, ShardedProblem

__all__ = [
    "AllAtOnceOperator", "AlphaCirculantPlan", "Context", "InnerSweep", "KrylovResult", "Ordering",
    "PreconditionerKind", "RieszJacobian1D", "RieszJacobian2D", "SolveReport", "SolverConfig",
    "TimeStencil", "apply_forward", "apply_inverse", "assemble_rhs", "bicgstab_left", "build_plan", "centred_weights", "tau_spectrum", "circulant_eigenvalues", "alpha_circulant_eigenvalues",
    "gmres_right", "gmres_right_callables", "kernel_launches", "KernelProfile", "MultiDevice", "ShardedProblem",
]
