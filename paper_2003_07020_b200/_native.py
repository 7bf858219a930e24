"""ctypes binding of libfracpint_b200.so (the C-ABI in include/fracpint_b200.h).

The shared library is the product: the CUDA kernels and the device-resident GMRES driver.
Loading fails loudly when it is missing -- there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FPC_LIB overrides the library path (development builds, e.g. the phase-timing build)
LIB_PATH = os.environ.get("FPC_LIB") or os.path.join(HERE, "libfracpint_b200.so")

FPC_OK, FPC_INVALID_ARGUMENT, FPC_RUNTIME_ERROR, FPC_CUDA_ERROR, FPC_UNSUPPORTED = 0, 1, 2, 3, 4
FPC_HOST, FPC_DEVICE = 0, 1
FPC_SWEEP_HALF, FPC_SWEEP_FULL = 0, 1
FPC_ORDER_REFERENCE, FPC_ORDER_COMMUTED = 0, 1

# every symbol include/fracpint_b200.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fpc_abi_version", "fpc_last_error", "fpc_context_create", "fpc_context_destroy",
    "fpc_context_set_stream", "fpc_context_stream", "fpc_synchronize", "fpc_device_alloc",
    "fpc_device_free", "fpc_problem_create_1d", "fpc_problem_create_2d", "fpc_problem_destroy",
    "fpc_problem_dims", "fpc_problem_first_column", "fpc_problem_tau_sigma", "fpc_matvec",
    "fpc_assemble_rhs", "fpc_plan_create", "fpc_plan_destroy", "fpc_plan_info", "fpc_plan_lambda",
    "fpc_plan_set_ordering", "fpc_pc_apply", "fpc_pc_forward", "fpc_gmres", "fpc_bicgstab", "fpc_kernel_launches", "fpc_profile_start",
    "fpc_profile_stop", "fpc_profile_entry", "fpc_shard_matvec", "fpc_shard_time_fwd", "fpc_shard_tau",
    "fpc_shard_time_inv", "fpc_shard_dots", "fpc_shard_update", "fpc_shard_lincomb",
    "fpc_shard_dst_levels", "fpc_shard_time_solve", "fpc_ipc_get_handle", "fpc_ipc_open", "fpc_ipc_close",
    "fpc_shard_scatter_p2p", "fpc_centred_weights", "fpc_tau_spectrum", "fpc_circulant_eigenvalues",
    "fpc_alpha_circulant_eigenvalues", "fpc_plan_scales", "fpc_gmres_callbacks",
    "fpc_multi_create", "fpc_multi_destroy", "fpc_sharded_create_1d", "fpc_sharded_create_2d",
    "fpc_sharded_destroy", "fpc_sharded_info", "fpc_sharded_matvec", "fpc_sharded_pc_apply", "fpc_sharded_gmres",
    "fpc_shard_dots_dev", "fpc_shard_update_dev",
]


class SolverConfigC(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int), ("sweep", C.c_int)]


class ReportC(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("restarts", C.c_int),
                ("reorthogonalizations", C.c_int), ("final_relative_residual", C.c_double),
                ("true_relative_residual", C.c_double), ("seconds", C.c_double),
                ("history_len", C.c_int), ("iterations_exact", C.c_double)]


_lib = None

# int (*)(const double* in, double* out, size_t n, void* user)  -- fpc_apply_fn
APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def load():
    """Load the native library (raises if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2003_07020_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, dp, ip = C.c_void_p, C.c_void_p, C.POINTER(C.c_int)
    d = C.c_double
    lib.fpc_last_error.restype = C.c_char_p
    lib.fpc_context_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.fpc_context_destroy.argtypes = [vp]
    lib.fpc_context_set_stream.argtypes = [vp, vp]
    lib.fpc_context_stream.restype = vp
    lib.fpc_context_stream.argtypes = [vp]
    lib.fpc_synchronize.argtypes = [vp]
    lib.fpc_device_alloc.argtypes = [vp, C.c_size_t, C.POINTER(C.c_void_p)]
    lib.fpc_device_free.argtypes = [vp, vp]
    lib.fpc_ipc_get_handle.argtypes = [vp, vp]
    lib.fpc_ipc_open.argtypes = [vp, vp, C.POINTER(C.c_void_p)]
    lib.fpc_ipc_close.argtypes = [vp, vp]
    lib.fpc_shard_scatter_p2p.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                          ip, ip, C.c_int, C.c_int, C.c_int]
    lib.fpc_problem_create_1d.argtypes = [vp, d, d, d, C.c_int, C.c_int, d, C.POINTER(C.c_void_p)]
    lib.fpc_problem_create_2d.argtypes = [vp, d, d, d, d, d, C.c_int, C.c_int, d, C.POINTER(C.c_void_p)]
    lib.fpc_problem_destroy.argtypes = [vp]
    lib.fpc_problem_dims.argtypes = [vp, ip, ip, ip]
    lib.fpc_problem_first_column.argtypes = [vp, C.c_int, dp]
    lib.fpc_problem_tau_sigma.argtypes = [vp, dp]
    lib.fpc_matvec.argtypes = [vp, dp, dp, C.c_int]
    lib.fpc_assemble_rhs.argtypes = [C.c_int, C.c_int, d, dp, dp, dp]
    lib.fpc_plan_create.argtypes = [vp, d, C.POINTER(C.c_void_p)]
    lib.fpc_plan_destroy.argtypes = [vp]
    lib.fpc_plan_info.argtypes = [vp, C.POINTER(d), C.POINTER(d), ip, ip]
    lib.fpc_plan_lambda.argtypes = [vp, dp]
    lib.fpc_plan_set_ordering.argtypes = [vp, C.c_int]
    lib.fpc_pc_apply.argtypes = [vp, dp, dp, C.c_int, C.c_int]
    lib.fpc_pc_forward.argtypes = [vp, dp, dp, C.c_int]
    lib.fpc_gmres.argtypes = [vp, dp, dp, C.POINTER(SolverConfigC), C.POINTER(ReportC), dp, C.c_int, C.c_int]
    lib.fpc_bicgstab.argtypes = [vp, dp, dp, C.POINTER(SolverConfigC), C.POINTER(ReportC), dp, C.c_int, C.c_int]
    lib.fpc_kernel_launches.restype = C.c_ulonglong
    lib.fpc_profile_entry.argtypes = [C.c_int, C.c_char_p, C.c_int, C.POINTER(d), C.POINTER(C.c_longlong)]
    lib.fpc_shard_matvec.argtypes = [vp, vp, vp, C.c_int, C.c_int]
    lib.fpc_shard_time_fwd.argtypes = [vp, vp, vp, C.c_int, d]
    lib.fpc_shard_tau.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int]
    lib.fpc_shard_time_inv.argtypes = [vp, vp, vp, C.c_int]
    lib.fpc_shard_dots.argtypes = [vp, vp, vp, C.c_int, vp, C.c_size_t, C.c_int, vp]
    lib.fpc_shard_update.argtypes = [vp, vp, vp, C.c_int, vp, C.c_size_t, vp]
    lib.fpc_shard_lincomb.argtypes = [vp, vp, vp, C.c_int, vp, C.c_size_t]
    lib.fpc_shard_dst_levels.argtypes = [vp, vp, vp, C.c_int, d]
    lib.fpc_shard_time_solve.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int]
    lib.fpc_centred_weights.argtypes = [d, C.c_int, dp]
    lib.fpc_tau_spectrum.argtypes = [dp, C.c_int, dp]
    lib.fpc_circulant_eigenvalues.argtypes = [dp, C.c_int, dp]
    lib.fpc_alpha_circulant_eigenvalues.argtypes = [d, C.c_int, dp]
    lib.fpc_plan_scales.argtypes = [vp, dp, dp]
    lib.fpc_gmres_callbacks.argtypes = [vp, C.c_size_t, APPLY_FN, vp, APPLY_FN, vp, dp, dp,
                                        C.POINTER(SolverConfigC), C.POINTER(ReportC), dp, C.c_int]
    lib.fpc_shard_dots_dev.argtypes = [vp, vp, vp, C.c_int, vp, C.c_size_t, C.c_int, vp]
    lib.fpc_shard_update_dev.argtypes = [vp, vp, vp, C.c_int, vp, C.c_size_t, vp]
    lib.fpc_multi_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]
    lib.fpc_multi_destroy.argtypes = [vp]
    lib.fpc_sharded_create_1d.argtypes = [vp, d, d, d, C.c_int, C.c_int, d, d, C.POINTER(C.c_void_p)]
    lib.fpc_sharded_create_2d.argtypes = [vp, d, d, d, d, d, C.c_int, C.c_int, d, d, C.POINTER(C.c_void_p)]
    lib.fpc_sharded_destroy.argtypes = [vp]
    lib.fpc_sharded_info.argtypes = [vp, ip, ip]
    lib.fpc_sharded_matvec.argtypes = [vp, dp, dp]
    lib.fpc_sharded_pc_apply.argtypes = [vp, dp, dp]
    lib.fpc_sharded_gmres.argtypes = [vp, dp, dp, C.POINTER(SolverConfigC), C.POINTER(ReportC), dp, C.c_int]
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code to the exception the reference throws for it."""
    if rc == FPC_OK:
        return
    msg = (_lib.fpc_last_error() or b"").decode()
    if rc == FPC_INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if rc == FPC_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)            # std::runtime_error / CUDA failure
