/*
 * fracpint_b200.h -- C-ABI of the B200-native preconditioned Krylov solve (libfracpint_b200.so).
 *
 * The drop-in boundary for the reference's hot path.  Every entry point replaces
 * one call of the reference's C++ solver API (namespace fracpint, /root/reference/proj/include):
 *
 *   fpc_problem_create_1d  <- RieszJacobian1D(g,k,h,n)         jacobian.hpp:21
 *                             + TimeStencil(nt)                 time_stencil.hpp:23
 *                             + AllAtOnceOperator(st, jac, dt)  all_at_once.hpp:21
 *   fpc_problem_create_2d  <- RieszJacobian2D(gx,gy,kx,ky,h,n)  jacobian.hpp:58 (+ as above)
 *   fpc_matvec             <- AllAtOnceOperator::apply          all_at_once.hpp:33
 *   fpc_assemble_rhs       <- assemble_rhs                      all_at_once.hpp:66
 *   fpc_plan_create        <- build_plan(kind, nt, dt, jac)     alpha_circulant.hpp:84
 *                             (PreconditionerKind::alpha_for    alpha_circulant.hpp:29)
 *   fpc_pc_apply           <- apply_inverse(plan, v, out, sw)   alpha_circulant.hpp:206
 *   fpc_pc_forward         <- apply_forward(plan, v, out)       alpha_circulant.hpp:212
 *   fpc_gmres              <- gmres_right(n, A, P^{-1}, b, cfg) krylov.hpp:84 (+ restart m)
 *   fpc_bicgstab           <- bicgstab_left(n, A, P^{-1}, b, cfg) krylov.hpp:204
 *
 * Plain pointers and sizes only.  Vectors are time-major fp64, v[k*n_space + p] (2D: p = ix*n+iy,
 * x slow; problems.hpp:164-165).  `where` = FPC_HOST (pointers are host memory: copied in and out,
 * the call returns when done) or FPC_DEVICE (device pointers on the context's device; the work is
 * stream-ordered on the context stream, 16-byte aligned pointers required).
 *
 * Threading (the reference's const applies are reentrant, toeplitz.hpp:14-18): every call may come
 * from any host thread.  Calls on one operator / plan are serialised by the library (they share the
 * plan's device spectrum scratch and the operator's host staging buffers) and all device work of a
 * context is ordered on the context's stream, so concurrent calls are safe and run one after the
 * other.  For concurrent device work use one context (stream) and one plan per worker.
 *
 * Status codes mirror the reference's exceptions: FPC_INVALID_ARGUMENT <-> std::invalid_argument,
 * FPC_RUNTIME_ERROR <-> std::runtime_error (numerical singularity), FPC_CUDA_ERROR (device failure),
 * FPC_UNSUPPORTED (a size the B200 kernels do not cover; never a silent CPU fallback).
 * The message of the last failure on the calling thread is fpc_last_error().
 */
#ifndef FRACPINT_B200_H
#define FRACPINT_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPC_OK 0
#define FPC_INVALID_ARGUMENT 1
#define FPC_RUNTIME_ERROR 2
#define FPC_CUDA_ERROR 3
#define FPC_UNSUPPORTED 4

#define FPC_HOST 0
#define FPC_DEVICE 1

#define FPC_SWEEP_HALF 0 /* InnerSweep::half (alpha_circulant.hpp:128) */
#define FPC_SWEEP_FULL 1 /* InnerSweep::full */

#define FPC_ORDER_REFERENCE 0 /* time FFT -> tau solves per frequency -> inverse time FFT (default) */
#define FPC_ORDER_COMMUTED 1  /* DST per time level -> per-mode time solve -> DST */

typedef struct fpc_context_s* fpc_context_t;
typedef struct fpc_problem_s* fpc_problem_t;
typedef struct fpc_plan_s* fpc_plan_t;

/* SolverConfig (krylov.hpp:25-28) + restart (0 = unrestarted, the reference's gmres_right). */
typedef struct {
  double tol;
  int max_iter;
  int restart;
  int sweep;
} fpc_solver_config;

/* SolveReport (krylov.hpp:30-37).  iterations_exact is the reference's double `iterations`
 * (BiCGSTAB converging at a half step reports k + 0.5); `iterations` is its integer part. */
typedef struct {
  int converged;
  int iterations;
  int restarts;
  int reorthogonalizations;
  double final_relative_residual;
  double true_relative_residual;
  double seconds;
  int history_len;
  double iterations_exact;
} fpc_report;

int fpc_abi_version(void);
const char* fpc_last_error(void);

/* host-side setup of the reference API (no device needed; bit-identical to the reference's
 * arithmetic when both are compiled with FMA contraction, as g++ does by default for C++):
 *   fpc_centred_weights            <- centred_weights(gamma, count)          weights.hpp:21-35
 *   fpc_tau_spectrum               <- tau_spectrum(first column)  (n values) tau.hpp:40-55
 *   fpc_circulant_eigenvalues      <- SymToeplitz ctor: FFT of the circulant embedding, real parts
 *                                     k = 0..L/2, L = next_pow2(2n)          toeplitz.hpp:23-35
 *   fpc_alpha_circulant_eigenvalues<- alpha_circulant_eigenvalues(alpha, nt) alpha_circulant.hpp:71-81
 *                                     (nt complex, interleaved re/im) */
int fpc_centred_weights(double gamma, int count, double* out);
int fpc_tau_spectrum(const double* col, int n, double* sigma);
int fpc_circulant_eigenvalues(const double* col, int n, double* eig);
int fpc_alpha_circulant_eigenvalues(double alpha, int nt, double* lambda_interleaved);

/* context: one device, one stream (default: a private non-blocking stream) */
int fpc_context_create(int device, fpc_context_t* out);
int fpc_context_destroy(fpc_context_t ctx);
int fpc_context_set_stream(fpc_context_t ctx, void* cuda_stream);
void* fpc_context_stream(fpc_context_t ctx);
int fpc_synchronize(fpc_context_t ctx);
int fpc_device_alloc(fpc_context_t ctx, size_t bytes, void** out);
int fpc_device_free(fpc_context_t ctx, void* ptr);

/* operator */
int fpc_problem_create_1d(fpc_context_t ctx, double gamma, double kappa, double h, int n_space,
                          int n_time, double dt, fpc_problem_t* out);
int fpc_problem_create_2d(fpc_context_t ctx, double gamma_x, double gamma_y, double kappa_x,
                          double kappa_y, double h, int n_per_dim, int n_time, double dt,
                          fpc_problem_t* out);
int fpc_problem_destroy(fpc_problem_t p);
int fpc_problem_dims(fpc_problem_t p, int* n_time, int* n_space, int* two_dim);
int fpc_problem_first_column(fpc_problem_t p, int axis, double* out);
int fpc_problem_tau_sigma(fpc_problem_t p, double* out);
int fpc_matvec(fpc_problem_t p, const double* v, double* out, int where);
int fpc_assemble_rhs(int n_time, int n_space, double dt, const double* f, const double* u0,
                     double* b);

/* preconditioner plan: alpha <= 0 selects PreconditionerKind::generalized() */
int fpc_plan_create(fpc_problem_t p, double alpha, fpc_plan_t* out);
int fpc_plan_destroy(fpc_plan_t plan);
int fpc_plan_info(fpc_plan_t plan, double* alpha, double* min_shift_margin, int* solve_count,
                  int* n_warnings);
int fpc_plan_lambda(fpc_plan_t plan, double* lambda_interleaved);
/* AlphaCirculantPlan::scale_fwd / scale_bwd (alpha^{+-k/Nt}, n_time values each) */
int fpc_plan_scales(fpc_plan_t plan, double* scale_fwd, double* scale_bwd);
/* half-sweep factor ordering of fpc_pc_apply / fpc_pc_forward / the Krylov solvers (the same
 * operator up to rounding; FPC_UNSUPPORTED for 2D or n_space + 1 > 8192 when commuted) */
int fpc_plan_set_ordering(fpc_plan_t plan, int ordering);
int fpc_pc_apply(fpc_plan_t plan, const double* v, double* out, int sweep, int where);
int fpc_pc_forward(fpc_plan_t plan, const double* v, double* out, int where);

/* right-preconditioned GMRES on the plan's operator, x0 = 0 */
int fpc_gmres(fpc_plan_t plan, const double* b, double* x, const fpc_solver_config* cfg,
              fpc_report* report, double* history, int history_cap, int where);

/* gmres_right(n, apply_a, apply_pinv, b, cfg) for arbitrary host callables (krylov.hpp:83-85, the
 * reference's generic plugin interface): out = op(in) on host arrays of n doubles, return 0 on
 * success (anything else aborts the solve with FPC_RUNTIME_ERROR).  b and x are host arrays.  The
 * Krylov basis lives on the context's device (the library's vector kernels run the Gram-Schmidt
 * with the reference's conditional re-orthogonalisation); each step calls apply_pinv then apply_a
 * once.  cfg->restart = m > 0: GMRES(m); cfg->sweep is ignored. */
typedef int (*fpc_apply_fn)(const double* in, double* out, size_t n, void* user);
int fpc_gmres_callbacks(fpc_context_t ctx, size_t n, fpc_apply_fn apply_a, void* a_user,
                        fpc_apply_fn apply_pinv, void* p_user, const double* b, double* x,
                        const fpc_solver_config* cfg, fpc_report* report, double* history,
                        int history_cap);

/* left-preconditioned BiCGSTAB on the plan's operator, x0 = 0 (cfg->restart is ignored) */
int fpc_bicgstab(fpc_plan_t plan, const double* b, double* x, const fpc_solver_config* cfg,
                 fpc_report* report, double* history, int history_cap, int where);

/* shard level: the per-rank pieces of the frequency-sharded multi-GPU solve
 * (paper_2003_07020_b200/distributed.py).  Device pointers, stream-ordered; sizes are local.
 *   matvec on nt_local time blocks starting at global level k_offset (the two previous blocks must
 *     sit right before v when k_offset > 0)                           all_at_once.hpp:33-55
 *   time_fwd / time_inv on ns_local spatial columns (row stride ns_local), Z half spectrum
 *     [Nt/2+1][ns_local] complex                                      alpha_circulant.hpp:146-198
 *   tau on frequency rows [row0, row0+nrows) of a [nrows][n_space] complex block  tau.hpp:98-136
 *   dots / update / lincomb: the Gram-Schmidt vector kernels on local shards   krylov.hpp:116-183
 * commuted ordering (n_space + 1 <= 8192), two all-to-alls per apply:
 *   dst_levels: out = s_in * S v for nt_local contiguous time levels (nt_local even)  dst.hpp:21-43
 *   time_solve: per spatial column p in [col0, col0 + ns_local) of a [Nt][ns_local] block,
 *     z = D^-1 F^* diag(1/(lambda_n - dt sigma_p)) F D u (forward != 0: multiply)  alpha_circulant.hpp:137-199 */
int fpc_shard_matvec(fpc_problem_t p, const double* v, double* y, int nt_local, int k_offset);
int fpc_shard_time_fwd(fpc_plan_t plan, const double* v, double* Z, int ns_local, double s_in);
int fpc_shard_tau(fpc_plan_t plan, double* Z, int row0, int nrows, int forward);
int fpc_shard_time_inv(fpc_plan_t plan, const double* Z, double* z, int ns_local);
int fpc_shard_dots(fpc_context_t ctx, const double* const* V, const double* scales, int nv,
                   const double* w, size_t n, int with_norm, double* out_host);
int fpc_shard_update(fpc_context_t ctx, const double* const* V, const double* coef, int nv,
                     double* w, size_t n, double* norm2_host);
/* the same two with the results left in device memory (stream-ordered, no host synchronisation):
 * the sharded solver all-reduces them on the device and reads the sum once per reduction */
int fpc_shard_dots_dev(fpc_context_t ctx, const double* const* V, const double* scales, int nv,
                       const double* w, size_t n, int with_norm, double* out_dev);
int fpc_shard_update_dev(fpc_context_t ctx, const double* const* V, const double* coef, int nv,
                         double* w, size_t n, double* norm2_dev);
int fpc_shard_lincomb(fpc_context_t ctx, const double* const* V, const double* coef, int nv,
                      double* u, size_t n);
int fpc_shard_dst_levels(fpc_plan_t plan, const double* v, double* out, int nt_local, double s_in);
int fpc_shard_time_solve(fpc_plan_t plan, const double* u, double* z, int col0, int ns_local, int forward);

/* Peer-store transport for the sharded PC apply's exchanges (replaces NCCL all_to_all_single + the
 * pack/unpack copies around it; distributed.py ShardedSolver(transport="p2p")).  The receive
 * buffers are plain device allocations shared by CUDA IPC:
 *   fpc_ipc_get_handle: 64-byte cudaIpcMemHandle_t of a device allocation (fpc_device_alloc)
 *   fpc_ipc_open: map a peer's handle (another process, same node) -> device pointer; fpc_ipc_close
 *   fpc_shard_scatter_p2p: src [rows][cols] elements of es doubles (1 real, 2 complex); the split
 *     dimension (columns if split_cols, else rows) is partitioned by off[0..nranks) (rank d owns
 *     [off[d], off[d+1]), off[nranks] = the dimension); element (i, j) owned by d is stored to
 *       split_cols: dst[d][(row_base + i) * stride[d] + col_base + (j - off[d])]
 *       split rows: dst[d][(row_base + i - off[d]) * stride[d] + col_base + j]
 *     (elements of es doubles), stream-ordered on the context stream, ending with a system-scope
 *     fence; the caller orders consumers behind a cross-rank barrier on the same stream.  nranks <= 8. */
int fpc_ipc_get_handle(const void* dptr, void* handle64);
int fpc_ipc_open(fpc_context_t ctx, const void* handle64, void** dptr);
int fpc_ipc_close(fpc_context_t ctx, void* dptr);
int fpc_shard_scatter_p2p(fpc_context_t ctx, const double* src, int rows, int cols, int es, int split_cols,
                          double* const* dst, const int* off, const int* stride, int nranks, int row_base,
                          int col_base);

/* Multi-device solve in ONE process: a context over 1..8 devices (peer access
 * enabled between distinct devices; a device may repeat, which runs the rank schedule on one GPU) and
 * the frequency-sharded operator on it -- time-sharded Krylov vectors, the BDF2 halo by peer copy,
 * the PC apply's four transpositions as peer-store kernels, the retained frequencies' tau solves
 * split across the ranks, Gram-Schmidt partials summed in rank order.  Host buffers hold the whole
 * time-major vector.  n_time must be divisible by the rank count (>= 2 levels per rank).
 * alpha <= 0 selects PreconditionerKind::generalized().  Replaces, for a C++ caller of
 * solve_all_at_once (driver.hpp:49-92), the Python/torchrun ShardedSolver. */
typedef struct fpc_multi_s* fpc_multi_t;
typedef struct fpc_sharded_s* fpc_sharded_t;
int fpc_multi_create(const int* devices, int n_ranks, fpc_multi_t* out);
int fpc_multi_destroy(fpc_multi_t m);
int fpc_sharded_create_1d(fpc_multi_t m, double gamma, double kappa, double h, int n_space, int n_time,
                          double dt, double alpha, fpc_sharded_t* out);
int fpc_sharded_create_2d(fpc_multi_t m, double gamma_x, double gamma_y, double kappa_x, double kappa_y,
                          double h, int n_per_dim, int n_time, double dt, double alpha, fpc_sharded_t* out);
int fpc_sharded_destroy(fpc_sharded_t s);
int fpc_sharded_info(fpc_sharded_t s, int* n_ranks, int* nt_local);
int fpc_sharded_matvec(fpc_sharded_t s, const double* v, double* out);
int fpc_sharded_pc_apply(fpc_sharded_t s, const double* v, double* out);
int fpc_sharded_gmres(fpc_sharded_t s, const double* b, double* x, const fpc_solver_config* cfg,
                      fpc_report* report, double* history, int history_cap);

/* instrumentation: number of kernels this library launched in this process */
unsigned long long fpc_kernel_launches(void);
/* live per-kernel device time: CUDA events on the launching stream around every launch while
 * enabled.  stop() synchronizes the device and returns the number of kernel categories. */
int fpc_profile_start(void);
int fpc_profile_stop(void);
int fpc_profile_entry(int index, char* name, int name_cap, double* total_ms, long long* launches);

#ifdef __cplusplus
}
#endif
#endif
