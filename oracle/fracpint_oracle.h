/*
 * fracpint_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the B200 build.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as the checker.
 * The product path (libfracpint_b200.so) never links or calls it.
 *
 * Every function restates one reference routine of /root/reference/proj/include/fracpint
 * (cited per function in fracpint_oracle.c).  Parity of this restatement is pinned against
 * the reference itself, compiled unchanged from its headers into oracle/_ref/ (see
 * oracle/Makefile and tests/test_oracle_pins.py), and against the reference's own
 * known-answer tests (tests/test_oracle_kat.py).
 *
 * Complex arrays are interleaved (re, im) doubles.  Status codes: 0 ok,
 * 1 invalid_argument, 2 runtime_error (message in orc_last_error()).
 */
#ifndef FRACPINT_ORACLE_H
#define FRACPINT_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* transforms */
void orc_fft_inplace(double* x, size_t n, int sign);
int orc_dst1_real(const double* x, double* y, size_t n);
int orc_dst1_complex(const double* x, double* y, size_t n);

/* discretisation */
int orc_centred_weights(double gamma, int count, double* out);
int orc_toeplitz_matvec(const double* col, size_t n, const double* v, double* out);
int orc_tau_spectrum(const double* col, size_t n, double* sigma);
int orc_tau_solve_shifted(const double* sigma, int nx, int ny, size_t n, double shift_re,
                          double shift_im, double dt, const double* rhs, double* out);
void orc_alpha_circulant_eigenvalues(double alpha, int n_time, double* lambda);
int orc_assemble_rhs(int n_time, int n_space, double dt, const double* f, const double* u0,
                     double* b);

/* problem = spatial Jacobian + time stencil + dt (+ preconditioner plan) */
typedef struct orc_problem orc_problem;

orc_problem* orc_problem_1d(double gamma, double kappa, double h, int n_space, int n_time,
                            double dt);
orc_problem* orc_problem_2d(double gamma_x, double gamma_y, double kappa_x, double kappa_y,
                            double h, int n_per_dim, int n_time, double dt);
void orc_problem_free(orc_problem* p);
size_t orc_problem_dim(const orc_problem* p);
int orc_problem_n_space(const orc_problem* p);
int orc_jacobian_column(const orc_problem* p, int axis, double* col);
int orc_jacobian_apply(const orc_problem* p, const double* v, double* out);
int orc_tau_sigma(const orc_problem* p, double* sigma);
int orc_matvec(const orc_problem* p, const double* v, double* out);

/* plan: alpha <= 0 selects the generalized policy min(0.5, 0.5 dt) */
int orc_build_plan(orc_problem* p, double alpha);
double orc_plan_alpha(const orc_problem* p);
double orc_plan_min_shift_margin(const orc_problem* p);
int orc_plan_n_warnings(const orc_problem* p);
int orc_plan_lambda(const orc_problem* p, double* lambda);
int orc_pc_apply(const orc_problem* p, const double* v, double* out, int full_sweep);
int orc_pc_forward(const orc_problem* p, const double* v, double* out);

/* GMRES (krylov.hpp) with restart emulation: restart <= 0 = unrestarted */
typedef struct {
  int converged;
  int iterations;
  int restarts;
  double final_relative_residual;
  double true_relative_residual;
  int history_len;
} orc_report;

int orc_gmres(const orc_problem* p, const double* b, double* x, double tol, int max_iter,
              int restart, int full_sweep, orc_report* rep, double* history, int history_cap);

/* BiCGSTAB (krylov.hpp:204-280), x0 = 0; *iterations = the reference's double count (k + 0.5
 * for a half-step convergence) */
int orc_bicgstab(const orc_problem* p, const double* b, double* x, double tol, int max_iter,
                 int full_sweep, double* iterations, orc_report* rep, double* history,
                 int history_cap);

#ifdef __cplusplus
}
#endif
#endif
