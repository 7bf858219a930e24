/*
 * fracpint_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY:
 * the checker for the CUDA path, never the thing measured or shipped (see fracpint_oracle.h).
 *
 * Reference = /root/reference/proj/include/fracpint/*.hpp (header-only C++20).  Each routine
 * below cites the reference lines it restates and keeps the reference's operation order so
 * the two agree to rounding (pinned in tests/test_oracle_pins.py against oracle/_ref, the
 * reference compiled unchanged).  The independent per-time-level / per-column / per-frequency
 * loops run on a fork-join pool like the reference's parallel_for (parallel.hpp:27-60, contiguous
 * static partition): every iteration writes disjoint outputs with its own scratch, so the numbers
 * do not depend on the thread count (ORC_THREADS, default all cores).  Reductions -- dots, norms --
 * stay serial left-to-right sums (krylov.hpp:52-56).
 */
#include "fracpint_oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

static const double kPi = 3.14159265358979323846264338327950288;

static _Thread_local char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- fork-join (parallel.hpp:24-60) */
typedef void (*range_fn)(void* ctx, size_t lo, size_t hi);
typedef struct {
  range_fn fn;
  void* ctx;
  size_t lo, hi;
} range_job;
static void* range_run(void* a) {
  range_job* j = (range_job*)a;
  if (j->lo < j->hi) j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}
static int thread_count(void) {
  const char* e = getenv("ORC_THREADS");
  long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  return t < 1 ? 1 : (t > 256 ? 256 : (int)t);
}
/* fn over [0, n) in contiguous chunks, one per thread (the calling thread takes the first). */
static void par_for(size_t n, range_fn fn, void* ctx) {
  int T = thread_count();
  if ((size_t)T > n) T = (int)(n ? n : 1);
  if (T <= 1) {
    if (n) fn(ctx, 0, n);
    return;
  }
  range_job jobs[256];
  pthread_t th[256];
  for (int t = 0; t < T; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].lo = n * (size_t)t / (size_t)T;
    jobs[t].hi = n * (size_t)(t + 1) / (size_t)T;
  }
  int started[256] = {0};
  for (int t = 1; t < T; ++t) started[t] = pthread_create(&th[t], NULL, range_run, &jobs[t]) == 0;
  range_run(&jobs[0]);
  for (int t = 1; t < T; ++t) {
    if (started[t]) pthread_join(th[t], NULL);
    else range_run(&jobs[t]);
  }
}

/* ---------------------------------------------------------------- FFT (fft.hpp) */

static size_t next_pow2(size_t n) { /* fft.hpp:17-21 */
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
static int is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; } /* fft.hpp:23 */

/* Pow2Plan (fft.hpp:28-39): bit-reversal table + twiddles polar(1, sign*2*pi*j/n), j<n/2.
 * Cached per (n, sign) like pow2_plan (fft.hpp:41-47). */
typedef struct {
  size_t n;
  int sign;
  uint32_t* rev;
  cplx* tw;
} pow2_plan_t;

static _Thread_local pow2_plan_t g_plans[64];
static _Thread_local int g_nplans;

static const pow2_plan_t* pow2_plan(size_t n, int sign) {
  int s = sign >= 0 ? 1 : -1;
  for (int i = 0; i < g_nplans; ++i)
    if (g_plans[i].n == n && g_plans[i].sign == s) return &g_plans[i];
  pow2_plan_t* p;
  if (g_nplans < 64) {
    p = &g_plans[g_nplans++];
  } else { /* evict slot 0 (oracle only ever uses a handful of sizes) */
    p = &g_plans[0];
    free(p->rev);
    free(p->tw);
  }
  p->n = n;
  p->sign = s;
  p->rev = (uint32_t*)calloc(n, sizeof(uint32_t));
  p->tw = (cplx*)malloc((n / 2 + 1) * sizeof(cplx));
  for (size_t i = 1; i < n; ++i)
    p->rev[i] = (p->rev[i >> 1] >> 1) | ((i & 1) ? (uint32_t)(n >> 1) : 0u);
  const double unit = 2.0 * kPi * (s >= 0 ? 1.0 : -1.0) / (double)n;
  for (size_t j = 0; j < n / 2; ++j) {
    const double th = unit * (double)j;
    p->tw[j] = cos(th) + I * sin(th); /* std::polar(1, th) */
  }
  return p;
}

/* fft_pow2 (fft.hpp:49-67): iterative radix-2 DIT after bit reversal. */
static void fft_pow2(cplx* x, size_t n, int sign) {
  if (n <= 1) return;
  const pow2_plan_t* plan = pow2_plan(n, sign);
  for (size_t i = 0; i < n; ++i)
    if (i < plan->rev[i]) {
      cplx t = x[i];
      x[i] = x[plan->rev[i]];
      x[plan->rev[i]] = t;
    }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len >> 1;
    const size_t step = n / len;
    for (size_t base = 0; base < n; base += len) {
      for (size_t j = 0; j < half; ++j) {
        const cplx w = plan->tw[j * step];
        const cplx u = x[base + j];
        const cplx v = x[base + j + half] * w;
        x[base + j] = u + v;
        x[base + j + half] = u - v;
      }
    }
  }
}

/* fft_bluestein (fft.hpp:71-89): chirp-z for non-power-of-two n. */
static void fft_bluestein(cplx* x, size_t n, int sign) {
  const size_t L = next_pow2(2 * n - 1);
  const double dir = sign >= 0 ? 1.0 : -1.0;
  cplx* chirp = (cplx*)malloc(n * sizeof(cplx));
  cplx* a = (cplx*)calloc(L, sizeof(cplx));
  cplx* b = (cplx*)calloc(L, sizeof(cplx));
  for (size_t m = 0; m < n; ++m) {
    const uint64_t sq = ((uint64_t)m * m) % (2 * n);
    const double th = dir * kPi * (double)sq / (double)n;
    chirp[m] = cos(th) + I * sin(th);
  }
  for (size_t j = 0; j < n; ++j) a[j] = x[j] * chirp[j];
  b[0] = conj(chirp[0]);
  for (size_t m = 1; m < n; ++m) b[m] = b[L - m] = conj(chirp[m]);
  fft_pow2(a, L, -1);
  fft_pow2(b, L, -1);
  for (size_t j = 0; j < L; ++j) a[j] *= b[j];
  fft_pow2(a, L, 1);
  const double inv_L = 1.0 / (double)L;
  for (size_t k = 0; k < n; ++k) x[k] = chirp[k] * a[k] * inv_L;
  free(chirp);
  free(a);
  free(b);
}

/* fft_inplace (fft.hpp:95-101): unnormalised, x[k] <- sum_j x[j] e^{sign 2 pi i jk/n}. */
static void fft_c(cplx* x, size_t n, int sign) {
  if (n <= 1) return;
  if (is_pow2(n))
    fft_pow2(x, n, sign);
  else
    fft_bluestein(x, n, sign);
}
void orc_fft_inplace(double* x, size_t n, int sign) { fft_c((cplx*)x, n, sign); }

/* ---------------------------------------------------------------- DST-I (dst.hpp:21-43) */

/* Orthonormal DST-I through the length-2(n+1) odd extension and one complex FFT with the
 * negative-exponent kernel; y[k] = sqrt(2/(n+1))/2 * i*V[k+1].  `complex_in` selects the
 * complex Scalar instantiation (dst.hpp:161-164). In/out may alias. */
static void dst1_any(const cplx* x, cplx* y, size_t n, int complex_out, double* yreal) {
  if (n == 0) return;
  const size_t L = 2 * (n + 1);
  cplx* v = (cplx*)calloc(L, sizeof(cplx));
  for (size_t j = 0; j < n; ++j) {
    v[j + 1] = x[j];
    v[L - 1 - j] = -x[j];
  }
  fft_c(v, L, -1);
  const double scale = sqrt(2.0 / (double)(n + 1)) * 0.5;
  for (size_t k = 0; k < n; ++k) {
    const cplx s = I * v[k + 1];
    if (complex_out)
      y[k] = scale * s;
    else
      yreal[k] = scale * creal(s);
  }
  free(v);
}

int orc_dst1_real(const double* x, double* y, size_t n) {
  cplx* t = (cplx*)malloc((n ? n : 1) * sizeof(cplx));
  for (size_t j = 0; j < n; ++j) t[j] = x[j];
  dst1_any(t, NULL, n, 0, y);
  free(t);
  return 0;
}
int orc_dst1_complex(const double* x, double* y, size_t n) {
  dst1_any((const cplx*)x, (cplx*)y, n, 1, NULL);
  return 0;
}

/* ---------------------------------------------------------------- weights.hpp:21-35 */

int orc_centred_weights(double gamma, int count, double* w) {
  if (!(gamma > 1.0) || !(gamma <= 2.0))
    return fail(1, "centred_weights: gamma must lie in (1, 2]");
  if (count < 1) return fail(1, "centred_weights: count must be at least 1");
  const double g0 = tgamma(1.0 + gamma / 2.0);
  w[0] = tgamma(1.0 + gamma) / (g0 * g0);
  for (int l = 0; l + 1 < count; ++l)
    w[l + 1] = w[l] * ((double)l - gamma / 2.0) / ((double)l + 1.0 + gamma / 2.0);
  return 0;
}

/* ---------------------------------------------------------------- SymToeplitz (toeplitz.hpp) */

typedef struct {
  size_t n, L;
  double* col;
  cplx* eigs;
} toep_t;

static int toep_init(toep_t* t, const double* col, size_t n) { /* toeplitz.hpp:23-35 */
  if (n == 0) return fail(1, "SymToeplitz: empty first column");
  t->n = n;
  t->L = next_pow2(2 * n);
  t->col = (double*)malloc(n * sizeof(double));
  memcpy(t->col, col, n * sizeof(double));
  t->eigs = (cplx*)calloc(t->L, sizeof(cplx));
  t->eigs[0] = col[0];
  for (size_t j = 1; j < n; ++j) {
    t->eigs[j] = col[j];
    t->eigs[t->L - j] = col[j];
  }
  fft_c(t->eigs, t->L, -1);
  return 0;
}
static void toep_free(toep_t* t) {
  free(t->col);
  free(t->eigs);
  t->col = NULL;
  t->eigs = NULL;
}

/* SymToeplitz::matvec (toeplitz.hpp:41-57): FFT(-1) -> x eigs -> FFT(+1) -> /L.
 * Real (double) or complex Scalar; `cin`/`cout` complex interleaved when is_complex. */
static void toep_matvec(const toep_t* t, const void* v, void* out, int is_complex, cplx* w) {
  const size_t n = t->n, L = t->L;
  memset(w, 0, L * sizeof(cplx));
  if (is_complex)
    for (size_t j = 0; j < n; ++j) w[j] = ((const cplx*)v)[j];
  else
    for (size_t j = 0; j < n; ++j) w[j] = ((const double*)v)[j];
  fft_c(w, L, -1);
  for (size_t j = 0; j < L; ++j) w[j] *= t->eigs[j];
  fft_c(w, L, +1);
  const double inv_L = 1.0 / (double)L;
  if (is_complex)
    for (size_t j = 0; j < n; ++j) ((cplx*)out)[j] = w[j] * inv_L;
  else
    for (size_t j = 0; j < n; ++j) ((double*)out)[j] = creal(w[j]) * inv_L;
}

int orc_toeplitz_matvec(const double* col, size_t n, const double* v, double* out) {
  toep_t t;
  int rc = toep_init(&t, col, n);
  if (rc) return rc;
  cplx* w = (cplx*)malloc(t.L * sizeof(cplx));
  toep_matvec(&t, v, out, 0, w);
  free(w);
  toep_free(&t);
  return 0;
}

/* ---------------------------------------------------------------- tau.hpp */

/* tau_spectrum (tau.hpp:40-55): c_l = a_l - a_{l+2}; sigma_i = DST(c)_i / DST(e1)_i. */
int orc_tau_spectrum(const double* a, size_t n, double* sigma) {
  double* corrected = (double*)malloc(n * sizeof(double));
  double* num = (double*)malloc(n * sizeof(double));
  memcpy(corrected, a, n * sizeof(double));
  for (size_t l = 0; l + 2 < n; ++l) corrected[l] -= a[l + 2];
  orc_dst1_real(corrected, num, n);
  const double root = sqrt(2.0 / (double)(n + 1));
  for (size_t i = 0; i < n; ++i) {
    const double denom = root * sin(kPi * (double)(i + 1) / (double)(n + 1));
    sigma[i] = num[i] / denom;
  }
  free(corrected);
  free(num);
  return 0;
}

/* dst_lattice_inplace (tau.hpp:79-96): 1D DST, or 2D rows (contiguous) then columns. */
static void dst_lattice(int nx, int ny, size_t n, cplx* z) {
  if (nx <= 0) {
    dst1_any(z, z, n, 1, NULL);
    return;
  }
  for (int ix = 0; ix < nx; ++ix) dst1_any(z + (size_t)ix * ny, z + (size_t)ix * ny, ny, 1, NULL);
  cplx* col = (cplx*)malloc((size_t)nx * sizeof(cplx));
  for (int iy = 0; iy < ny; ++iy) {
    for (int ix = 0; ix < nx; ++ix) col[ix] = z[(size_t)ix * ny + iy];
    dst1_any(col, col, nx, 1, NULL);
    for (int ix = 0; ix < nx; ++ix) z[(size_t)ix * ny + iy] = col[ix];
  }
  free(col);
}

/* tau_shifted<Solve> (tau.hpp:98-119). */
static int tau_shifted(int solve, const double* sigma, int nx, int ny, size_t n, cplx shift,
                       double dt, const cplx* rhs, cplx* out) {
  for (size_t i = 0; i < n; ++i) out[i] = rhs[i];
  dst_lattice(nx, ny, n, out);
  if (solve) {
    double max_sigma = 0.0;
    for (size_t i = 0; i < n; ++i) max_sigma = fmax(max_sigma, fabs(sigma[i]));
    const double floor_ = 1e-14 * (cabs(shift) + fabs(dt) * max_sigma);
    for (size_t i = 0; i < n; ++i) {
      const cplx denom = shift - dt * sigma[i];
      if (cabs(denom) <= floor_)
        return fail(2, "tau_solve_shifted: shift is numerically singular");
      out[i] /= denom;
    }
  } else {
    for (size_t i = 0; i < n; ++i) out[i] *= shift - dt * sigma[i];
  }
  dst_lattice(nx, ny, n, out);
  return 0;
}

int orc_tau_solve_shifted(const double* sigma, int nx, int ny, size_t n, double sr, double si,
                          double dt, const double* rhs, double* out) {
  return tau_shifted(1, sigma, nx, ny, n, sr + I * si, dt, (const cplx*)rhs, (cplx*)out);
}

/* ---------------------------------------------------------------- alpha_circulant.hpp:71-81 */

static void lambda_c(double alpha, int nt, cplx* lambda) {
  const double a = pow(alpha, 1.0 / (double)nt);
  for (int i = 0; i < nt; ++i) {
    const double ang1 = 2.0 * kPi * (double)(i % nt) / nt;
    const double ang2 = 2.0 * kPi * (double)((2 * i) % nt) / nt;
    lambda[i] = 1.5 - 2.0 * a * (cos(ang1) + I * sin(ang1)) +
                0.5 * a * a * (cos(ang2) + I * sin(ang2));
  }
}
void orc_alpha_circulant_eigenvalues(double alpha, int nt, double* lambda) {
  lambda_c(alpha, nt, (cplx*)lambda);
}

/* assemble_rhs (all_at_once.hpp:66-80). */
int orc_assemble_rhs(int nt, int ns, double dt, const double* f, const double* u0, double* b) {
  const size_t NS = (size_t)ns, NT = (size_t)nt;
  for (size_t k = 0; k < NT; ++k)
    for (size_t i = 0; i < NS; ++i) b[k * NS + i] = dt * f[k * NS + i];
  for (size_t i = 0; i < NS; ++i) {
    b[i] += u0[i];
    b[NS + i] -= 0.5 * u0[i];
  }
  return 0;
}

/* ---------------------------------------------------------------- problem (jacobian.hpp) */

struct orc_problem {
  int two_dim;
  int n;   /* 1D: n_space; 2D: n per dim */
  int ns;  /* spatial unknowns */
  int nt;
  double dt;
  double sx, sy;  /* 2D scalings kappa/h^gamma (jacobian.hpp:67-68) */
  toep_t tx, ty;  /* 1D uses tx only (already scaled column, jacobian.hpp:27-31) */
  double* sigma;  /* jac.tau() */
  /* plan (alpha_circulant.hpp:52-67) */
  int has_plan;
  double alpha;
  cplx* lambda;
  double* scale_fwd;
  double* scale_bwd;
  int solve_count;
  double min_shift_margin;
  int n_warnings;
};

static orc_problem* problem_alloc(void) { return (orc_problem*)calloc(1, sizeof(orc_problem)); }

/* RieszJacobian1D ctor (jacobian.hpp:21-32). */
orc_problem* orc_problem_1d(double gamma, double kappa, double h, int n, int nt, double dt) {
  if (!(kappa > 0.0)) return fail(1, "RieszJacobian1D: kappa must be positive"), NULL;
  if (!(h > 0.0)) return fail(1, "RieszJacobian1D: h must be positive"), NULL;
  if (n < 1) return fail(1, "RieszJacobian1D: n_space must be at least 1"), NULL;
  if (nt < 3) return fail(1, "TimeStencil: need at least 3 time levels"), NULL;
  if (!(dt > 0.0)) return fail(1, "AllAtOnceOperator: dt must be positive"), NULL;
  double* w = (double*)malloc((size_t)n * sizeof(double));
  if (orc_centred_weights(gamma, n, w)) {
    free(w);
    return NULL;
  }
  const double scale = -kappa / pow(h, gamma);
  for (int l = 0; l < n; ++l) w[l] = scale * w[l];
  orc_problem* p = problem_alloc();
  p->n = n;
  p->ns = n;
  p->nt = nt;
  p->dt = dt;
  toep_init(&p->tx, w, (size_t)n);
  p->sigma = (double*)malloc((size_t)n * sizeof(double));
  orc_tau_spectrum(p->tx.col, (size_t)n, p->sigma); /* jacobian.hpp:45 */
  free(w);
  return p;
}

/* RieszJacobian2D ctor (jacobian.hpp:58-69) + tau (96-98, tau.hpp:59-73). */
orc_problem* orc_problem_2d(double gx, double gy, double kx, double ky, double h, int n, int nt,
                            double dt) {
  if (!(kx > 0.0) || !(ky > 0.0))
    return fail(1, "RieszJacobian2D: diffusion coefficients must be positive"), NULL;
  if (!(h > 0.0)) return fail(1, "RieszJacobian2D: h must be positive"), NULL;
  if (n < 1) return fail(1, "RieszJacobian2D: n_per_dim must be at least 1"), NULL;
  if (nt < 3) return fail(1, "TimeStencil: need at least 3 time levels"), NULL;
  if (!(dt > 0.0)) return fail(1, "AllAtOnceOperator: dt must be positive"), NULL;
  double* wx = (double*)malloc((size_t)n * sizeof(double));
  double* wy = (double*)malloc((size_t)n * sizeof(double));
  if (orc_centred_weights(gx, n, wx) || orc_centred_weights(gy, n, wy)) {
    free(wx);
    free(wy);
    return NULL;
  }
  orc_problem* p = problem_alloc();
  p->two_dim = 1;
  p->n = n;
  p->ns = n * n;
  p->nt = nt;
  p->dt = dt;
  toep_init(&p->tx, wx, (size_t)n);
  toep_init(&p->ty, wy, (size_t)n);
  p->sx = kx / pow(h, gx);
  p->sy = ky / pow(h, gy);
  double* sgx = (double*)malloc((size_t)n * sizeof(double));
  double* sgy = (double*)malloc((size_t)n * sizeof(double));
  orc_tau_spectrum(wx, (size_t)n, sgx);
  orc_tau_spectrum(wy, (size_t)n, sgy);
  p->sigma = (double*)malloc((size_t)n * n * sizeof(double));
  for (int ix = 0; ix < n; ++ix)
    for (int iy = 0; iy < n; ++iy)
      p->sigma[(size_t)ix * n + iy] = (-p->sx) * sgx[ix] + (-p->sy) * sgy[iy];
  free(sgx);
  free(sgy);
  free(wx);
  free(wy);
  return p;
}

void orc_problem_free(orc_problem* p) {
  if (!p) return;
  toep_free(&p->tx);
  if (p->two_dim) toep_free(&p->ty);
  free(p->sigma);
  free(p->lambda);
  free(p->scale_fwd);
  free(p->scale_bwd);
  free(p);
}

size_t orc_problem_dim(const orc_problem* p) { return (size_t)p->nt * (size_t)p->ns; }
int orc_problem_n_space(const orc_problem* p) { return p->ns; }

int orc_jacobian_column(const orc_problem* p, int axis, double* col) {
  const toep_t* t = (axis == 1 && p->two_dim) ? &p->ty : &p->tx;
  memcpy(col, t->col, t->n * sizeof(double));
  return 0;
}

int orc_tau_sigma(const orc_problem* p, double* sigma) {
  memcpy(sigma, p->sigma, (size_t)p->ns * sizeof(double));
  return 0;
}

/* jac.apply<double>: 1D = Toeplitz (jacobian.hpp:40-43); 2D = rows then columns
 * (jacobian.hpp:77-94). `scratch` holds >= max(L) complex; `buf`,`res` >= n doubles. */
static void jac_apply(const orc_problem* p, const double* v, double* out, cplx* scratch,
                      double* buf, double* res) {
  if (!p->two_dim) {
    toep_matvec(&p->tx, v, out, 0, scratch);
    return;
  }
  const size_t n = (size_t)p->n;
  for (size_t ix = 0; ix < n; ++ix) {
    toep_matvec(&p->ty, v + ix * n, res, 0, scratch);
    for (size_t iy = 0; iy < n; ++iy) out[ix * n + iy] = -p->sy * res[iy];
  }
  for (size_t iy = 0; iy < n; ++iy) {
    for (size_t ix = 0; ix < n; ++ix) buf[ix] = v[ix * n + iy];
    toep_matvec(&p->tx, buf, res, 0, scratch);
    for (size_t ix = 0; ix < n; ++ix) out[ix * n + iy] -= p->sx * res[ix];
  }
}

static size_t scratch_len(const orc_problem* p) {
  size_t L = p->tx.L;
  if (p->two_dim && p->ty.L > L) L = p->ty.L;
  return L;
}

int orc_jacobian_apply(const orc_problem* p, const double* v, double* out) {
  cplx* s = (cplx*)malloc(scratch_len(p) * sizeof(cplx));
  double* buf = (double*)malloc((size_t)p->n * sizeof(double));
  double* res = (double*)malloc((size_t)p->n * sizeof(double));
  jac_apply(p, v, out, s, buf, res);
  free(s);
  free(buf);
  free(res);
  return 0;
}

/* AllAtOnceOperator::apply (all_at_once.hpp:33-55): y_k = C-stencil(v)_k - dt A v_k. */
typedef struct {
  const orc_problem* p;
  const double* v;
  double* out;
} mv_ctx;
static void matvec_levels(void* c_, size_t k0, size_t k1) {
  const mv_ctx* c = (const mv_ctx*)c_;
  const orc_problem* p = c->p;
  const double* v = c->v;
  const size_t ns = (size_t)p->ns;
  cplx* s = (cplx*)malloc(scratch_len(p) * sizeof(cplx));
  double* buf = (double*)malloc((size_t)p->n * sizeof(double));
  double* res = (double*)malloc((size_t)p->n * sizeof(double));
  for (size_t k = k0; k < k1; ++k) {
    double* o = c->out + k * ns;
    jac_apply(p, v + k * ns, o, s, buf, res);
    const double* vk = v + k * ns;
    const double* vk1 = k >= 1 ? v + (k - 1) * ns : NULL;
    const double* vk2 = k >= 2 ? v + (k - 2) * ns : NULL;
    for (size_t i = 0; i < ns; ++i) {
      double c_k;
      if (k == 0)
        c_k = vk[i];
      else if (k == 1)
        c_k = 1.5 * vk[i] + -2.0 * vk1[i];
      else
        c_k = 1.5 * vk[i] + -2.0 * vk1[i] + 0.5 * vk2[i];
      o[i] = c_k - p->dt * o[i];
    }
  }
  free(s);
  free(buf);
  free(res);
}
int orc_matvec(const orc_problem* p, const double* v, double* out) {
  mv_ctx c = {p, v, out};
  par_for((size_t)p->nt, matvec_levels, &c);
  return 0;
}

/* ---------------------------------------------------------------- plan (alpha_circulant.hpp:83-126) */

int orc_build_plan(orc_problem* p, double alpha_in) {
  const int nt = p->nt;
  const double dt = p->dt;
  /* PreconditionerKind::alpha_for (alpha_circulant.hpp:29-34); alpha_in<=0 => generalized */
  const double a = alpha_in <= 0.0 ? fmin(0.5, 0.5 * dt) : alpha_in;
  if (!(a > 0.0) || a > 1.0) return fail(1, "PreconditionerKind: alpha must lie in (0, 1]");
  free(p->lambda);
  free(p->scale_fwd);
  free(p->scale_bwd);
  p->alpha = a;
  p->n_warnings = a < 1e-8 ? 1 : 0;
  p->lambda = (cplx*)malloc((size_t)nt * sizeof(cplx));
  lambda_c(a, nt, p->lambda);
  p->scale_fwd = (double*)malloc((size_t)nt * sizeof(double));
  p->scale_bwd = (double*)malloc((size_t)nt * sizeof(double));
  for (int k = 0; k < nt; ++k) {
    const double e = (double)k / (double)nt;
    p->scale_fwd[k] = pow(a, e);
    p->scale_bwd[k] = pow(a, -e);
  }
  p->solve_count = nt / 2 + 1;
  double max_sigma = 0.0;
  for (int i = 0; i < p->ns; ++i) max_sigma = fmax(max_sigma, fabs(p->sigma[i]));
  double margin = INFINITY;
  for (int n = 0; n < p->solve_count; ++n) {
    const cplx l = p->lambda[n];
    const double floor_ = 1e-14 * (cabs(l) + dt * max_sigma);
    for (int i = 0; i < p->ns; ++i) {
      const double d = cabs(l - dt * p->sigma[i]);
      margin = fmin(margin, d);
      if (d <= floor_) {
        p->has_plan = 0;
        return fail(2, "build_plan: an inner shifted system is numerically singular");
      }
    }
  }
  p->min_shift_margin = margin;
  p->has_plan = 1;
  return 0;
}

double orc_plan_alpha(const orc_problem* p) { return p->alpha; }
double orc_plan_min_shift_margin(const orc_problem* p) { return p->min_shift_margin; }
int orc_plan_n_warnings(const orc_problem* p) { return p->n_warnings; }
int orc_plan_lambda(const orc_problem* p, double* lambda) {
  if (!p->has_plan) return fail(1, "no plan");
  memcpy(lambda, p->lambda, (size_t)p->nt * sizeof(cplx));
  return 0;
}

/* alpha_circulant_action<Solve> (alpha_circulant.hpp:137-199). */
typedef struct {
  const orc_problem* p;
  int solve;
  const double* v;
  cplx* rows;
  cplx* blocks;
  int* rcs;
} pc_ctx;
static void pc_fwd_cols(void* c_, size_t j0, size_t j1) { /* alpha_circulant.hpp:146-152 */
  const pc_ctx* c = (const pc_ctx*)c_;
  const size_t nt = (size_t)c->p->nt, ns = (size_t)c->p->ns;
  for (size_t j = j0; j < j1; ++j) {
    cplx* row = c->rows + j * nt;
    for (size_t k = 0; k < nt; ++k) row[k] = c->p->scale_fwd[k] * c->v[k * ns + j];
    fft_c(row, nt, +1);
  }
}
static void pc_transpose_fwd(void* c_, size_t n0, size_t n1) { /* alpha_circulant.hpp:153-156 */
  const pc_ctx* c = (const pc_ctx*)c_;
  const size_t nt = (size_t)c->p->nt, ns = (size_t)c->p->ns;
  for (size_t n = n0; n < n1; ++n)
    for (size_t j = 0; j < ns; ++j) c->blocks[n * ns + j] = c->rows[j * nt + n];
}
static void pc_tau(void* c_, size_t n0, size_t n1) { /* alpha_circulant.hpp:158-166 */
  const pc_ctx* c = (const pc_ctx*)c_;
  const orc_problem* p = c->p;
  const size_t ns = (size_t)p->ns;
  const int nx = p->two_dim ? p->n : 0, ny = p->two_dim ? p->n : 0;
  for (size_t n = n0; n < n1; ++n) {
    cplx* z = c->blocks + n * ns;
    c->rcs[n] = tau_shifted(c->solve, p->sigma, nx, ny, ns, p->lambda[n], p->dt, z, z);
  }
}
static void pc_inv_cols(void* c_, size_t j0, size_t j1) { /* alpha_circulant.hpp:176-186 */
  const pc_ctx* c = (const pc_ctx*)c_;
  const size_t nt = (size_t)c->p->nt, ns = (size_t)c->p->ns;
  for (size_t j = j0; j < j1; ++j) {
    cplx* row = c->rows + j * nt;
    for (size_t k = 0; k < nt; ++k) row[k] = c->blocks[k * ns + j];
    fft_c(row, nt, -1);
  }
}

static int pc_action(const orc_problem* p, int solve, int full_sweep, const double* v,
                     double* out) {
  if (!p->has_plan) return fail(1, "alpha-circulant action: no plan built");
  const size_t nt = (size_t)p->nt, ns = (size_t)p->ns;
  pc_ctx c = {p, solve, v, NULL, NULL, NULL};
  c.rows = (cplx*)malloc(nt * ns * sizeof(cplx)); /* space-major rows[j*nt+k] */
  par_for(ns, pc_fwd_cols, &c);
  c.blocks = (cplx*)malloc(nt * ns * sizeof(cplx)); /* time-major blocks[n*ns+j] */
  par_for(nt, pc_transpose_fwd, &c);
  const size_t active = (solve && !full_sweep) ? (size_t)p->solve_count : nt;
  c.rcs = (int*)calloc(active ? active : 1, sizeof(int));
  par_for(active, pc_tau, &c);
  int rc = 0;
  for (size_t n = 0; n < active && !rc; ++n) rc = c.rcs[n];
  free(c.rcs);
  cplx* rows = c.rows;
  cplx* blocks = c.blocks;
  if (rc) {
    free(rows);
    free(blocks);
    return fail(rc, "tau_solve_shifted: shift is numerically singular"); /* the worker's message */
  }
  if (solve && !full_sweep) {
    for (size_t n = 1; n < (size_t)p->solve_count; ++n) {
      const size_t q = nt - n;
      if (q < (size_t)p->solve_count) continue;
      for (size_t j = 0; j < ns; ++j) blocks[q * ns + j] = conj(blocks[n * ns + j]);
    }
  }
  par_for(ns, pc_inv_cols, &c);
  const double inv_nt = 1.0 / (double)nt;
  double imag_sq = 0.0, total_sq = 0.0;
  for (size_t k = 0; k < nt; ++k) {
    const double s = p->scale_bwd[k] * inv_nt;
    for (size_t j = 0; j < ns; ++j) {
      const cplx z = s * rows[j * nt + k];
      out[k * ns + j] = creal(z);
      imag_sq += cimag(z) * cimag(z);
      total_sq += creal(z) * creal(z) + cimag(z) * cimag(z);
    }
  }
  free(rows);
  free(blocks);
  if (total_sq > 0.0 && sqrt(imag_sq) > 1e-10 * sqrt(total_sq))
    return fail(2, "alpha-circulant action: imaginary residue exceeds 1e-10 of the output norm");
  return 0;
}

int orc_pc_apply(const orc_problem* p, const double* v, double* out, int full_sweep) {
  return pc_action(p, 1, full_sweep, v, out); /* apply_inverse, alpha_circulant.hpp:206-209 */
}
int orc_pc_forward(const orc_problem* p, const double* v, double* out) {
  return pc_action(p, 0, 1, v, out); /* apply_forward, alpha_circulant.hpp:212-215 */
}

/* ---------------------------------------------------------------- GMRES (krylov.hpp:83-192) */

static double dot(const double* a, const double* b, size_t n) { /* krylov.hpp:52-56 */
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double norm2(const double* a, size_t n) { return sqrt(dot(a, a, n)); }
static void axpy(double al, const double* x, double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] += al * x[i];
}

/* One unrestarted gmres_right call (x0 = 0). Returns status; fills x, iterations, etc. */
static int gmres_right(const orc_problem* p, const double* b, double* x, double tol,
                       int max_iter, int full_sweep, int* out_conv, int* out_steps,
                       double* hist, int hist_off, int hist_cap, int* hist_len, double* last_rel) {
  const size_t n = orc_problem_dim(p);
  memset(x, 0, n * sizeof(double));
  *out_conv = 0;
  *out_steps = 0;
  const double norm_b = norm2(b, n);
  if (norm_b == 0.0) {
    *out_conv = 1;
    return 0;
  }
  const int cap = max_iter + 1;
  double** basis = (double**)calloc((size_t)cap, sizeof(double*));
  double** hcols = (double**)calloc((size_t)cap, sizeof(double*));
  double* gc = (double*)calloc((size_t)cap, sizeof(double));
  double* gs = (double*)calloc((size_t)cap, sizeof(double));
  double* g = (double*)calloc((size_t)cap + 1, sizeof(double));
  basis[0] = (double*)malloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) basis[0][i] = b[i] / norm_b;
  g[0] = norm_b;
  double* z = (double*)malloc(n * sizeof(double));
  double* w = (double*)malloc(n * sizeof(double));
  const double reorth = 0.70710678118654752;
  int steps = 0, rc = 0, nb = 1;
  for (int j = 0; j < max_iter; ++j) {
    if ((rc = orc_pc_apply(p, basis[j], z, full_sweep))) break;
    orc_matvec(p, z, w);
    double* h = hcols[j] = (double*)calloc((size_t)j + 2, sizeof(double));
    const double norm_before = norm2(w, n);
    for (int i = 0; i <= j; ++i) {
      const double hij = dot(basis[i], w, n);
      h[i] = hij;
      axpy(-hij, basis[i], w, n);
    }
    double norm_w = norm2(w, n);
    if (norm_w < reorth * norm_before) {
      for (int i = 0; i <= j; ++i) {
        const double c = dot(basis[i], w, n);
        h[i] += c;
        axpy(-c, basis[i], w, n);
      }
      norm_w = norm2(w, n);
    }
    h[j + 1] = norm_w;
    for (int i = 0; i < j; ++i) {
      const double hi = h[i], hi1 = h[i + 1];
      h[i] = gc[i] * hi + gs[i] * hi1;
      h[i + 1] = -gs[i] * hi + gc[i] * hi1;
    }
    const double hj = h[j], hj1 = h[j + 1];
    const double rad = hypot(hj, hj1);
    const double cs = rad > 0.0 ? hj / rad : 1.0;
    const double sn = rad > 0.0 ? hj1 / rad : 0.0;
    gc[j] = cs;
    gs[j] = sn;
    h[j] = rad;
    h[j + 1] = 0.0;
    g[j + 1] = -sn * g[j];
    g[j] *= cs;
    steps = j + 1;
    const double rel = fabs(g[j + 1]) / norm_b;
    if (hist && hist_off + *hist_len < hist_cap) hist[hist_off + *hist_len] = rel;
    ++*hist_len;
    *last_rel = rel;
    if (rel <= tol) {
      *out_conv = 1;
      break;
    }
    if (norm_w <= 1e-14 * fmax(1.0, norm_before)) break;
    basis[j + 1] = (double*)malloc(n * sizeof(double));
    nb = j + 2;
    for (size_t i = 0; i < n; ++i) basis[j + 1][i] = w[i] / norm_w;
  }
  if (!rc) {
    double* y = (double*)calloc((size_t)steps + 1, sizeof(double));
    for (int i = steps - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < steps; ++k) s -= hcols[k][i] * y[k];
      y[i] = s / hcols[i][i];
    }
    double* u = (double*)calloc(n, sizeof(double));
    for (int k = 0; k < steps; ++k) axpy(y[k], basis[k], u, n);
    rc = orc_pc_apply(p, u, x, full_sweep);
    free(u);
    free(y);
  }
  *out_steps = steps;
  for (int i = 0; i < nb; ++i) free(basis[i]);
  for (int i = 0; i < cap; ++i) free(hcols[i]);
  free(basis);
  free(hcols);
  free(gc);
  free(gs);
  free(g);
  free(z);
  free(w);
  return rc;
}

/* GMRES entry. restart <= 0: exactly the reference's unrestarted gmres_right. restart = m > 0:
 * the restart emulation of SURVEY §8(c) built on the unrestarted routine (x0 = 0 each cycle):
 *   r = b; x = 0; loop { d = gmres_right(r, tol*||b||/||r||, min(m, budget)); x += d;
 *                        stop if converged; r = b - A x }.
 * The history records rel residuals w.r.t. ||b|| (the inner ones rescaled by ||r||/||b||). */
int orc_gmres(const orc_problem* p, const double* b, double* x, double tol, int max_iter,
              int restart, int full_sweep, orc_report* rep, double* history, int history_cap) {
  const size_t n = orc_problem_dim(p);
  memset(rep, 0, sizeof *rep);
  int hist_len = 0, rc = 0;
  double last_rel = -1.0;
  const double norm_b = norm2(b, n);
  if (restart <= 0 || restart >= max_iter) {
    int conv = 0, steps = 0;
    rc = gmres_right(p, b, x, tol, max_iter, full_sweep, &conv, &steps, history, 0, history_cap,
                     &hist_len, &last_rel);
    rep->converged = conv;
    rep->iterations = steps;
  } else {
    double* r = (double*)malloc(n * sizeof(double));
    double* d = (double*)malloc(n * sizeof(double));
    double* ax = (double*)malloc(n * sizeof(double));
    memcpy(r, b, n * sizeof(double));
    memset(x, 0, n * sizeof(double));
    int budget = max_iter, total = 0, conv = 0;
    while (budget > 0) {
      const double norm_r = norm2(r, n);
      if (norm_r == 0.0) {
        conv = 1;
        break;
      }
      const int m = restart < budget ? restart : budget;
      int c = 0, steps = 0, hl0 = hist_len;
      rc = gmres_right(p, r, d, tol * norm_b / norm_r, m, full_sweep, &c, &steps, history, 0,
                       history_cap, &hist_len, &last_rel);
      if (rc) break;
      for (int i = hl0; i < hist_len && i < history_cap; ++i)
        history[i] *= norm_r / norm_b;
      if (last_rel >= 0.0) last_rel *= norm_r / norm_b;
      axpy(1.0, d, x, n);
      total += steps;
      budget -= steps;
      if (c) {
        conv = 1;
        break;
      }
      if (steps == 0) break;
      ++rep->restarts;
      orc_matvec(p, x, ax);
      for (size_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
    }
    rep->converged = conv;
    rep->iterations = total;
    free(r);
    free(d);
    free(ax);
  }
  if (rc) return rc;
  rep->history_len = hist_len;
  rep->final_relative_residual = hist_len == 0 ? 1.0 : last_rel;
  if (norm_b == 0.0) {
    rep->true_relative_residual = 0.0;
    rep->final_relative_residual = 0.0;
    return 0;
  }
  /* fresh_relative_residual (krylov.hpp:64-75) */
  double* ax = (double*)malloc(n * sizeof(double));
  orc_matvec(p, x, ax);
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double dd = b[i] - ax[i];
    s += dd * dd;
  }
  free(ax);
  rep->true_relative_residual = sqrt(s) / norm_b;
  return 0;
}

/* ---------------------------------------------------------------- BiCGSTAB (krylov.hpp:204-280) */

/* bicgstab_left: BiCGSTAB on P^{-1} A x = P^{-1} b, x0 = 0, the unpreconditioned residual carried
 * alongside from the same matvec outputs (q = A p, t_orig = A s).  *iterations counts a half-step
 * convergence as k + 0.5 (krylov.hpp:244-249). */
int orc_bicgstab(const orc_problem* p, const double* b, double* x, double tol, int max_iter,
                 int full_sweep, double* iterations, orc_report* rep, double* history,
                 int history_cap) {
  const size_t n = orc_problem_dim(p);
  memset(rep, 0, sizeof *rep);
  memset(x, 0, n * sizeof(double));
  *iterations = 0.0;
  int hl = 0, rc = 0;
  const double norm_b = norm2(b, n); /* :210 */
  if (norm_b == 0.0) {
    rep->converged = 1;
    return 0;
  }
  const double floor_ = 1e-300; /* :215 */
  double* r = (double*)malloc(n * sizeof(double));
  double* rt = (double*)malloc(n * sizeof(double));
  double* rhat = (double*)malloc(n * sizeof(double));
  double* pp = (double*)calloc(n, sizeof(double));
  double* q = (double*)calloc(n, sizeof(double));
  double* v = (double*)calloc(n, sizeof(double));
  double* s = (double*)calloc(n, sizeof(double));
  double* st = (double*)calloc(n, sizeof(double));
  double* to = (double*)calloc(n, sizeof(double));
  double* t = (double*)calloc(n, sizeof(double));
  memcpy(rt, b, n * sizeof(double));
  if ((rc = orc_pc_apply(p, b, r, full_sweep))) goto done; /* :219 */
  memcpy(rhat, r, n * sizeof(double));
  double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
  for (int k = 0; k < max_iter; ++k) {
    const double rho = dot(rhat, r, n); /* :224 */
    if (fabs(rho) < floor_) break;
    if (k == 0) {
      memcpy(pp, r, n * sizeof(double));
    } else {
      const double beta = (rho / rho_prev) * (alpha / omega);
      for (size_t i = 0; i < n; ++i) pp[i] = r[i] + beta * (pp[i] - omega * v[i]);
    }
    orc_matvec(p, pp, q); /* :234-235 */
    if ((rc = orc_pc_apply(p, q, v, full_sweep))) break;
    const double denom = dot(rhat, v, n);
    if (fabs(denom) < floor_) break;
    alpha = rho / denom;
    for (size_t i = 0; i < n; ++i) { /* :239-242 */
      s[i] = r[i] - alpha * v[i];
      st[i] = rt[i] - alpha * q[i];
    }
    const double rel_half = norm2(st, n) / norm_b;
    if (history && hl < history_cap) history[hl] = rel_half;
    ++hl;
    if (rel_half <= tol) { /* :244-250 */
      axpy(alpha, pp, x, n);
      *iterations = k + 0.5;
      rep->converged = 1;
      rep->final_relative_residual = rel_half;
      break;
    }
    orc_matvec(p, s, to); /* :251-252 */
    if ((rc = orc_pc_apply(p, to, t, full_sweep))) break;
    const double tt = dot(t, t, n);
    if (tt < floor_) break;
    omega = dot(t, s, n) / tt;
    for (size_t i = 0; i < n; ++i) { /* :256-260 */
      x[i] += alpha * pp[i] + omega * s[i];
      r[i] = s[i] - omega * t[i];
      rt[i] = st[i] - omega * to[i];
    }
    const double rel = norm2(rt, n) / norm_b;
    if (history && hl < history_cap) history[hl] = rel;
    ++hl;
    *iterations = k + 1.0;
    rep->final_relative_residual = rel;
    if (rel <= tol) {
      rep->converged = 1;
      break;
    }
    if (fabs(omega) < floor_) break;
    rho_prev = rho;
  }
  if (!rc) { /* :274-275 fresh residual */
    orc_matvec(p, x, q);
    for (size_t i = 0; i < n; ++i) q[i] = b[i] - q[i];
    rep->true_relative_residual = norm2(q, n) / norm_b;
  }
done:
  rep->iterations = (int)*iterations;
  rep->history_len = hl;
  free(r); free(rt); free(rhat); free(pp); free(q); free(v); free(s); free(st); free(to); free(t);
  return rc;
}
