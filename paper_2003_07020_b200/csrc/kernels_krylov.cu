// kernels_krylov.cu -- GMRES vector kernels (krylov.hpp:52-62 dot/norm/axpy, 116-131 the
// Gram-Schmidt pass, 166-167 basis append, 180-183 u = V y, 64-75 fresh residual).
//
// All reductions are deterministic: a fixed grid (kDotsGrid CTAs) walks the vector with a fixed
// grid-stride assignment, reduces in-CTA by a fixed shuffle/shared-memory tree, and a single-CTA
// kernel sums the per-CTA partials in index order.  Vectors are 16-byte aligned (double2 loads);
// an odd tail element is handled by CTA 0.
#include <cstdlib>
#include <string>

#include "kernels.cuh"

namespace fpc {

int carveout_pct(size_t dyn_smem, int threads) {
  static const bool maxed = [] {
    const char* e = std::getenv("FPC_CARVEOUT");
    return e && std::string(e) == "max";
  }();
  if (maxed) return 100;
  // CTAs per SM at ~128 registers per thread (16 warps): 64-thread CTAs of the small-grid tilings fit 8
  const int by_regs = threads <= 64 ? 8 : threads <= 128 ? 4 : threads <= 256 ? 2 : 1;
  const size_t per_cta = dyn_smem + 2048;  // + static shared memory and the 1 KB system reserve
  const int by_smem = int((228u * 1024u) / per_cta);
  const int ctas = by_smem < by_regs ? (by_smem > 0 ? by_smem : 1) : by_regs;
  const size_t need = size_t(ctas) * per_cta;
  // The driver takes the smallest capacity >= pct% of 228 KB: rounding the percentage UP overshoots
  // the capacity aimed at (164 KB -> 72% = 164.2 KB -> 196 KB), so round it down (71% = 161.9 KB ->
  // 164 KB).  FPC_CARVE_ROUND=up restores the round-1 behaviour (A/B).
  static const bool round_up = [] {
    const char* e = std::getenv("FPC_CARVE_ROUND");
    return e && e[0] == 'u';
  }();
  static const int caps[] = {0, 8, 16, 32, 64, 100, 132, 164, 196, 228};
  for (int c : caps)
    if (size_t(c) * 1024 >= need) return round_up ? (c * 100 + 227) / 228 : (c * 100) / 228;
  return 100;
}

constexpr int kDotsThreads = 256;
#ifndef FPC_DOTS_GRID
#define FPC_DOTS_GRID (148 * 8)  // B200 config 1: Q1 200 -> 187 us, lincomb 347 -> 281 us vs 148 * 4
#endif
constexpr int kDotsGrid = FPC_DOTS_GRID;
int dots_grid() { return kDotsGrid; }

template <int NACC>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NACC], double* out) {
  __shared__ double red[kDotsThreads / 32][NACC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    double a = acc[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (lane == 0) red[warp][i] = a;
  }
  __syncthreads();
  if (threadIdx.x < NACC) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kDotsThreads / 32; ++w) s += red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// partial[blk*stride + col0 + i] = s_i * <v_i, w>, i < NV;  (+ <w,w> at col0 + NV if NORM)
template <int NV, bool NORM>
__global__ void __launch_bounds__(kDotsThreads)
    k_dots(VecSet vs, const double* __restrict__ w, size_t n, double* __restrict__ partial,
           int stride, int col0) {
  constexpr int NACC = NV + (NORM ? 1 : 0);
  double acc[NACC > 0 ? NACC : 1];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  const size_t n2 = n / 2;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n2;
       e += size_t(kDotsGrid) * kDotsThreads) {
    const double2 wv = w2[e];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 x = reinterpret_cast<const double2*>(vs.v[i])[e];
      acc[i] = fma(x.x, wv.x, acc[i]);
      acc[i] = fma(x.y, wv.y, acc[i]);
    }
    if (NORM) {
      acc[NV] = fma(wv.x, wv.x, acc[NV]);
      acc[NV] = fma(wv.y, wv.y, acc[NV]);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double wl = w[n - 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = fma(vs.v[i][n - 1], wl, acc[i]);
    if (NORM) acc[NV] = fma(wl, wl, acc[NV]);
  }
  double tmp[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) tmp[i] = acc[i];
  __shared__ double outb[NACC];
  block_reduce_store<NACC>(tmp, outb);
  __syncthreads();
  if (threadIdx.x < NACC) {
    const double sc = threadIdx.x < NV ? vs.s[threadIdx.x] : 1.0;
    partial[size_t(blockIdx.x) * stride + col0 + threadIdx.x] = outb[threadIdx.x] * sc;
  }
}

cudaError_t launch_dots(const VecSet& vs, int nv, const double* w, size_t n, double* partial,
                        int stride, int col0, bool with_norm, cudaStream_t st) {
#define DOTS(NVV)                                                                             \
  case NVV:                                                                                   \
    if (with_norm)                                                                            \
      k_dots<NVV, true><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, w, n, partial, stride, col0);  \
    else                                                                                      \
      k_dots<NVV, false><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, w, n, partial, stride, col0); \
    note_launch();                                                                            \
    break;
  switch (nv) {
    case 0:
      k_dots<0, true><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, w, n, partial, stride, col0); note_launch();
      break;
    DOTS(1) DOTS(2) DOTS(3) DOTS(4) DOTS(5) DOTS(6) DOTS(7) DOTS(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef DOTS
  return cudaGetLastError();
}

// One CTA per output: thread t sums partials b = t, t+256, ... in order, then a fixed
// shuffle/smem tree -> the result is independent of scheduling (deterministic).  The thread's
// loads are all issued before the first add (same summation order).  Column of CTA i: i, or for a
// Q1 reduction (nab > 0) the used columns only: a_0..a_{nab-1}, b_0..b_{nab-1}, the three extras.
__global__ void __launch_bounds__(kDotsThreads)
    k_reduce(const double* __restrict__ partial, int stride, int count, double* __restrict__ out,
             int accumulate, int nab) {
  const int i = nab > 0 ? (int(blockIdx.x) < nab       ? int(blockIdx.x)
                           : int(blockIdx.x) < 2 * nab ? kDots2B + int(blockIdx.x) - nab
                                                       : kDots2X + int(blockIdx.x) - 2 * nab)
                        : int(blockIdx.x);
  constexpr int PER = (kDotsGrid + kDotsThreads - 1) / kDotsThreads;
  double x[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int b = int(threadIdx.x) + u * kDotsThreads;
    x[u] = b < kDotsGrid ? partial[size_t(b) * stride + i] : 0.0;
  }
  double acc[1] = {0.0};
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (int(threadIdx.x) + u * kDotsThreads < kDotsGrid) acc[0] += x[u];
  __shared__ double outb[1];
  block_reduce_store<1>(acc, outb);
  __syncthreads();
  if (threadIdx.x == 0) out[i] = accumulate ? out[i] + outb[0] : outb[0];
}

cudaError_t launch_reduce(const double* partial, int stride, int count, double* out,
                          bool accumulate, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  k_reduce<<<count, kDotsThreads, 0, st>>>(partial, stride, count, out, accumulate ? 1 : 0, 0); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_reduce_dots2(const double* partial, int stride, int nab, double* out, cudaStream_t st) {
  if (nab <= 0 || nab > kDots2B) return cudaErrorInvalidValue;
  k_reduce<<<2 * nab + 3, kDotsThreads, 0, st>>>(partial, stride, 2 * nab + 3, out, 0, nab); note_launch();
  return cudaGetLastError();
}

constexpr int kMaxVecs = 256;

// w <- w - sum_i (coef_i * s_i) v_i (in order i = 0..nv-1, as the reference's sequential
// axpys); partial[blk] = sum w_new^2.
__global__ void __launch_bounds__(kDotsThreads)
    k_update(const double* const* __restrict__ vptr, const double* __restrict__ scales,
             const double* __restrict__ coef, int nv, double* __restrict__ w, size_t n,
             double* __restrict__ partial) {
  __shared__ const double2* sp[kMaxVecs];
  __shared__ double sc[kMaxVecs];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    sp[i] = reinterpret_cast<const double2*>(vptr[i]);
    sc[i] = coef[i] * scales[i];
  }
  __syncthreads();
  double acc[1] = {0.0};
  const size_t n2 = n / 2;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n2;
       e += size_t(kDotsGrid) * kDotsThreads) {
    double2 a = w2[e];
    for (int i = 0; i < nv; ++i) {
      const double2 x = sp[i][e];
      a.x = fma(-sc[i], x.x, a.x);
      a.y = fma(-sc[i], x.y, a.y);
    }
    w2[e] = a;
    acc[0] = fma(a.x, a.x, acc[0]);
    acc[0] = fma(a.y, a.y, acc[0]);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double a = w[n - 1];
    for (int i = 0; i < nv; ++i) a = fma(-sc[i], reinterpret_cast<const double*>(sp[i])[n - 1], a);
    w[n - 1] = a;
    acc[0] = fma(a, a, acc[0]);
  }
  __shared__ double outb[1];
  block_reduce_store<1>(acc, outb);
  __syncthreads();
  if (threadIdx.x == 0) partial[blockIdx.x] = outb[0];
}

cudaError_t launch_update(const double* const* vptr, const double* scales, const double* coef,
                          int nv, double* w, size_t n, double* partial, cudaStream_t st) {
  if (nv > kMaxVecs) return cudaErrorInvalidValue;
  k_update<<<kDotsGrid, kDotsThreads, 0, st>>>(vptr, scales, coef, nv, w, n, partial); note_launch();
  return cudaGetLastError();
}

// u = sum_i (coef_i s_i) v_i, accumulated in order from u = 0 (krylov.hpp:180-182)
__global__ void __launch_bounds__(kDotsThreads)
    k_lincomb(const double* const* __restrict__ vptr, const double* __restrict__ scales,
              const double* __restrict__ coef, int nv, double* __restrict__ u, size_t n) {
  __shared__ const double* sp[kMaxVecs];
  __shared__ double sc[kMaxVecs];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    sp[i] = vptr[i];
    sc[i] = coef[i] * scales[i];
  }
  __syncthreads();
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n;
       e += size_t(kDotsGrid) * kDotsThreads) {
    double a = 0.0;
    for (int i = 0; i < nv; ++i) a = fma(sc[i], sp[i][e], a);
    u[e] = a;
  }
}

cudaError_t launch_lincomb(const double* const* vptr, const double* scales, const double* coef,
                           int nv, double* u, size_t n, cudaStream_t st) {
  if (nv > kMaxVecs) return cudaErrorInvalidValue;
  k_lincomb<<<kDotsGrid, kDotsThreads, 0, st>>>(vptr, scales, coef, nv, u, n); note_launch();
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kDotsThreads)
    k_resid_norm(const double* __restrict__ b, const double* __restrict__ y, size_t n,
                 double* __restrict__ partial) {
  double acc[1] = {0.0};
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n;
       e += size_t(kDotsGrid) * kDotsThreads) {
    const double d = b[e] - y[e];
    acc[0] = fma(d, d, acc[0]);
  }
  __shared__ double outb[1];
  block_reduce_store<1>(acc, outb);
  __syncthreads();
  if (threadIdx.x == 0) partial[blockIdx.x] = outb[0];
}

cudaError_t launch_resid_norm(const double* b, const double* y, size_t n, double* partial,
                              cudaStream_t st) {
  k_resid_norm<<<kDotsGrid, kDotsThreads, 0, st>>>(b, y, n, partial); note_launch();
  return cudaGetLastError();
}

__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, size_t n) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += size_t(gridDim.x) * blockDim.x)
    y[e] += a * x[e];
}
cudaError_t launch_axpy(double a, const double* x, double* y, size_t n, cudaStream_t st) {
  k_axpy<<<kDotsGrid, kDotsThreads, 0, st>>>(a, x, y, n); note_launch();
  return cudaGetLastError();
}

__global__ void k_rsub(const double* __restrict__ b, double* __restrict__ y, size_t n) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += size_t(gridDim.x) * blockDim.x)
    y[e] = b[e] - y[e];
}
cudaError_t launch_rsub(const double* b, double* y, size_t n, cudaStream_t st) {
  k_rsub<<<kDotsGrid, kDotsThreads, 0, st>>>(b, y, n); note_launch();
  return cudaGetLastError();
}

}  // namespace fpc

namespace fpc {

// Fused Gram-Schmidt step: w' = w - sum_i (coef_i s_i) v_i (sequential order, as the reference's
// axpys, krylov.hpp:116-121), and in the same pass the re-orthogonalisation dots
// partial[i] = s_i <v_i, w'> plus ||w'||^2 (krylov.hpp:122-130).  One read of the basis instead of
// two when the reference's reorthogonalisation test fires.
template <int NV>
__global__ void __launch_bounds__(kDotsThreads)
    k_update_dots(VecSetN vs, const double* __restrict__ coef, double* __restrict__ w, size_t n,
                  double* __restrict__ partial, int stride) {
  double c[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) c[i] = coef[i] * vs.s[i];
  double acc[NV + 1];
#pragma unroll
  for (int i = 0; i <= NV; ++i) acc[i] = 0.0;
  const size_t n2 = n / 2;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n2;
       e += size_t(kDotsGrid) * kDotsThreads) {
    double2 x[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) x[i] = reinterpret_cast<const double2*>(vs.v[i])[e];
    double2 a = w2[e];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      a.x = fma(-c[i], x[i].x, a.x);
      a.y = fma(-c[i], x[i].y, a.y);
    }
    w2[e] = a;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      acc[i] = fma(x[i].x, a.x, acc[i]);
      acc[i] = fma(x[i].y, a.y, acc[i]);
    }
    acc[NV] = fma(a.x, a.x, acc[NV]);
    acc[NV] = fma(a.y, a.y, acc[NV]);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double a = w[n - 1];
    double xl[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      xl[i] = vs.v[i][n - 1];
      a = fma(-c[i], xl[i], a);
    }
    w[n - 1] = a;
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = fma(xl[i], a, acc[i]);
    acc[NV] = fma(a, a, acc[NV]);
  }
  __shared__ double outb[NV + 1];
  block_reduce_store<NV + 1>(acc, outb);
  __syncthreads();
  if (threadIdx.x <= NV) {
    const double sc = threadIdx.x < NV ? vs.s[threadIdx.x] : 1.0;
    partial[size_t(blockIdx.x) * stride + threadIdx.x] = outb[threadIdx.x] * sc;
  }
}

cudaError_t launch_update_dots(const VecSetN& vs, int nv, const double* coef, double* w, size_t n,
                               double* partial, int stride, cudaStream_t st) {
  switch (nv) {
#define UD(NVV) \
  case NVV: k_update_dots<NVV><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, coef, w, n, partial, stride); note_launch(); break;
    UD(1) UD(2) UD(3) UD(4) UD(5) UD(6) UD(7) UD(8) UD(9) UD(10) UD(11) UD(12)
    UD(13) UD(14) UD(15) UD(16) UD(17) UD(18) UD(19) UD(20) UD(21) UD(22) UD(23) UD(24)
#undef UD
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace fpc

// ---------------------------------------------------------------------------------------------
// BiCGSTAB vector kernels (krylov.hpp:204-280, bicgstab_left).  Elementwise, so the in-place
// aliasing below (s over r, s_true over r_true, t_orig over q) keeps the reference's values.
namespace fpc {

// p = r (first) or p = r + beta (p - omega v)                                 krylov.hpp:228-233
__global__ void __launch_bounds__(kDotsThreads)
    k_bicg_p(const double* __restrict__ r, const double* __restrict__ v, double* __restrict__ p,
             double beta, double omega, size_t n, int first) {
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n;
       e += size_t(kDotsGrid) * kDotsThreads)
    p[e] = first ? r[e] : r[e] + beta * (p[e] - omega * v[e]);
}

// alpha = rho / denom (device scalars); s = r - alpha v (into r); s_true = r_true - alpha q (into
// r_true); partial[blk] = ||s_true||^2                                          krylov.hpp:236-243
__global__ void __launch_bounds__(kDotsThreads)
    k_bicg_s(double* __restrict__ r, double* __restrict__ rt, const double* __restrict__ v,
             const double* __restrict__ q, const double* __restrict__ rho_denom, size_t n,
             double* __restrict__ partial) {
  const double alpha = rho_denom[0] / rho_denom[1];
  double acc[1] = {0.0};
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n;
       e += size_t(kDotsGrid) * kDotsThreads) {
    r[e] = r[e] - alpha * v[e];
    const double st = rt[e] - alpha * q[e];
    rt[e] = st;
    acc[0] = fma(st, st, acc[0]);
  }
  __shared__ double outb[1];
  block_reduce_store<1>(acc, outb);
  __syncthreads();
  if (threadIdx.x == 0) partial[blockIdx.x] = outb[0];
}

// x += alpha p + omega s; r = s - omega t (s lives in r); r_true = s_true - omega t_orig;
// partial[blk*2 + 0] = ||r_true||^2, partial[blk*2 + 1] = <rhat, r> (the next rho)  :253-259, 221
__global__ void __launch_bounds__(kDotsThreads)
    k_bicg_x(double* __restrict__ x, const double* __restrict__ p, double* __restrict__ r,
             const double* __restrict__ t, double* __restrict__ rt, const double* __restrict__ to,
             const double* __restrict__ rhat, double alpha, double omega, size_t n,
             double* __restrict__ partial) {
  double acc[2] = {0.0, 0.0};
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n;
       e += size_t(kDotsGrid) * kDotsThreads) {
    const double s = r[e];
    x[e] += alpha * p[e] + omega * s;
    const double rn = s - omega * t[e];
    r[e] = rn;
    const double rtn = rt[e] - omega * to[e];
    rt[e] = rtn;
    acc[0] = fma(rtn, rtn, acc[0]);
    acc[1] = fma(rhat[e], rn, acc[1]);
  }
  __shared__ double outb[2];
  block_reduce_store<2>(acc, outb);
  __syncthreads();
  if (threadIdx.x < 2) partial[size_t(blockIdx.x) * 2 + threadIdx.x] = outb[threadIdx.x];
}

cudaError_t launch_bicg_p(const double* r, const double* v, double* p, double beta, double omega,
                          size_t n, bool first, cudaStream_t st) {
  k_bicg_p<<<kDotsGrid, kDotsThreads, 0, st>>>(r, v, p, beta, omega, n, first ? 1 : 0); note_launch();
  return cudaGetLastError();
}
cudaError_t launch_bicg_s(double* r, double* rt, const double* v, const double* q,
                          const double* rho_denom, size_t n, double* partial, cudaStream_t st) {
  k_bicg_s<<<kDotsGrid, kDotsThreads, 0, st>>>(r, rt, v, q, rho_denom, n, partial); note_launch();
  return cudaGetLastError();
}
cudaError_t launch_bicg_x(double* x, const double* p, double* r, const double* t, double* rt,
                          const double* to, const double* rhat, double alpha, double omega,
                          size_t n, double* partial, cudaStream_t st) {
  k_bicg_x<<<kDotsGrid, kDotsThreads, 0, st>>>(x, p, r, t, rt, to, rhat, alpha, omega, n, partial); note_launch();
  return cudaGetLastError();
}

}  // namespace fpc

// ---------------------------------------------------------------------------------------------
// Delayed re-orthogonalisation Gram-Schmidt (two basis passes per Arnoldi step; api.cu
// gmres_inner_lagged).  Q1 = k_dots2: a_i = s_i <v_i, U>, b_i = s_i <v_i, W> (+ <U,W>, <U,U>,
// <W,W>).  Q2 = k_update2: U' = U - sum ca_i v_i, W' = cw W + cu U + sum cd_i v_i, ||W'||^2.
namespace fpc {

// partial[blk*stride + col0 + i] = a_i, [.. + kDots2B + col0 + i] = b_i, [.. + kDots2X + 0..2] =
// <U,W>, <U,U>, <W,W> (EXTRA only)
template <int NV, bool EXTRA>
__global__ void __launch_bounds__(kDotsThreads)
    k_dots2(VecSet16 vs, const double* __restrict__ U, const double* __restrict__ W, size_t n,
            double* __restrict__ partial, int stride, int col0) {
  constexpr int NACC = 2 * NV + (EXTRA ? 3 : 0);
  double acc[NACC > 0 ? NACC : 1];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  const size_t n2 = n / 2;
  const double2* u2 = reinterpret_cast<const double2*>(U);
  const double2* w2 = reinterpret_cast<const double2*>(W);
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n2;
       e += size_t(kDotsGrid) * kDotsThreads) {
    const double2 uv = u2[e], wv = w2[e];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 x = reinterpret_cast<const double2*>(vs.v[i])[e];
      acc[i] = fma(x.x, uv.x, acc[i]);
      acc[i] = fma(x.y, uv.y, acc[i]);
      acc[NV + i] = fma(x.x, wv.x, acc[NV + i]);
      acc[NV + i] = fma(x.y, wv.y, acc[NV + i]);
    }
    if (EXTRA) {
      acc[2 * NV] = fma(uv.x, wv.x, acc[2 * NV]);
      acc[2 * NV] = fma(uv.y, wv.y, acc[2 * NV]);
      acc[2 * NV + 1] = fma(uv.x, uv.x, acc[2 * NV + 1]);
      acc[2 * NV + 1] = fma(uv.y, uv.y, acc[2 * NV + 1]);
      acc[2 * NV + 2] = fma(wv.x, wv.x, acc[2 * NV + 2]);
      acc[2 * NV + 2] = fma(wv.y, wv.y, acc[2 * NV + 2]);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double ul = U[n - 1], wl = W[n - 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double x = vs.v[i][n - 1];
      acc[i] = fma(x, ul, acc[i]);
      acc[NV + i] = fma(x, wl, acc[NV + i]);
    }
    if (EXTRA) {
      acc[2 * NV] = fma(ul, wl, acc[2 * NV]);
      acc[2 * NV + 1] = fma(ul, ul, acc[2 * NV + 1]);
      acc[2 * NV + 2] = fma(wl, wl, acc[2 * NV + 2]);
    }
  }
  __shared__ double outb[NACC > 0 ? NACC : 1];
  block_reduce_store<NACC>(acc, outb);
  __syncthreads();
  for (int t = threadIdx.x; t < NACC; t += kDotsThreads) {
    double* prow = partial + size_t(blockIdx.x) * stride;
    if (t < NV)
      prow[col0 + t] = outb[t] * vs.s[t];
    else if (t < 2 * NV)
      prow[kDots2B + col0 + (t - NV)] = outb[t] * vs.s[t - NV];
    else
      prow[kDots2X + (t - 2 * NV)] = outb[t];
  }
}

cudaError_t launch_dots2(const VecSet16& vs, int nv, const double* U, const double* W, size_t n,
                         double* partial, int stride, int col0, bool extra, cudaStream_t st) {
#define D2(NVV)                                                                                      \
  case NVV:                                                                                          \
    if (extra)                                                                                       \
      { k_dots2<NVV, true><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, U, W, n, partial, stride, col0); note_launch(); }    \
    else                                                                                             \
      { k_dots2<NVV, false><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, U, W, n, partial, stride, col0); note_launch(); }   \
    break;
  switch (nv) {
    case 0:
      k_dots2<0, true><<<kDotsGrid, kDotsThreads, 0, st>>>(vs, U, W, n, partial, stride, col0); note_launch();
      break;
    D2(1) D2(2) D2(3) D2(4) D2(5) D2(6) D2(7) D2(8)
    D2(9) D2(10) D2(11) D2(12) D2(13) D2(14) D2(15) D2(16)
    default:
      return cudaErrorInvalidValue;
  }
#undef D2
  return cudaGetLastError();
}

// U <- U - sum_i ca_i v_i ; W <- cw W + cu U_old + sum_i cd_i v_i  (coefficients already carry the
// basis scales); NORM: partial[blk] = ||W_new||^2.  FIRST: the cw/cu terms are applied (a later
// group of basis vectors only adds its sums in place).
// KEEPU: U is left as stored (the re-orthogonalisation of the previous vector is carried in the
// host's basis-transformation matrix instead, api.cu gmres_inner_lagged): no U update, no U write,
// and no U read at all in the later groups.
template <int NV, bool FIRST, bool NORM, bool KEEPU>
__global__ void __launch_bounds__(kDotsThreads)
    k_update2(Update2Args a, double* __restrict__ U, double* __restrict__ W, size_t n,
              double* __restrict__ partial) {
  double acc[1] = {0.0};
  const size_t n2 = n / 2;
  double2* u2 = reinterpret_cast<double2*>(U);
  double2* w2 = reinterpret_cast<double2*>(W);
  for (size_t e = size_t(blockIdx.x) * kDotsThreads + threadIdx.x; e < n2;
       e += size_t(kDotsGrid) * kDotsThreads) {
    const double2 wv = w2[e];
    double2 uv = make_double2(0.0, 0.0);
    if (FIRST || !KEEPU) uv = u2[e];
    double2 nu = uv, nw;
    if (FIRST) {
      nw.x = fma(a.cw, wv.x, a.cu * uv.x);
      nw.y = fma(a.cw, wv.y, a.cu * uv.y);
    } else {
      nw = wv;
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double2 x = reinterpret_cast<const double2*>(a.v[i])[e];
      if (!KEEPU) {
        nu.x = fma(-a.ca[i], x.x, nu.x);
        nu.y = fma(-a.ca[i], x.y, nu.y);
      }
      nw.x = fma(a.cd[i], x.x, nw.x);
      nw.y = fma(a.cd[i], x.y, nw.y);
    }
    if (!KEEPU) u2[e] = nu;
    w2[e] = nw;
    if (NORM) {
      acc[0] = fma(nw.x, nw.x, acc[0]);
      acc[0] = fma(nw.y, nw.y, acc[0]);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double ul = U[n - 1], wl = W[n - 1];
    double nu = ul, nw = FIRST ? fma(a.cw, wl, a.cu * ul) : wl;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const double x = a.v[i][n - 1];
      nu = fma(-a.ca[i], x, nu);
      nw = fma(a.cd[i], x, nw);
    }
    if (!KEEPU) U[n - 1] = nu;
    W[n - 1] = nw;
    if (NORM) acc[0] = fma(nw, nw, acc[0]);
  }
  if (NORM) {
    __shared__ double outb[1];
    block_reduce_store<1>(acc, outb);
    __syncthreads();
    if (threadIdx.x == 0) partial[blockIdx.x] = outb[0];
  }
}

cudaError_t launch_update2(const Update2Args& a, int nv, bool first, bool norm, double* U, double* W,
                           size_t n, double* partial, cudaStream_t st, bool keep_u) {
#define U2K(NVV, F, NRM)                                                                               \
  {                                                                                                    \
    if (keep_u)                                                                                        \
      k_update2<NVV, F, NRM, true><<<kDotsGrid, kDotsThreads, 0, st>>>(a, U, W, n, partial);           \
    else                                                                                               \
      k_update2<NVV, F, NRM, false><<<kDotsGrid, kDotsThreads, 0, st>>>(a, U, W, n, partial);          \
    note_launch();                                                                                     \
  }
#define U2(NVV)                                                                                        \
  case NVV:                                                                                            \
    if (first && norm)                                                                                 \
      U2K(NVV, true, true)                                                                             \
    else if (first)                                                                                    \
      U2K(NVV, true, false)                                                                            \
    else if (norm)                                                                                     \
      U2K(NVV, false, true)                                                                            \
    else                                                                                               \
      U2K(NVV, false, false)                                                                           \
    break;
  switch (nv) {
    U2(0) U2(1) U2(2) U2(3) U2(4) U2(5) U2(6) U2(7) U2(8) U2(9) U2(10) U2(11) U2(12)
    U2(13) U2(14) U2(15) U2(16) U2(17) U2(18) U2(19) U2(20) U2(21) U2(22) U2(23) U2(24)
    default:
      return cudaErrorInvalidValue;
  }
#undef U2K
#undef U2
  return cudaGetLastError();
}

}  // namespace fpc
