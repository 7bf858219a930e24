// kernels_tsplit.cu -- the preconditioner's time FFTs (alpha_circulant.hpp:146-198) for
// Nt = 1024 / 2048 on 2-CTA clusters, split by time parity.
//
// A column tile is B = 8 spatial columns (64-byte row segments, the DRAM unit the 1-CTA kernels
// were tuned to) of the packed series x_m = r_{2m} + i r_{2m+1}, m < M = Nt/2.  The 1-CTA kernels
// (kernels_1d.cu K2/K4, kernels_commuted.cu) hold the whole tile (8 x M complex, 136 KB at
// Nt = 2048) in one 512-thread CTA per SM, so their strided load phase never overlaps FFT work.
// Here the M-point transform is split by decimation in time (forward) / in frequency (inverse):
//   forward:  rank q transforms x_{2m'+q} (time rows = 2q, 2q+1 mod 4: the two ranks read disjoint
//             rows, every row once):  E = FFT_H(x_even), O = FFT_H(x_odd), H = M/2, and
//             X_k = E_{k mod H} + w^k O_{k mod H},  w = e^{+2 pi i/M};
//   spectrum: the Hermitian post-processing pairs bins (n, M-n); bins n, H+n, H-n, M-n are all built
//             from slots n and H-n of E and O, so one task per slot pair (n, H-n) reads and writes
//             only those slots of both ranks' buffers (DSMEM; no task touches another's slots);
//   inverse:  x_{2m'} = IFFT_H(U), x_{2m'+1} = IFFT_H(V), U_k = Y_k + Y_{k+H},
//             V_k = (Y_k - Y_{k+H}) conj(w^k): each rank inverts its own buffer and writes its own
//             time rows.
// Half the shared memory per CTA (68 KB) and half the threads (256), so two CTAs share an SM and one
// CTA's loads overlap the other's transforms.  Same formulas as K2/K4 (rounding-level differences
// from the different FFT factorisation only).
#include <cooperative_groups.h>

#include <cstdint>

#include "fft_block.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fpc {

__host__ __device__ constexpr int skewed_s(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}

template <int LOGH>
struct SGeo {
  static constexpr int H = 1 << LOGH, M = 2 * H, NTIME = 2 * M, B = 8, E = 16;
  static constexpr int NT = B * H / E;
  static constexpr int BS = skewed_s(H);
  static constexpr size_t SMEM = size_t(B) * BS * sizeof(double2);
  static constexpr int NTASK = B * (H / 2 + 1);  // (column, n) with n = 0..H/2
};

// rank q's time row of packed-slot element kk (kk = 2 m' + part)
template <int LOGH>
__device__ __forceinline__ int split_row(int kk, int q) {
  return ((kk >> 1) << 2) + 2 * q + (kk & 1);
}

template <int LOGH>
__device__ __forceinline__ void split_prefetch(const double* u, int ns, int p0, int q) {
  using G = SGeo<LOGH>;
  for (int r = threadIdx.x; r < G::M; r += G::NT) {  // rows 2q, 2q+1 mod 4: 2 of every 4
    const int row = ((r >> 1) << 2) + 2 * q + (r & 1);
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(u + size_t(row) * ns + p0);
    const uintptr_t l0 = a0 & ~uintptr_t(127), l1 = (a0 + uintptr_t(G::B * 8) - 1) & ~uintptr_t(127);
    for (uintptr_t l = l0; l <= l1; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
  }
}

// forward: E (q = 0) or O (q = 1) of the B columns, in smem
template <int LOGH>
__device__ __forceinline__ void split_forward(double2* smem, const double* __restrict__ u, int ns, int p0, int q,
                                              const double* __restrict__ sf, double s_in,
                                              const double2* __restrict__ twb) {
  using G = SGeo<LOGH>;
  block_fft_columns_from<LOGH, 1, G::B, G::BS, G::E>(smem, twb + G::H, [&](int c, int kk) {
    const int p = p0 + c;
    const int row = split_row<LOGH>(kk, q);
    return p < ns ? __ldg(sf + row) * (s_in * u[size_t(row) * ns + p]) : 0.0;
  });
}

// The four spectrum bins of slot pair (n, H-n) from E and O (n >= 1):
//   X_n = E_n + w^n O_n, X_{H+n} = E_n - w^n O_n, X_{H-n} = E_{H-n} + w^{H-n} O_{H-n},
//   X_{M-n} = E_{H-n} - w^{H-n} O_{H-n};  w^{H-n} = -conj(w^n) exactly.
struct Bins4 {
  double2 xn, xhpn, xhmn, xmmn;
};
__device__ __forceinline__ Bins4 split_bins(double2 En, double2 On, double2 E2, double2 O2, double2 wn) {
  const double2 t1 = cmul(wn, On);
  const double2 w2 = make_double2(-wn.x, wn.y);  // -conj(wn)
  const double2 t2 = cmul(w2, O2);
  return {cadd(En, t1), csub(En, t1), cadd(E2, t2), csub(E2, t2)};
}

// K2 post-processing of bins (a = X_n, bq = X_{M-n}), n >= 1 (kernels_1d.cu k_time_fwd):
// Z_n = (P - i w Q)/2, Z_{M-n} = conj(P + i w Q)/2, w = e^{+2 pi i n/Nt} = conj(wc)
__device__ __forceinline__ void half_spectrum(double2 a, double2 bq, double2 wc, double2& zn, double2& zmn) {
  const double2 w = cconj(wc);
  const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
  const double2 iwQ = mul_si<1>(cmul(w, Q));
  zn = cscale(csub(P, iwQ), 0.5);
  zmn = cscale(cconj(cadd(P, iwQ)), 0.5);
}
// K4 pre-processing (kernels_1d.cu k_time_inv): slots n and M-n of the inverse input from the
// solved bins ya = Y~_n, yb = Y~_{M-n}
__device__ __forceinline__ void inverse_input(double2 ya, double2 yb, double2 wc, double2& sn, double2& smn) {
  const double2 A = cadd(ya, cconj(yb));
  const double2 Bn = cmul(csub(ya, cconj(yb)), wc);
  sn = cadd(A, mul_si<1>(Bn));
  smn = cadd(cconj(A), mul_si<1>(cconj(Bn)));
}

// U_k = Y_k + Y_{k+H}, V_k = (Y_k - Y_{k+H}) conj(w^k)
__device__ __forceinline__ void uv(double2 yk, double2 ykh, double2 wk, double2& U, double2& V) {
  U = cadd(yk, ykh);
  V = cmul(csub(yk, ykh), cconj(wk));
}

// inverse of the own buffer and the rows of rank q: z[row][p] = sb[row]/Nt * x_row
template <int LOGH>
__device__ __forceinline__ void split_inverse_store(double2* smem, double* __restrict__ z, int ns, int p0, int q,
                                                    const double* __restrict__ sb,
                                                    const double2* __restrict__ twb) {
  using G = SGeo<LOGH>;
  block_fft<LOGH, -1, G::BS, G::E>(smem, twb + G::H, G::B);
  const double inv_nt = 1.0 / double(G::NTIME);
  for (int e = threadIdx.x; e < G::B * G::M; e += G::NT) {
    const int c = e % G::B, kk = e / G::B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const int row = split_row<LOGH>(kk, q);
    const double val = reinterpret_cast<const double*>(smem + c * G::BS + pad16(kk >> 1))[kk & 1];
    z[size_t(row) * ns + p] = (__ldg(sb + row) * inv_nt) * val;
  }
}

// ---------------------------------------------------------------------------------------------
// K2 split: Z[n][p], n = 0..M (half spectrum, alpha_circulant.hpp:146-156)
// ---------------------------------------------------------------------------------------------
template <int LOGH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SGeo<LOGH>::NT, SGeo<LOGH>::NT <= 128 ? 4 : SGeo<LOGH>::NT <= 256 ? 2 : 1)
    k_time_fwd_split(const double* __restrict__ v, double2* __restrict__ Z, int ns, const double* __restrict__ sf,
                     double s_in, const double2* __restrict__ twb) {
  using G = SGeo<LOGH>;
  constexpr int H = G::H, M = G::M, B = G::B, BS = G::BS;
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const int p0 = int(blockIdx.x >> 1) * B;
  split_prefetch<LOGH>(v, ns, p0, q);
  split_forward<LOGH>(smem, v, ns, p0, q, sf, s_in, twb);
  cluster.sync();
  const double2* Eb = cluster.map_shared_rank(smem, 0);
  const double2* Ob = cluster.map_shared_rank(smem, 1);
  const double2* twM = twb + M;      // e^{-2 pi i t/M}
  const double2* twT = twb + 2 * M;  // e^{-2 pi i t/Nt}
  constexpr int HALF = (G::NTASK + 1) / 2;
  const int t1 = q == 0 ? HALF : G::NTASK;
  for (int t = q * HALF + int(threadIdx.x); t < t1; t += G::NT) {
    const int c = t % B, n = t / B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const double2 En = Eb[c * BS + pad16(n)], On = Ob[c * BS + pad16(n)];
    if (n == 0) {
      const double2 x0 = cadd(En, On), xh = csub(En, On);  // X_0, X_H
      Z[p] = make_double2(x0.x + x0.y, 0.0);
      Z[size_t(M) * ns + p] = make_double2(x0.x - x0.y, 0.0);
      double2 zh, zh2;
      half_spectrum(xh, xh, __ldg(twT + H), zh, zh2);  // n = M/2 = H: its own mirror
      Z[size_t(H) * ns + p] = zh;
      continue;
    }
    const int n2 = H - n;
    const double2 E2 = Eb[c * BS + pad16(n2)], O2 = Ob[c * BS + pad16(n2)];
    const Bins4 X = split_bins(En, On, E2, O2, cconj(__ldg(twM + n)));
    const double2 wc = __ldg(twT + n);
    double2 zn, zmn;
    half_spectrum(X.xn, X.xmmn, wc, zn, zmn);  // bins n, M-n
    Z[size_t(n) * ns + p] = zn;
    Z[size_t(M - n) * ns + p] = zmn;
    if (n2 != n) {
      const double2 wc2 = make_double2(-wc.y, -wc.x);  // e^{-2 pi i (H-n)/Nt} = -i conj(wc)
      double2 z2, zm2;
      half_spectrum(X.xhmn, X.xhpn, wc2, z2, zm2);  // bins H-n, M-(H-n) = H+n
      Z[size_t(n2) * ns + p] = z2;
      Z[size_t(H + n) * ns + p] = zm2;
    }
  }
  cluster_sync_exit(cluster);  // the partner's buffer stays alive until every read of it is done
}

// ---------------------------------------------------------------------------------------------
// K4 split: z from Z[n][p], n = 0..M (alpha_circulant.hpp:167-198)
// ---------------------------------------------------------------------------------------------
template <int LOGH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SGeo<LOGH>::NT, SGeo<LOGH>::NT <= 128 ? 4 : SGeo<LOGH>::NT <= 256 ? 2 : 1)
    k_time_inv_split(const double2* __restrict__ Z, double* __restrict__ z, int ns, const double* __restrict__ sb,
                     const double2* __restrict__ twb) {
  using G = SGeo<LOGH>;
  constexpr int H = G::H, M = G::M, B = G::B, BS = G::BS;
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const int p0 = int(blockIdx.x >> 1) * B;
  double2* Ub = cluster.map_shared_rank(smem, 0);
  double2* Vb = cluster.map_shared_rank(smem, 1);
  const double2* twM = twb + M;
  const double2* twT = twb + 2 * M;
  constexpr int HALF = (G::NTASK + 1) / 2;
  const int t1 = q == 0 ? HALF : G::NTASK;
  {  // L2 prefetch of the four Z rows (n, M-n, H-n, H+n) of every task of this rank, 128-byte segments
    const int n0 = (q * HALF) / B, n1 = (t1 - 1) / B;
    for (int r = threadIdx.x; r < 4 * (n1 - n0 + 1); r += G::NT) {
      const int n = n0 + (r >> 2), w = r & 3;
      const int row = w == 0 ? n : w == 1 ? M - n : w == 2 ? H - n : H + n;
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(Z + size_t(row) * ns + p0);
      const uintptr_t l0 = a0 & ~uintptr_t(127), l1 = (a0 + uintptr_t(B * 16) - 1) & ~uintptr_t(127);
      for (uintptr_t l = l0; l <= l1; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
    }
  }
  cluster_sync_relaxed(cluster);  // the partner has started (its shared memory is ours to write)
#ifndef FPC_TSPLIT_UI
#define FPC_TSPLIT_UI 2
#endif
  constexpr int UI = FPC_TSPLIT_UI;
  for (int t0 = q * HALF + int(threadIdx.x); t0 < t1; t0 += UI * G::NT) {
    double2 a[UI], am[UI], b[UI], bm[UI];
#pragma unroll
    for (int u = 0; u < UI; ++u) {  // the four rows' loads of UI tasks in flight together
      const int t = t0 + u * G::NT;
      const int c = t % B, n = t / B, p = p0 + c;
      const bool ok = t < t1 && p < ns;
      const int n2 = n == 0 ? H : H - n;
      a[u] = ok ? Z[size_t(n) * ns + p] : make_double2(0.0, 0.0);
      am[u] = ok ? Z[size_t(M - n) * ns + p] : make_double2(0.0, 0.0);
      b[u] = ok && n != 0 ? Z[size_t(n2) * ns + p] : make_double2(0.0, 0.0);
      bm[u] = ok ? Z[size_t(M - n2) * ns + p] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < UI; ++u) {
      const int t = t0 + u * G::NT;
      if (t >= t1) continue;
      const int c = t % B, n = t / B;
      double2* U = Ub + c * BS;
      double2* V = Vb + c * BS;
      if (n == 0) {
        // slot 0 of the inverse input from Z_0, Z_M (K4's n = 0); slot H from Z_H (own mirror)
        const double2 A = cadd(a[u], am[u]), Bv = csub(a[u], am[u]);
        const double2 y0 = cadd(A, mul_si<1>(Bv));
        double2 yh, yh2;
        inverse_input(bm[u], bm[u], __ldg(twT + H), yh, yh2);
        double2 U0, V0;
        uv(y0, yh, make_double2(1.0, 0.0), U0, V0);
        U[0] = U0;
        V[0] = V0;
        continue;
      }
      const int n2 = H - n;
      const double2 wc = __ldg(twT + n);
      double2 yn, ymn;
      inverse_input(a[u], am[u], wc, yn, ymn);  // slots n, M-n
      const double2 wn = cconj(__ldg(twM + n));  // w^n = e^{+2 pi i n/M}
      if (n2 == n) {  // n = H/2: M - n = H + n
        double2 Un, Vn;
        uv(yn, ymn, wn, Un, Vn);
        U[pad16(n)] = Un;
        V[pad16(n)] = Vn;
        continue;
      }
      const double2 wc2 = make_double2(-wc.y, -wc.x);
      double2 y2, yhpn;
      inverse_input(b[u], bm[u], wc2, y2, yhpn);  // slots H-n, M-(H-n) = H+n
      double2 Un, Vn, U2, V2;
      uv(yn, yhpn, wn, Un, Vn);                              // k = n:   Y_n, Y_{n+H}
      uv(y2, ymn, make_double2(-wn.x, wn.y), U2, V2);        // k = H-n: Y_{H-n}, Y_{M-n}; w^{H-n} = -conj(w^n)
      U[pad16(n)] = Un;
      V[pad16(n)] = Vn;
      U[pad16(n2)] = U2;
      V[pad16(n2)] = V2;
    }
  }
  cluster.sync();
  const int p0s = p0;
  split_inverse_store<LOGH>(smem, z, ns, p0s, q, sb, twb);
}

// ---------------------------------------------------------------------------------------------
// Commuted ordering column solve (kernels_commuted.cu k_time_solve): forward split, divide (MODE 1)
// or multiply (MODE 2) by lambda_n - dt sigma_p, inverse split.  In place allowed: rank q writes
// only rows it read itself, after the cluster barrier that follows its loads.
// ---------------------------------------------------------------------------------------------
template <int LOGH, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SGeo<LOGH>::NT, SGeo<LOGH>::NT <= 128 ? 4 : SGeo<LOGH>::NT <= 256 ? 2 : 1)
    k_time_solve_split(const double* __restrict__ u, double* __restrict__ z, int ns, const double* __restrict__ sf,
                       const double* __restrict__ sb, double s_in, const double2* __restrict__ lam,
                       const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  using G = SGeo<LOGH>;
  constexpr int H = G::H, M = G::M, B = G::B, BS = G::BS;
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const int p0 = int(blockIdx.x >> 1) * B;
  split_prefetch<LOGH>(u, ns, p0, q);
  split_forward<LOGH>(smem, u, ns, p0, q, sf, s_in, twb);
  cluster.sync();
  double2* Eb = cluster.map_shared_rank(smem, 0);
  double2* Ob = cluster.map_shared_rank(smem, 1);
  const double2* twM = twb + M;
  const double2* twT = twb + 2 * M;
  constexpr int HALF = (G::NTASK + 1) / 2;
  const int t1 = q == 0 ? HALF : G::NTASK;
  for (int t = q * HALF + int(threadIdx.x); t < t1; t += G::NT) {
    const int c = t % B, n = t / B;
    const int p = p0 + c;
    const double sg = p < ns ? __ldg(sigma + p) : 0.0;
    double2* E = Eb + c * BS;
    double2* O = Ob + c * BS;
    const double2 En = E[pad16(n)], On = O[pad16(n)];
    auto solve = [&](double2 zv, int k) {  // Z_k / (lambda_k - dt sigma_p)
      const double2 l = __ldg(lam + k);
      return shift_apply<MODE>(zv, l.x - dt * sg, l.y);
    };
    if (n == 0) {
      const double2 x0 = cadd(En, On), xh = csub(En, On);
      const double2 ya = solve(make_double2(x0.x + x0.y, 0.0), 0);
      const double2 yb = solve(make_double2(x0.x - x0.y, 0.0), M);
      const double2 A = cadd(ya, yb), Bv = csub(ya, yb);
      const double2 y0 = cadd(A, mul_si<1>(Bv));
      const double2 wch = __ldg(twT + H);
      double2 zh, zh2, yh, yh2;
      half_spectrum(xh, xh, wch, zh, zh2);
      const double2 sh = solve(zh, H);
      inverse_input(sh, sh, wch, yh, yh2);
      double2 U0, V0;
      uv(y0, yh, make_double2(1.0, 0.0), U0, V0);
      E[0] = U0;
      O[0] = V0;
      continue;
    }
    const int n2 = H - n;
    const double2 E2 = E[pad16(n2)], O2 = O[pad16(n2)];
    const double2 wn = cconj(__ldg(twM + n));
    const Bins4 X = split_bins(En, On, E2, O2, wn);
    const double2 wc = __ldg(twT + n);
    double2 zn, zmn, yn, ymn;
    half_spectrum(X.xn, X.xmmn, wc, zn, zmn);
    inverse_input(solve(zn, n), solve(zmn, M - n), wc, yn, ymn);
    if (n2 == n) {
      double2 Un, Vn;
      uv(yn, ymn, wn, Un, Vn);
      E[pad16(n)] = Un;
      O[pad16(n)] = Vn;
      continue;
    }
    const double2 wc2 = make_double2(-wc.y, -wc.x);
    double2 z2, zhp, y2, yhpn;
    half_spectrum(X.xhmn, X.xhpn, wc2, z2, zhp);
    inverse_input(solve(z2, n2), solve(zhp, H + n), wc2, y2, yhpn);
    double2 Un, Vn, U2, V2;
    uv(yn, yhpn, wn, Un, Vn);
    uv(y2, ymn, make_double2(-wn.x, wn.y), U2, V2);
    E[pad16(n)] = Un;
    O[pad16(n)] = Vn;
    E[pad16(n2)] = U2;
    O[pad16(n2)] = V2;
  }
  cluster.sync();
  split_inverse_store<LOGH>(smem, z, ns, p0, q, sb, twb);
}

// ---------------------------------------------------------------------------------------------
// launchers (Nt = 1024, 2048; other sizes: the 1-CTA kernels)
// ---------------------------------------------------------------------------------------------
#ifndef FPC_TSPLIT
#define FPC_TSPLIT 1
#endif

bool time_split_supported(int n_time) { return FPC_TSPLIT && (n_time == 1024 || n_time == 2048); }

template <class K>
static cudaError_t prep_s(K kernel, size_t smem, int threads) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       carveout_pct(smem, threads));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

template <int LOGH>
static cudaError_t fwd_split(const double* v, double2* Z, int ns, const double* sf, double s_in, const double2* tw,
                             cudaStream_t st) {
  using G = SGeo<LOGH>;
  cudaError_t e = prep_s(k_time_fwd_split<LOGH>, G::SMEM, G::NT);
  if (e != cudaSuccess) return e;
  k_time_fwd_split<LOGH><<<2 * ((ns + G::B - 1) / G::B), G::NT, G::SMEM, st>>>(v, Z, ns, sf, s_in, tw); note_launch();
  return cudaGetLastError();
}
template <int LOGH>
static cudaError_t inv_split(const double2* Z, double* z, int ns, const double* sb, const double2* tw,
                             cudaStream_t st) {
  using G = SGeo<LOGH>;
  cudaError_t e = prep_s(k_time_inv_split<LOGH>, G::SMEM, G::NT);
  if (e != cudaSuccess) return e;
  k_time_inv_split<LOGH><<<2 * ((ns + G::B - 1) / G::B), G::NT, G::SMEM, st>>>(Z, z, ns, sb, tw); note_launch();
  return cudaGetLastError();
}
template <int LOGH, int MODE>
static cudaError_t solve_split(const double* u, double* z, int ns, const double* sf, const double* sb, double s_in,
                               const double2* lam, const double* sigma, double dt, const double2* tw,
                               cudaStream_t st) {
  using G = SGeo<LOGH>;
  cudaError_t e = prep_s(k_time_solve_split<LOGH, MODE>, G::SMEM, G::NT);
  if (e != cudaSuccess) return e;
  k_time_solve_split<LOGH, MODE><<<2 * ((ns + G::B - 1) / G::B), G::NT, G::SMEM, st>>>(u, z, ns, sf, sb, s_in, lam,
                                                                                       sigma, dt, tw); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_time_fwd_split(const double* v, double2* Z, int n_space, int n_time, const double* scale_fwd,
                                  double s_in, const double2* tw_base, cudaStream_t st) {
  if (n_time == 2048) return fwd_split<9>(v, Z, n_space, scale_fwd, s_in, tw_base, st);
  if (n_time == 1024) return fwd_split<8>(v, Z, n_space, scale_fwd, s_in, tw_base, st);
  return cudaErrorInvalidValue;
}
cudaError_t launch_time_inv_split(const double2* Z, double* z, int n_space, int n_time, const double* scale_bwd,
                                  const double2* tw_base, cudaStream_t st) {
  if (n_time == 2048) return inv_split<9>(Z, z, n_space, scale_bwd, tw_base, st);
  if (n_time == 1024) return inv_split<8>(Z, z, n_space, scale_bwd, tw_base, st);
  return cudaErrorInvalidValue;
}
cudaError_t launch_time_solve_split(const double* u, double* z, int n_space, int n_time, const double* scale_fwd,
                                    const double* scale_bwd, double s_in, const double2* lambda,
                                    const double* sigma, double dt, const double2* tw_base, cudaStream_t st,
                                    bool forward) {
  if (n_time == 2048)
    return forward ? solve_split<9, 2>(u, z, n_space, scale_fwd, scale_bwd, s_in, lambda, sigma, dt, tw_base, st)
                   : solve_split<9, 1>(u, z, n_space, scale_fwd, scale_bwd, s_in, lambda, sigma, dt, tw_base, st);
  if (n_time == 1024)
    return forward ? solve_split<8, 2>(u, z, n_space, scale_fwd, scale_bwd, s_in, lambda, sigma, dt, tw_base, st)
                   : solve_split<8, 1>(u, z, n_space, scale_fwd, scale_bwd, s_in, lambda, sigma, dt, tw_base, st);
  return cudaErrorInvalidValue;
}

}  // namespace fpc
