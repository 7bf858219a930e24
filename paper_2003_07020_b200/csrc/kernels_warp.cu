// kernels_warp.cu -- lattice-row kernels on warp-owned register FFTs (warp_fft.cuh), sm_100a.
//
// Rows matvec (all_at_once.hpp:33-55 with toeplitz.hpp:41-57 along contiguous rows; the 2D
// y-direction half of jacobian.hpp:84-87): one row of length ns <= M - 1 per group of R lanes,
// real packing of the length-L = 2M circulant embedding into an M = R*R point complex transform,
// so a 255-point row (config 2, L = 512) is one 256-point FFT per direction held in 16 lanes x 16
// registers.  Per row: three global row reads (v_k and the BDF2 stencil's v_{k-1}, v_{k-2}, all
// issued up front: 48 loads in flight per lane), forward FFT, the packed pointwise product with
// the circulant eigenvalues (each bin with its mirror M - k, exchanged through the group's tile),
// inverse FFT -- which returns each lane exactly the positions it loaded -- and one coalesced row
// write.  No CTA barrier: a CTA is 8 independent warps.
#include <cstdlib>

#include "bulk_copy.cuh"
#include "kernels.cuh"
#include "warp_dst.cuh"
#include "warp_fft.cuh"

namespace fpc {

namespace {

// Pointwise circulant product on the packed spectrum for bin k of an M-point packed transform
// (the spectral loop of kernels_1d.cu k_matvec_1d, per bin): own = Z_k, mir = Z_{M-k}; returns the
// packed inverse-transform input U_k.  eig = eig' (M + 1 values, -dt eig/(2L) pre-folded),
// twL = tw_L (L = 2M).
template <int M>
__device__ __forceinline__ double2 packed_eig_product(double2 own, double2 mir, int k, const double* __restrict__ eig,
                                                      const double2* __restrict__ twL) {
  if (k == 0) {
    const double y0 = __ldg(eig) * (2.0 * (own.x + own.y));
    const double ym = __ldg(eig + M) * (2.0 * (own.x - own.y));
    return make_double2(y0 + ym, y0 - ym);
  }
  const bool lo = k <= M / 2;
  const int kk = lo ? k : M - k;
  const double2 a = lo ? own : mir, bq = lo ? mir : own;
  const double2 w = __ldg(twL + kk);  // e^{-2 pi i kk/L}
  const double ek = __ldg(eig + kk), em = __ldg(eig + M - kk);
  const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
  const double2 iwQ = mul_si<1>(cmul(w, Q));
  const double2 Yk = cscale(csub(P, iwQ), ek);
  const double2 Ym = cscale(cconj(cadd(P, iwQ)), em);
  const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
  return lo ? cadd(A, mul_si<1>(cmul(D, cconj(w)))) : cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
}

// The packed circulant product of a whole group spectrum with each mirror pair (k, M - k) formed
// once: lane t computes the pairs of its bins k = t + 16 p, p < 8 (k < M/2), keeps U_k and stores
// U_{M-k} into the tile slot of bin M - k -- a slot only this lane reads (its mirror operand,
// read just before) -- then reads its bins p >= 8 back; bin M/2 (lane 0, p = 8) pairs with itself.
// Same per-pair arithmetic as k_matvec_1d's spectral loop (kernels_1d.cu).
#ifndef FPC_MV_SHFL
#define FPC_MV_SHFL 1
#endif
// The same with the mirror operands and the partners' results exchanged by width-16 shuffles instead
// of the tile (B200: a double2 through the tile is a 4-wavefront store plus a 4-wavefront load on the
// L1/shared pipe these kernels are bound on; the DST's mirror exchange gained 3% this way).
__device__ __forceinline__ void warp_packed_product_shfl(double2 (&z)[16], int t, const double* __restrict__ eig,
                                                         const double2* __restrict__ twL) {
  constexpr int R = 16, M = 256, H = 8;
  const int src = (R - t) & (R - 1);
  const double2 mid = z[H];  // lane 0: bin M/2
  double2 um[H];             // U_{M-k} of this lane's pairs k = t + 16 p, p < 8
#pragma unroll
  for (int p = 0; p < H; ++p) {
    const int k = t + R * p;
    const double2 a = z[p];
    // Z_{M-k}: lane (16 - t) mod 16, register 15 - p (t != 0); this lane's register 16 - p (t = 0)
    double2 bq;
    bq.x = __shfl_sync(0xffffffffu, z[R - 1 - p].x, src, R);
    bq.y = __shfl_sync(0xffffffffu, z[R - 1 - p].y, src, R);
    if (t == 0) bq = z[(R - p) & (R - 1)];
    if (k == 0) {
      const double y0 = __ldg(eig) * (2.0 * (a.x + a.y));
      const double ym = __ldg(eig + M) * (2.0 * (a.x - a.y));
      z[p] = make_double2(y0 + ym, y0 - ym);
      um[p] = make_double2(0.0, 0.0);
      continue;
    }
    const double2 w = __ldg(twL + k);  // e^{-2 pi i k/L}
    const double ek = __ldg(eig + k), em = __ldg(eig + M - k);
    const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), em);
    const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
    z[p] = cadd(A, mul_si<1>(cmul(D, cconj(w))));
    um[p] = cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
  }
  double2 zmid = mid;
  if (t == 0) {  // the self pair k = M/2
    const double2 w = __ldg(twL + M / 2);
    const double ek = __ldg(eig + M / 2);
    const double2 P = cadd(mid, cconj(mid)), Q = csub(mid, cconj(mid));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), ek);
    const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
    zmid = cadd(A, mul_si<1>(cmul(D, cconj(w))));
  }
  // bin k' = t + 16 p' (p' >= 8) = M - k with k = (16 - t) + 16 (15 - p'): lane 16 - t, pair 15 - p'
  // (t != 0); lane 0: k' = 16 p' = M - 16 (16 - p'): its own pair 16 - p' (p' >= 9), p' = 8 the self pair
#pragma unroll
  for (int pp = H; pp < R; ++pp) {
    double2 u;
    u.x = __shfl_sync(0xffffffffu, um[R - 1 - pp].x, src, R);
    u.y = __shfl_sync(0xffffffffu, um[R - 1 - pp].y, src, R);
    if (t == 0) u = pp == H ? zmid : um[(R - pp) & (H - 1)];
    z[pp] = u;
  }
}

template <int R>
__device__ __forceinline__ void warp_packed_product(double2 (&z)[R], double2* __restrict__ xs, int t,
                                                    const double* __restrict__ eig, const double2* __restrict__ twL) {
  constexpr int M = R * R, LD = WarpFftTile<R>::LD, H = R / 2;
  if constexpr (R == 16 && FPC_MV_SHFL) {
    warp_packed_product_shfl(z, t, eig, twL);
    return;
  }
#pragma unroll
  for (int p = 0; p < R; ++p) xs[p * LD + t] = z[p];
  __syncwarp();
  const int tm = (R - t) & (R - 1);
  const double2 mid = z[H];  // lane 0: bin M/2
#pragma unroll
  for (int p = 0; p < H; ++p) {
    const int k = t + R * p;
    const double2 a = z[p];
    if (k == 0) {
      const double y0 = __ldg(eig) * (2.0 * (a.x + a.y));
      const double ym = __ldg(eig + M) * (2.0 * (a.x - a.y));
      z[p] = make_double2(y0 + ym, y0 - ym);
      continue;
    }
    const int pm = t == 0 ? ((R - p) & (R - 1)) : (R - 1 - p);
    double2* slot = xs + pm * LD + tm;
    const double2 bq = *slot;
    const double2 w = __ldg(twL + k);  // e^{-2 pi i k/L}
    const double ek = __ldg(eig + k), em = __ldg(eig + M - k);
    const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), em);
    const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
    z[p] = cadd(A, mul_si<1>(cmul(D, cconj(w))));
    *slot = cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
  }
  if (t == 0) {  // the self pair k = M/2
    const double2 w = __ldg(twL + M / 2);
    const double ek = __ldg(eig + M / 2);
    const double2 P = cadd(mid, cconj(mid)), Q = csub(mid, cconj(mid));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), ek);
    const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
    z[H] = cadd(A, mul_si<1>(cmul(D, cconj(w))));
  }
  __syncwarp();
#pragma unroll
  for (int p = H; p < R; ++p)
    if (!(t == 0 && p == H)) z[p] = xs[p * LD + t];
  __syncwarp();
}

// BDF2 stencil part (time_stencil.hpp:16-26, same association as all_at_once.hpp:44-53)
__device__ __forceinline__ double bdf2(int k, double x0, double x1, double x2) {
  if (k == 0) return x0;
  if (k == 1) return 1.5 * x0 + -2.0 * x1;
  return 1.5 * x0 + -2.0 * x1 + 0.5 * x2;
}

#ifndef FPC_COL_WARPS
#define FPC_COL_WARPS 4  // B200 config 2: matvec columns 4 warps (8 columns) per CTA, tau columns 4 (8 columns)
#endif
#ifndef FPC_TAU_COL_WARPS
#define FPC_TAU_COL_WARPS 4  // with FPC_TAU_COL_OCC 12 (170 registers, no spills): config-2 tau solve 505 -> 496 us
#endif
constexpr int kTauColWarps = FPC_TAU_COL_WARPS;
#ifndef FPC_TAU_COL_OCC
#define FPC_TAU_COL_OCC 12
#endif
constexpr int kTauColOcc = FPC_TAU_COL_OCC;
#ifndef FPC_COL_OCC
#define FPC_COL_OCC 16
#endif
constexpr int kColOcc = FPC_COL_OCC;
constexpr int kWarpsPerCta = FPC_COL_WARPS;  // column kernels: a CTA covers 2 * kWarpsPerCta adjacent columns
// Row kernels (contiguous rows: nothing shared between a CTA's warps): smaller CTAs, the same 16
// warps per SM -- the warps of a CTA start together and so wait on their row loads together; more,
// smaller CTAs spread those phases (FPC_ROW_WARPS: build knob).
#ifndef FPC_ROW_WARPS
#define FPC_ROW_WARPS 1  // config 2: matvec 518 (4 warps) -> 511 (2) -> 500 us (1), tau solve 527 -> 524 us
#endif
constexpr int kRowWarps = FPC_ROW_WARPS;
#ifndef FPC_ROW_OCC
#define FPC_ROW_OCC 16  // resident warps per SM the row kernels are compiled for (register cap 65536 / 32 / occ)
#endif
constexpr int kRowOcc = FPC_ROW_OCC;
#ifndef FPC_DST_ROW_OCC
#define FPC_DST_ROW_OCC 12  // config 2: tau solve 527 (16 warps per SM, 128 registers, 16-192 B of spills) -> 506 us (12 or 10 warps); 8: 527
#endif
constexpr int kDstRowOcc = FPC_DST_ROW_OCC;

// Row data read once (no reuse inside the SM): L2-only loads keep the L1 for the twiddle and
// eigenvalue tables.  FPC_WARP_CG=0 restores plain loads (A/B).
#ifndef FPC_WARP_CG
#define FPC_WARP_CG 1
#endif
#ifndef FPC_COLS_RED
#define FPC_COLS_RED 1
#endif
__device__ __forceinline__ double ld_once(const double* p) {
#if FPC_WARP_CG
  return __ldcg(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ double2 ld_once(const double2* p) {
#if FPC_WARP_CG
  return __ldcg(p);
#else
  return *p;
#endif
}

// Shared-memory carveout of the warp kernels (two 256-thread CTAs per SM): FPC_WARP_CARVE = percent,
// "auto" = the smallest capacity that holds two CTAs (kernels.cuh carveout_pct), unset = driver default.
cudaError_t set_warp_carveout(const void* kernel, size_t smem) {
  static const int mode = [] {
    const char* e = std::getenv("FPC_WARP_CARVE");
    if (!e || !e[0]) return -1;
    if (e[0] == 'a') return -2;
    return std::atoi(e);
  }();
  if (mode == -1) return cudaSuccess;
  const int pct = mode == -2 ? carveout_pct(smem, 32 * kWarpsPerCta) : mode;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

}  // namespace

bool warp_kernels_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPC_WARP");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int R>
__global__ void __launch_bounds__(32 * kRowWarps, kRowOcc / kRowWarps)
    k_mv_rows_warp(const double* __restrict__ v, double* __restrict__ y, int ns, int nrows, int rpt,
                   int sstride, int koff, const double* __restrict__ eig, const double2* __restrict__ twb) {
  constexpr int M = R * R, L = 2 * M, G = 32 / R, H = R / 2;
  constexpr int LD = WarpFftTile<R>::LD;
  extern __shared__ double2 wsm[];
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;
  const int row = int(blockIdx.x) * (kRowWarps * G) + grp;
  const bool valid = row < nrows;
  const int rr = valid ? row : nrows - 1;  // out-of-range groups compute a duplicate, store nothing
  const int k = rr / rpt + koff;
  const double* vr = v + size_t(rr) * ns;
  double2* xs = wsm + grp * WarpFftTile<R>::SIZE;

  // packed slot m = t + R r holds (x_{2m}, x_{2m+1}); slots with 2m >= ns are the zero padding of
  // the embedding (all of r >= R/2, since ns <= M - 1)
  double2 z[R];
  double x1[2 * H], x2[2 * H];
#pragma unroll
  for (int r = 0; r < H; ++r) {
    const int i0 = 2 * (t + R * r);
    const bool ok0 = i0 < ns, ok1 = i0 + 1 < ns;
    z[r] = make_double2(ok0 ? ld_once(vr + i0) : 0.0, ok1 ? ld_once(vr + i0 + 1) : 0.0);
    x1[2 * r] = (ok0 && k >= 1) ? ld_once(vr + (i0 - sstride)) : 0.0;
    x1[2 * r + 1] = (ok1 && k >= 1) ? ld_once(vr + (i0 + 1 - sstride)) : 0.0;
    x2[2 * r] = (ok0 && k >= 2) ? ld_once(vr + i0 - 2 * size_t(sstride)) : 0.0;
    x2[2 * r + 1] = (ok1 && k >= 2) ? ld_once(vr + i0 + 1 - 2 * size_t(sstride)) : 0.0;
  }
#pragma unroll
  for (int r = H; r < R; ++r) z[r] = make_double2(0.0, 0.0);
  // stencil part, formed now so the two earlier rows' registers are free during the transforms
  double c[2 * H];
#pragma unroll
  for (int r = 0; r < H; ++r) {
    c[2 * r] = bdf2(k, z[r].x, x1[2 * r], x2[2 * r]);
    c[2 * r + 1] = bdf2(k, z[r].y, x1[2 * r + 1], x2[2 * r + 1]);
  }

  // the zero-padded upper half in, the truncated lower half out (pruned first / last passes)
  warp_fft_sq<R, -1, true, false>(z, xs, t, twb);  // lane t now holds Z_{t + R p}
  warp_packed_product<R>(z, xs, t, eig, twb + L);   // each mirror pair (k, M - k) once
  warp_fft_sq<R, 1, false, true>(z, xs, t, twb);   // lane t holds the packed inverse at slots t + R r < M/2

  if (valid) {
    double* yr = y + size_t(row) * ns;
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int i0 = 2 * (t + R * r);
      if (i0 < ns) yr[i0] = c[2 * r] + z[r].x;
      if (i0 + 1 < ns) yr[i0 + 1] = c[2 * r + 1] + z[r].y;
    }
  }
}

// Rows matvec on warp FFTs for M = R*R (R = 16: M = 256, rows of 129..255 points).  Returns
// cudaErrorNotSupported for other sizes (the caller keeps the CTA-level kernel).
cudaError_t launch_matvec_rows_warp(const double* v, double* y, int len, int nrows, int rpt, int sstride,
                                    int log_m, const double* eig_scaled, const double2* tw_base,
                                    cudaStream_t st, int koff) {
  if (log_m != 8) return cudaErrorNotSupported;
  constexpr int R = 16, G = 32 / R;
  const int rows_per_cta = kRowWarps * G;
  const size_t smem = size_t(kRowWarps) * G * WarpFftTile<R>::SIZE * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(k_mv_rows_warp<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  if ((e = set_warp_carveout((const void*)k_mv_rows_warp<R>, smem)) != cudaSuccess) return e;
  k_mv_rows_warp<R><<<(nrows + rows_per_cta - 1) / rows_per_cta, 32 * kRowWarps, smem, st>>>(
      v, y, len, nrows, rpt, sstride, koff, eig_scaled, tw_base); note_launch();
  return cudaGetLastError();
}

// DST-I rows of n = 255 complex points on 16-lane groups (warp_dst.cuh), in place: MODE 0 = the
// row DSTs of the 2D tau solve (tau.hpp:85-86); MODE 1 / 2 = the 1D tau solve / forward action of
// frequency row r (tau.hpp:98-136): DST, divide (multiply) by lambda_r - dt sigma_i, DST, with the
// intermediate kept in the group's tile.
template <int MODE>
__global__ void __launch_bounds__(32 * kRowWarps, kDstRowOcc / kRowWarps)
    k_dst_rows_warp(double2* __restrict__ Z, int n_rows, const double2* __restrict__ lam,
                    const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  constexpr int R = 16, G = 2, NSR = 255;
  extern __shared__ double2 wsm[];
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;
  const int row = int(blockIdx.x) * (kRowWarps * G) + grp;
  const bool valid = row < n_rows;
  const int rr = valid ? row : n_rows - 1;
  double2* zr = Z + size_t(rr) * NSR;
  double2* xs = wsm + grp * kDstTileSize;
  const double scale = 0.088388347648318440550;  // sqrt(2/256)
  warp_dst256([&](int j) { return zr[j - 1]; }, xs, t, twb, scale);
  if constexpr (MODE != 0) {
    const double2 l = __ldg(lam + rr);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = t + R * r;
      if (i < NSR) xs[dst_slot(i)] = shift_apply<MODE>(xs[dst_slot(i)], l.x - dt * __ldg(sigma + i), l.y);
    }
    __syncwarp();
    warp_dst256([&](int j) { return xs[dst_slot(j - 1)]; }, xs, t, twb, scale);
  }
  if (valid) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = t + R * r;
      if (i < NSR) zr[i] = xs[dst_slot(i)];
    }
  }
}

cudaError_t launch_dst_rows_warp(double2* Z, int n, int n_rows, const double2* lambda, const double* sigma,
                                 double dt, const double2* tw_base, cudaStream_t st, int mode) {
  if (n != 255) return cudaErrorNotSupported;
  constexpr int R = 16, G = 2;
  const int rows_per_cta = kRowWarps * G;
  const size_t smem = size_t(kRowWarps) * G * kDstTileSize * sizeof(double2);
  const unsigned grid = unsigned((n_rows + rows_per_cta - 1) / rows_per_cta);
#define FPC_DSTW(MODE)                                                                                        \
  {                                                                                                           \
    cudaError_t e = cudaFuncSetAttribute(k_dst_rows_warp<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                         int(smem));                                                          \
    if (e != cudaSuccess) return e;                                                                           \
    if ((e = set_warp_carveout((const void*)k_dst_rows_warp<MODE>, smem)) != cudaSuccess) return e;           \
    k_dst_rows_warp<MODE><<<grid, 32 * kRowWarps, smem, st>>>(Z, n_rows, lambda, sigma, dt, tw_base);     \
    note_launch();                                                                                            \
  }
  if (mode == 0)
    FPC_DSTW(0)
  else if (mode == 1)
    FPC_DSTW(1)
  else
    FPC_DSTW(2)
#undef FPC_DSTW
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// 2D matvec, x-direction half (jacobian.hpp:88-93): y[k][ix][iy] += (dt sx / 2L) (T_x v[k][.][iy])[ix]
// for n <= 255 (M = 256).  A CTA owns 16 columns iy of one time level: the [256][16] tile is
// loaded cooperatively (128-byte row segments, coalesced) into shared memory, each 16-lane group
// transforms one column straight from the tile (no CTA barrier inside the transforms), writes the
// result back into its tile column, and the CTA adds the tile to y row by row (coalesced).
constexpr int kColTile = 2 * kWarpsPerCta;  // columns per CTA = groups per CTA
constexpr int kColPitch = 17;        // tile row pitch in doubles: the groups' column reads hit 16 bank pairs
__global__ void __launch_bounds__(32 * kWarpsPerCta, kColOcc / kWarpsPerCta)
    k_mv_cols_warp(const double* __restrict__ v, double* __restrict__ y, int n, const double* __restrict__ eig,
                   const double2* __restrict__ twb) {
  constexpr int R = 16, M = R * R, L = 2 * M, H = R / 2, G = 2;
  constexpr int LD = WarpFftTile<R>::LD;
  constexpr int NTHR = 32 * kWarpsPerCta;
  extern __shared__ double2 wsm[];
  double* tile = reinterpret_cast<double*>(wsm + kWarpsPerCta * G * WarpFftTile<R>::SIZE);  // [M][kColPitch]
  const int tiles = (n + kColTile - 1) / kColTile;
  const int k = int(blockIdx.x) / tiles;
  const int iy0 = (int(blockIdx.x) - k * tiles) * kColTile;
  const size_t base = size_t(k) * size_t(n) * size_t(n);
  const int ncol = min(kColTile, n - iy0);
  // 1. tile load: element (ix, c) = v[k][ix][iy0 + c], rows ix >= n zero (16 loads in flight per thread)
  constexpr int UL = M * kColTile / NTHR;  // 16
  double x[UL];
#pragma unroll
  for (int u = 0; u < UL; ++u) {
    const int e = int(threadIdx.x) + u * NTHR;
    const int ix = e / kColTile, c = e % kColTile;
    x[u] = (ix < n && c < ncol) ? v[base + size_t(ix) * n + iy0 + c] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < UL; ++u) {
    const int e = int(threadIdx.x) + u * NTHR;
    tile[(e / kColTile) * kColPitch + e % kColTile] = x[u];
  }
  __syncthreads();
  // 2. one column per group: packed slot m = t + R r holds (x_{2m}, x_{2m+1}) of the column
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;  // = the tile column
  double2* xs = wsm + grp * WarpFftTile<R>::SIZE;
  double2 z[R];
#pragma unroll
  for (int r = 0; r < H; ++r) {
    const int m = t + R * r;
    z[r] = make_double2(tile[(2 * m) * kColPitch + grp], tile[(2 * m + 1) * kColPitch + grp]);
  }
#pragma unroll
  for (int r = H; r < R; ++r) z[r] = make_double2(0.0, 0.0);
  warp_fft_sq<R, -1>(z, xs, t, twb);
#pragma unroll
  for (int p = 0; p < R; ++p) xs[p * LD + t] = z[p];
  __syncwarp();
  const int tm = (R - t) & (R - 1);
#pragma unroll
  for (int p = 0; p < R; ++p) {
    const int pm = t == 0 ? ((R - p) & (R - 1)) : (R - 1 - p);
    z[p] = packed_eig_product<M>(z[p], xs[pm * LD + tm], t + R * p, eig, twb + L);
  }
  __syncwarp();
  warp_fft_sq<R, 1>(z, xs, t, twb);
#pragma unroll
  for (int r = 0; r < H; ++r) {
    const int m = t + R * r;
    tile[(2 * m) * kColPitch + grp] = z[r].x;
    tile[(2 * m + 1) * kColPitch + grp] = z[r].y;
  }
  __syncthreads();
  // 3. y += tile, row segments of ncol doubles (coalesced read-modify-write)
  double yo[UL];
#pragma unroll
  for (int u = 0; u < UL; ++u) {
    const int e = int(threadIdx.x) + u * NTHR;
    const int ix = e / kColTile, c = e % kColTile;
    yo[u] = (ix < n && c < ncol) ? y[base + size_t(ix) * n + iy0 + c] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < UL; ++u) {
    const int e = int(threadIdx.x) + u * NTHR;
    const int ix = e / kColTile, c = e % kColTile;
    if (ix < n && c < ncol) y[base + size_t(ix) * n + iy0 + c] = yo[u] + tile[ix * kColPitch + c];
  }
}

// The same column pass without the shared tile: each group loads its column straight into
// registers (a warp's two groups read 16 B per row; a CTA's 8 warps cover 128-byte row segments, so
// the L2 sectors are shared within the CTA) and adds its result to y directly -- warps never wait
// on each other.  FPC_COLS_TILE=1 selects the tiled kernel above (A/B).
__global__ void __launch_bounds__(32 * kWarpsPerCta, kColOcc / kWarpsPerCta)
    k_mv_cols_direct(const double* __restrict__ v, double* __restrict__ y, int n, const double* __restrict__ eig,
                     const double2* __restrict__ twb) {
  constexpr int R = 16, M = R * R, L = 2 * M, H = R / 2, G = 2;
  constexpr int LD = WarpFftTile<R>::LD;
  extern __shared__ double2 wsm[];
  const int tiles = (n + kColTile - 1) / kColTile;
  const int k = int(blockIdx.x) / tiles;
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;
  const int iy = (int(blockIdx.x) - k * tiles) * kColTile + grp;
  const bool valid = iy < n;
  const double* vc = v + size_t(k) * size_t(n) * size_t(n) + (valid ? iy : 0);
  double2* xs = wsm + grp * WarpFftTile<R>::SIZE;
  double2 z[R];
#pragma unroll
  for (int r = 0; r < H; ++r) {
    const int i0 = 2 * (t + R * r);
    z[r] = make_double2(i0 < n ? vc[size_t(i0) * n] : 0.0, i0 + 1 < n ? vc[size_t(i0 + 1) * n] : 0.0);
  }
#pragma unroll
  for (int r = H; r < R; ++r) z[r] = make_double2(0.0, 0.0);
  warp_fft_sq<R, -1, true, false>(z, xs, t, twb);
  warp_packed_product<R>(z, xs, t, eig, twb + L);
  warp_fft_sq<R, 1, false, true>(z, xs, t, twb);
  if (valid) {
    double* yc = y + size_t(k) * size_t(n) * size_t(n) + iy;
#if FPC_COLS_RED
    // y += result as reductions performed at the L2 (RED.ADD.F64, no return value): every element
    // receives exactly one add, so the sum is the same double as load-add-store, without the
    // strided read of y, its registers or the wait for it at the end of the task
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int i0 = 2 * (t + R * r);
      if (i0 < n) atomicAdd(yc + size_t(i0) * n, z[r].x);
      if (i0 + 1 < n) atomicAdd(yc + size_t(i0 + 1) * n, z[r].y);
    }
#else
    double yo[2 * H];
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int i0 = 2 * (t + R * r);
      yo[2 * r] = i0 < n ? yc[size_t(i0) * n] : 0.0;
      yo[2 * r + 1] = i0 + 1 < n ? yc[size_t(i0 + 1) * n] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int i0 = 2 * (t + R * r);
      if (i0 < n) yc[size_t(i0) * n] = yo[2 * r] + z[r].x;
      if (i0 + 1 < n) yc[size_t(i0 + 1) * n] = yo[2 * r + 1] + z[r].y;
    }
#endif
  }
}

cudaError_t launch_matvec_cols_warp(const double* v, double* y, int n, int n_time, int log_m, const double* eig_x,
                                    const double2* tw_base, cudaStream_t st) {
  if (log_m != 8) return cudaErrorNotSupported;
  constexpr int R = 16, G = 2, M = 256;
  const int tiles = (n + kColTile - 1) / kColTile;
  static const bool tiled = [] {
    const char* e = std::getenv("FPC_COLS_TILE");
    return e && e[0] == '1';
  }();
  if (!tiled) {
    const size_t smem = size_t(kWarpsPerCta) * G * WarpFftTile<R>::SIZE * sizeof(double2);
    cudaError_t e = cudaFuncSetAttribute(k_mv_cols_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    if ((e = set_warp_carveout((const void*)k_mv_cols_direct, smem)) != cudaSuccess) return e;
    k_mv_cols_direct<<<unsigned(n_time) * unsigned(tiles), 32 * kWarpsPerCta, smem, st>>>(v, y, n, eig_x, tw_base);
    note_launch();
    return cudaGetLastError();
  }
  const size_t smem = size_t(kWarpsPerCta) * G * WarpFftTile<R>::SIZE * sizeof(double2) +
                      size_t(M) * kColPitch * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_mv_cols_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k_mv_cols_warp<<<unsigned(n_time) * unsigned(tiles), 32 * kWarpsPerCta, smem, st>>>(v, y, n, eig_x, tw_base);
  note_launch();
  return cudaGetLastError();
}

// 2D tau solve, column pass (tau.hpp:79-119 along ix): for frequency plane r and column iy, DST over
// ix, divide (MODE 1) / multiply (MODE 2) by lambda_r - dt sigma[ix n + iy], DST over ix, in place.
// sigma = the plan's table [ix][iy] followed by its transpose [iy][ix] (read here: contiguous in ix).
// One 16-lane group per column, loads straight from global memory (a warp's two groups read
// adjacent 16-byte elements of each row; a CTA's 16 groups cover 256-byte row segments), the
// intermediate kept in the group's tile.  n = 255.
template <int MODE>
__global__ void __launch_bounds__(32 * kTauColWarps, kTauColOcc / kTauColWarps)
    k_tau_cols_warp(double2* __restrict__ Z, int n_planes, const double2* __restrict__ lam,
                    const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  constexpr int R = 16, G = 2, NSR = 255, NG = kTauColWarps * G;
  extern __shared__ double2 wsm[];
  constexpr int tiles = (NSR + NG - 1) / NG;
  const int rp = int(blockIdx.x) / tiles;
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;
  const int iy = (int(blockIdx.x) - rp * tiles) * NG + grp;
  const bool valid = iy < NSR;
  double2* zc = Z + size_t(rp) * NSR * NSR + (valid ? iy : 0);
  double2* xs = wsm + grp * kDstTileSize;
  const double scale = 0.088388347648318440550;  // sqrt(2/256)
  const double* sg = sigma + size_t(NSR) * NSR + size_t(valid ? iy : 0) * NSR;  // transposed table: row iy
  warp_dst256([&](int j) { return zc[size_t(j - 1) * NSR]; }, xs, t, twb, scale);
  const double2 l = __ldg(lam + rp);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = t + R * r;
    if (i < NSR) xs[dst_slot(i)] = shift_apply<MODE>(xs[dst_slot(i)], l.x - dt * __ldg(sg + i), l.y);
  }
  __syncwarp();
  warp_dst256([&](int j) { return xs[dst_slot(j - 1)]; }, xs, t, twb, scale);
  if (valid) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = t + R * r;
      if (i < NSR) zc[size_t(i) * NSR] = xs[dst_slot(i)];
    }
  }
}

// The tau column pass with the CTA's 16 columns staged through the groups' own tiles: the CTA copies
// row segments of 16 complex values (256 bytes: two rows per warp instruction, against one element
// of 16 different rows per instruction in the direct kernel -- on the L1 data pipe these kernels
// are bound on, a strided access costs a wavefront per row touched) straight into the DST's slot
// layout, each group transforms from and into its tile, and the CTA writes the tile back the same
// way.  Tile c is shifted by c mod 8 slots so the 8 columns of a quarter warp hit 8 different banks.
constexpr int kDstTileStage = kDstTileSize + 16;  // 304 double2: a multiple of 8, + the shift
#ifndef FPC_TAU_STAGED_WARPS
#define FPC_TAU_STAGED_WARPS 4
#endif
constexpr int kTauStWarps = FPC_TAU_STAGED_WARPS;  // 8 columns per CTA (128-byte row segments), four CTAs per SM
template <int MODE>
__global__ void __launch_bounds__(32 * kTauStWarps, kTauColOcc / kTauStWarps)
    k_tau_cols_staged(double2* __restrict__ Z, int n_planes, const double2* __restrict__ lam,
                      const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  constexpr int R = 16, G = 2, NSR = 255, NG = kTauStWarps * G, NT = 32 * kTauStWarps, RS = NT / NG;
  extern __shared__ double2 wsm[];
  constexpr int tiles = (NSR + NG - 1) / NG;
  const int rp = int(blockIdx.x) / tiles;
  const int iy0 = (int(blockIdx.x) - rp * tiles) * NG;
  const int ncol = min(NG, NSR - iy0);
  double2* zb = Z + size_t(rp) * NSR * NSR + iy0;
  const int c = int(threadIdx.x) % NG, ix0 = int(threadIdx.x) / NG;
  const bool okc = c < ncol;
  {
    double2* dst = wsm + c * kDstTileStage + (c & 7);
    const double2* zc = zb + (okc ? c : 0);
#pragma unroll
    for (int u = 0; u < (NSR + RS - 1) / RS; ++u) {
      const int ix = ix0 + u * RS;
      if (ix < NSR) cp_async16_zfill(dst + dst_slot(ix), zc + size_t(ix) * NSR, okc);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;
  double2* xs = wsm + grp * kDstTileStage + (grp & 7);
  const double scale = 0.088388347648318440550;  // sqrt(2/256)
  const double* sg = sigma + size_t(NSR) * NSR + size_t(min(iy0 + grp, NSR - 1)) * NSR;  // transposed table
  warp_dst256([&](int j) { return xs[dst_slot(j - 1)]; }, xs, t, twb, scale);
  const double2 l = __ldg(lam + rp);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = t + R * r;
    if (i < NSR) xs[dst_slot(i)] = shift_apply<MODE>(xs[dst_slot(i)], l.x - dt * __ldg(sg + i), l.y);
  }
  __syncwarp();
  warp_dst256([&](int j) { return xs[dst_slot(j - 1)]; }, xs, t, twb, scale);
  __syncthreads();
  if (okc) {
    const double2* src = wsm + c * kDstTileStage + (c & 7);
#pragma unroll
    for (int u = 0; u < (NSR + RS - 1) / RS; ++u) {
      const int ix = ix0 + u * RS;
      if (ix < NSR) zb[size_t(ix) * NSR + c] = src[dst_slot(ix)];
    }
  }
}

// Row transforms with a transposed store, for the 2D tau solve without strided loads (tau.hpp:79-119):
// plane p of `in` holds 255 contiguous rows; each 16-lane group transforms one row (MODE 0: DST;
// MODE 1 / 2: DST, divide / multiply by lambda_p - dt sigma, DST), and the CTA's 8 rows r0..r0+7 are
// written to out[p][c][r0..r0+7] -- 128-byte segments -- from the groups' tiles.  Two such passes
// and an in-place row pass make the solve: Z -> (DST_y, transpose) -> ZT -> (DST_x, shift, DST_x,
// transpose back) -> Z -> DST_y.  sigT = the transposed sigma table [iy][ix].
template <int MODE>
__global__ void __launch_bounds__(32 * 4, 3)
    k_dst_rows_T(const double2* __restrict__ in, double2* __restrict__ out, const double2* __restrict__ lam,
                 const double* __restrict__ sigT, double dt, const double2* __restrict__ twb) {
  constexpr int R = 16, G = 2, NSR = 255, NG = 4 * G, TPP = (NSR + NG - 1) / NG;
  extern __shared__ double2 wsm[];
  const int p = int(blockIdx.x) / TPP;
  const int r0 = (int(blockIdx.x) - p * TPP) * NG;
  const int lane = int(threadIdx.x) & 31;
  const int t = lane & (R - 1);
  const int grp = (int(threadIdx.x) >> 5) * G + lane / R;
  const int rr = min(r0 + grp, NSR - 1);  // a group past the plane's last row repeats it, stores nothing
  const double2* zr = in + (size_t(p) * NSR + rr) * NSR;
  double2* xs = wsm + grp * kDstTileStage + (grp & 7);
  const double scale = 0.088388347648318440550;  // sqrt(2/256)
  warp_dst256([&](int j) { return zr[j - 1]; }, xs, t, twb, scale);
  if constexpr (MODE != 0) {
    const double2 l = __ldg(lam + p);
    const double* sg = sigT + size_t(rr) * NSR;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = t + R * r;
      if (i < NSR) xs[dst_slot(i)] = shift_apply<MODE>(xs[dst_slot(i)], l.x - dt * __ldg(sg + i), l.y);
    }
    __syncwarp();
    warp_dst256([&](int j) { return xs[dst_slot(j - 1)]; }, xs, t, twb, scale);
  }
  __syncthreads();
  const int g = int(threadIdx.x) % NG, c0 = int(threadIdx.x) / NG;
  if (r0 + g < NSR) {
    const double2* src = wsm + g * kDstTileStage + (g & 7);
    double2* oc = out + size_t(p) * NSR * NSR + r0 + g;
#pragma unroll
    for (int u = 0; u < (NSR + 15) / 16; ++u) {
      const int c = c0 + 16 * u;
      if (c < NSR) oc[size_t(c) * NSR] = src[dst_slot(c)];
    }
  }
}

// mode 0: out = transpose(DST rows of in); 1 / 2: out = transpose(DST, shift (solve / forward), DST)
cudaError_t launch_dst_rows_T(const double2* in, double2* out, int n, int n_planes, const double2* lambda,
                              const double* sigma, double dt, const double2* tw_base, cudaStream_t st, int mode) {
  if (n != 255) return cudaErrorNotSupported;
  const size_t smem = size_t(8) * kDstTileStage * sizeof(double2);
  const unsigned grid = unsigned(n_planes) * 32u;
  const double* sigT = sigma ? sigma + size_t(255) * 255 : nullptr;
  cudaError_t e = cudaSuccess;
#define FPC_DSTT(MODE)                                                                                         \
  {                                                                                                            \
    if ((e = cudaFuncSetAttribute(k_dst_rows_T<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) \
        != cudaSuccess)                                                                                        \
      return e;                                                                                                \
    k_dst_rows_T<MODE><<<grid, 128, smem, st>>>(in, out, lambda, sigT, dt, tw_base);                           \
    note_launch();                                                                                             \
  }
  if (mode == 0)
    FPC_DSTT(0)
  else if (mode == 1)
    FPC_DSTT(1)
  else
    FPC_DSTT(2)
#undef FPC_DSTT
  return cudaGetLastError();
}

cudaError_t launch_tau_cols_warp(double2* Z, int n, int n_planes, const double2* lambda, const double* sigma,
                                 double dt, const double2* tw_base, cudaStream_t st, bool forward) {
  if (n != 255) return cudaErrorNotSupported;
  constexpr int NG = kTauColWarps * 2;
  const unsigned grid = unsigned(n_planes) * unsigned((255 + NG - 1) / NG);
  cudaError_t e = cudaSuccess;
  // FPC_TAU_COLS_STAGED=1: the staged kernel (A/B).  Measured at config 2: 0.551 ms per tau solve in
  // 8-warp CTAs, 0.525 in 4-warp CTAs, against 0.528-0.532 direct -- at n = 255 the CTA barriers cost
  // what the saved wavefronts gain (the n = 1023 kernels, one element of 32 rows per direct
  // instruction, do gain: kernels_warp32.cu)
  static const bool staged = [] {
    const char* v = std::getenv("FPC_TAU_COLS_STAGED");
    return v && v[0] == '1';
  }();
  if (staged) {
    constexpr int NGS = kTauStWarps * 2;
    const size_t smem = size_t(NGS) * kDstTileStage * sizeof(double2);
    const unsigned grid = unsigned(n_planes) * unsigned((255 + NGS - 1) / NGS);
    if (forward) {
      if ((e = cudaFuncSetAttribute(k_tau_cols_staged<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
          cudaSuccess)
        return e;
      if ((e = set_warp_carveout((const void*)k_tau_cols_staged<2>, smem)) != cudaSuccess) return e;
      k_tau_cols_staged<2><<<grid, 32 * kTauStWarps, smem, st>>>(Z, n_planes, lambda, sigma, dt, tw_base);
    } else {
      if ((e = cudaFuncSetAttribute(k_tau_cols_staged<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
          cudaSuccess)
        return e;
      if ((e = set_warp_carveout((const void*)k_tau_cols_staged<1>, smem)) != cudaSuccess) return e;
      k_tau_cols_staged<1><<<grid, 32 * kTauStWarps, smem, st>>>(Z, n_planes, lambda, sigma, dt, tw_base);
    }
    note_launch();
    return cudaGetLastError();
  }
  const size_t smem = size_t(NG) * kDstTileSize * sizeof(double2);
  if (forward) {
    if ((e = cudaFuncSetAttribute(k_tau_cols_warp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
        cudaSuccess)
      return e;
    if ((e = set_warp_carveout((const void*)k_tau_cols_warp<2>, smem)) != cudaSuccess) return e;
    k_tau_cols_warp<2><<<grid, 32 * kTauColWarps, smem, st>>>(Z, n_planes, lambda, sigma, dt, tw_base);
  } else {
    if ((e = cudaFuncSetAttribute(k_tau_cols_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
        cudaSuccess)
      return e;
    if ((e = set_warp_carveout((const void*)k_tau_cols_warp<1>, smem)) != cudaSuccess) return e;
    k_tau_cols_warp<1><<<grid, 32 * kTauColWarps, smem, st>>>(Z, n_planes, lambda, sigma, dt, tw_base);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace fpc
