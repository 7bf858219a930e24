// kernels_warp32.cu -- lattice kernels for n = 1023 (M = 1024) on warp-owned 1024-point register
// transforms (warp_fft32.cuh): the rows and columns of BASELINE config 3 (2D 1023^2 x 1024), and 1D
// rows of 513..1023 points.  One row / column per warp, 32 lanes x 32 complex registers, one
// shared-memory transpose per transform, no CTA barrier inside a transform.
//
// Rows matvec (all_at_once.hpp:33-55 + toeplitz.hpp:41-57 along contiguous rows; the 2D
// y-direction half of jacobian.hpp:84-87) and the x-direction column pass (jacobian.hpp:88-93).
#include <cstdlib>

#include "bulk_copy.cuh"
#include "kernels.cuh"
#include "warp_dst32.cuh"
#include "warp_fft32.cuh"

namespace fpc {

namespace {

#ifndef FPC_W32_ROWW
#define FPC_W32_ROWW 4
#endif
constexpr int kW32Warps = FPC_W32_ROWW;  // matvec rows: warps per CTA; 8 warps per SM (255 registers per thread)
// DST rows: one warp per CTA -- a 4-warp CTA's slots stay empty until its slowest warp is done (tau
// solve at 1023^2 x 64: 1.40 ms in 4-warp CTAs, 1.24 in 2-warp, 1.21 in 1-warp; the matvec rows, with
// their three row loads up front, measured the other way: 1.495 / 1.507 / 1.558 ms)
#ifndef FPC_W32_DSTW
#define FPC_W32_DSTW 1
#endif
constexpr int kW32DstWarps = FPC_W32_DSTW;
// column kernels: warps (= adjacent columns) per CTA, 8 warps per SM either way (build knobs, A/B on
// 1023^2 x 64): the matvec columns (8-byte elements) gain from 64-byte row segments with 8 columns
// (844 -> 750 us), the tau columns (16-byte elements, 64-byte segments already) lose the overlap of
// two CTAs' staging phases (1.41 -> 1.47 ms per tau solve)
#ifndef FPC_W32_MV_COLW
#define FPC_W32_MV_COLW 8
#endif
#ifndef FPC_W32_TAU_COLW
#define FPC_W32_TAU_COLW 4
#endif
constexpr int kW32MvColWarps = FPC_W32_MV_COLW, kW32TauColWarps = FPC_W32_TAU_COLW;
static_assert((kW32MvColWarps == 4 || kW32MvColWarps == 8) &&
                  (kW32TauColWarps == 2 || kW32TauColWarps == 4 || kW32TauColWarps == 8),
              "column kernels: 4 or 8 (tau: 2, 4 or 8) columns per CTA");

__device__ __forceinline__ double bdf2_w32(int k, double x0, double x1, double x2) {
  if (k == 0) return x0;
  if (k == 1) return 1.5 * x0 + -2.0 * x1;
  return 1.5 * x0 + -2.0 * x1 + 0.5 * x2;
}

// Shared-memory carveout for 8 warps per SM in CTAs of `warps` warps: the smallest capacity that
// holds them (dynamic + the 1 KB system reserve per CTA), the rest of the 256 KB array stays L1 for
// the twiddle / eigenvalue tables.  The driver takes the smallest capacity >= pct% of 228 KB, so the
// percentage is rounded down (kernels_krylov.cu carveout_pct).
cudaError_t prep_w32(const void* kernel, size_t smem, int warps = kW32Warps) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const size_t need = size_t(8 / warps) * (smem + 1024);
  int pct = 100;
  for (int c : {8, 16, 32, 64, 100, 132, 164, 196, 228})
    if (size_t(c) * 1024 >= need) {
      pct = (c * 100) / 228;
      break;
    }
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

}  // namespace

bool warp32_kernels_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPC_W32");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Smallest row count the row kernels take (one warp per row: below a wave of 8 warps per SM the
// CTA-level kernels, which spread a row over a CTA, keep more SMs busy; measured on 1D 1023 x n_time:
// ahead from ~1000 rows, behind at 513).  FPC_W32_MIN_ROWS overrides.
int warp32_min_rows() {
  static const int v = [] {
    const char* e = std::getenv("FPC_W32_MIN_ROWS");
    return (e && e[0]) ? std::atoi(e) : 1000;
  }();
  return v;
}

// One row of ns <= 1023 reals per warp.  The BDF2 stencil part of the row (three rows of v) is
// formed first and parked in shared memory (one double per (lane, slot): conflict free) so that the
// 128 data registers of the transforms are all that is live across them.
__global__ void __launch_bounds__(32 * kW32Warps, 8 / kW32Warps)
    k_mv_rows_w32(const double* __restrict__ v, double* __restrict__ y, int ns, int nrows, int rpt, int sstride,
                  int koff, const double* __restrict__ eig, const double2* __restrict__ twb) {
  constexpr int R = 32, M = 1024, L = 2 * M, H = 16;
  extern __shared__ double2 wsm[];
  const int t = int(threadIdx.x) & 31;
  const int w = int(threadIdx.x) >> 5;
  const int row = int(blockIdx.x) * kW32Warps + w;
  if (row >= nrows) return;  // warps are independent: no CTA barrier below
  const int k = row / rpt + koff;
  const double* vr = v + size_t(row) * ns;
  double2* xs = wsm + w * kW32Tile;
  double* cs = reinterpret_cast<double*>(wsm + kW32Warps * kW32Tile) + w * (2 * H * 32);

  // packed slot m = t + 32 r holds (x_{2m}, x_{2m+1}); slots with 2m >= ns are the zero padding
  double2 z[R];
#pragma unroll
  for (int r = 0; r < H; ++r) {
    const int i0 = 2 * (t + R * r);
    z[r] = make_double2(i0 < ns ? __ldcg(vr + i0) : 0.0, i0 + 1 < ns ? __ldcg(vr + i0 + 1) : 0.0);
  }
#pragma unroll
  for (int r = H; r < R; ++r) z[r] = make_double2(0.0, 0.0);
  {
    double x1[2 * H], x2[2 * H];
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const int i0 = 2 * (t + R * r);
      const bool ok0 = i0 < ns, ok1 = i0 + 1 < ns;
      x1[2 * r] = (ok0 && k >= 1) ? __ldcg(vr + (i0 - sstride)) : 0.0;
      x1[2 * r + 1] = (ok1 && k >= 1) ? __ldcg(vr + (i0 + 1 - sstride)) : 0.0;
      x2[2 * r] = (ok0 && k >= 2) ? __ldcg(vr + i0 - 2 * size_t(sstride)) : 0.0;
      x2[2 * r + 1] = (ok1 && k >= 2) ? __ldcg(vr + i0 + 1 - 2 * size_t(sstride)) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < H; ++r) {
      cs[(2 * r) * 32 + t] = bdf2_w32(k, z[r].x, x1[2 * r], x2[2 * r]);
      cs[(2 * r + 1) * 32 + t] = bdf2_w32(k, z[r].y, x1[2 * r + 1], x2[2 * r + 1]);
    }
  }
  warp_fft_1024<-1, true, false>(z, xs, t, twb);
  warp_packed_product_1024(z, t, eig, twb + L);
  warp_fft_1024<1, false, true>(z, xs, t, twb);
  double* yr = y + size_t(row) * ns;
#pragma unroll
  for (int r = 0; r < H; ++r) {
    const int i0 = 2 * (t + R * r);
    if (i0 < ns) yr[i0] = cs[(2 * r) * 32 + t] + z[r].x;
    if (i0 + 1 < ns) yr[i0 + 1] = cs[(2 * r + 1) * 32 + t] + z[r].y;
  }
}

cudaError_t launch_matvec_rows_w32(const double* v, double* y, int len, int nrows, int rpt, int sstride,
                                   const double* eig_scaled, const double2* tw_base, cudaStream_t st, int koff) {
  const size_t smem = size_t(kW32Warps) * (kW32Tile * sizeof(double2) + 32 * 32 * sizeof(double));
  cudaError_t e = prep_w32((const void*)k_mv_rows_w32, smem);
  if (e != cudaSuccess) return e;
  k_mv_rows_w32<<<(nrows + kW32Warps - 1) / kW32Warps, 32 * kW32Warps, smem, st>>>(v, y, len, nrows, rpt, sstride,
                                                                                  koff, eig_scaled, tw_base);
  note_launch();
  return cudaGetLastError();
}

// x-direction column pass of the 2D matvec for n <= 1023: y[k][ix][iy] += (T_x v[k][.][iy])[ix].
// A CTA owns C = kW32MvColWarps adjacent columns of one time level, one per warp.  The column tile is
// staged through the warps' own transpose tiles (free before the first transform and after the
// last): the CTA copies row segments of C doubles (32 / C rows per warp instruction, instead of one
// element of 32 different rows) and column c lands in warp c's tile; the results go back the same way
// and are added to y as L2 reductions (RED.ADD.F64: each element receives exactly one add, so the
// sum is the same double as load-add-store).
__global__ void __launch_bounds__(32 * kW32MvColWarps, 8 / kW32MvColWarps)
    k_mv_cols_w32(const double* __restrict__ v, double* __restrict__ y, int n, const double* __restrict__ eig,
                  const double2* __restrict__ twb) {
  constexpr int R = 32, M = 1024, L = 2 * M, H = 16, C = kW32MvColWarps, NT = 32 * kW32MvColWarps;
  constexpr int CP = 2 * kW32Tile;  // doubles per warp tile (2112)
  // staged column of warp c: element ix = 2 m + h (packed slot m = tt + 32 r) at (2 r + h) * SH + tt,
  // shifted by c * SC: a lane's reads are unit stride over tt, and a staging instruction spreads over
  // all sixteen 8-byte banks twice (C = 4: 8 rows = 4 m x 2 h per column, m: 0..3, h: +4, c: +8 mod 16;
  // C = 8: 4 rows = 2 m x 2 h per column, c: +2 mod 16)
  constexpr int SH = 36, SC = C == 4 ? 8 : 2;
  static_assert(31 * SH + 32 + (C - 1) * SC <= CP, "staged column fits the tile");
  extern __shared__ double2 wsm[];
  double* tiles = reinterpret_cast<double*>(wsm);
  const int ntile = (n + C - 1) / C;
  const int k = int(blockIdx.x) / ntile;
  const int iy0 = (int(blockIdx.x) - k * ntile) * C;
  const size_t base = size_t(k) * size_t(n) * size_t(n) + iy0;
  const int ncol = min(C, n - iy0);
  const int t = int(threadIdx.x) & 31;
  const int w = int(threadIdx.x) >> 5;
  // 1. stage: thread tid copies column c = tid % C of rows ix = tid / C + u (NT / C)
  {
    const int c = int(threadIdx.x) % C, ix0 = int(threadIdx.x) / C;
    constexpr int RS = NT / C;  // rows per sweep (32)
    const bool okc = c < ncol;
    double* dst = tiles + c * CP + c * SC;
    const double* vb = v + base + (okc ? c : 0);
#pragma unroll 8
    for (int ix = ix0; ix < M; ix += RS) {
      const bool ok = okc && ix < n;
      const int m = ix >> 1, h = ix & 1;
      cp_async8_zfill(dst + ((m >> 5) * 2 + h) * SH + (m & 31), vb + size_t(ok ? ix : 0) * n, ok);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  double* mine = tiles + w * CP + w * SC;
  double2* xs = wsm + w * kW32Tile;
  double2 z[R];
#pragma unroll
  for (int r = 0; r < H; ++r) z[r] = make_double2(mine[(2 * r) * SH + t], mine[(2 * r + 1) * SH + t]);
#pragma unroll
  for (int r = H; r < R; ++r) z[r] = make_double2(0.0, 0.0);
  __syncwarp();
  warp_fft_1024<-1, true, false>(z, xs, t, twb);
  warp_packed_product_1024(z, t, eig, twb + L);
  warp_fft_1024<1, false, true>(z, xs, t, twb);
#pragma unroll
  for (int r = 0; r < H; ++r) {
    mine[(2 * r) * SH + t] = z[r].x;
    mine[(2 * r + 1) * SH + t] = z[r].y;
  }
  __syncthreads();
  {
    const int c = int(threadIdx.x) % C, ix0 = int(threadIdx.x) / C;
    constexpr int RS = NT / C;
    const bool okc = c < ncol;
    const double* src = tiles + c * CP + c * SC;
#pragma unroll 8
    for (int ix = ix0; ix < n; ix += RS) {
      const int m = ix >> 1, h = ix & 1;
      const double r = src[((m >> 5) * 2 + h) * SH + (m & 31)];
      if (okc) atomicAdd(y + base + size_t(ix) * n + c, r);
    }
  }
}

cudaError_t launch_matvec_cols_w32(const double* v, double* y, int n, int n_time, const double* eig_x,
                                   const double2* tw_base, cudaStream_t st) {
  const size_t smem = size_t(kW32MvColWarps) * kW32Tile * sizeof(double2);
  cudaError_t e = prep_w32((const void*)k_mv_cols_w32, smem, kW32MvColWarps);
  if (e != cudaSuccess) return e;
  const unsigned grid = unsigned(n_time) * unsigned((n + kW32MvColWarps - 1) / kW32MvColWarps);
  k_mv_cols_w32<<<grid, 32 * kW32MvColWarps, smem, st>>>(v, y, n, eig_x, tw_base);
  note_launch();
  return cudaGetLastError();
}

// DST-I rows of n = 1023 complex points, one row per warp, in place: MODE 0 = the row DSTs of the
// 2D tau solve (tau.hpp:85-86); MODE 1 / 2 = the 1D tau solve / forward action of frequency row r
// (tau.hpp:98-136): DST, divide (multiply) by lambda_r - dt sigma_i, DST, the intermediate kept in
// the warp's tile.
template <int MODE>
__global__ void __launch_bounds__(32 * kW32DstWarps, 8 / kW32DstWarps)
    k_dst_rows_w32(double2* __restrict__ Z, int n_rows, const double2* __restrict__ lam,
                   const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  constexpr int NSR = 1023;
  extern __shared__ double2 wsm[];
  const int t = int(threadIdx.x) & 31;
  const int w = int(threadIdx.x) >> 5;
  const int row = int(blockIdx.x) * kW32DstWarps + w;
  if (row >= n_rows) return;
  double2* zr = Z + size_t(row) * NSR;
  double2* xs = wsm + w * kDst32Tile;
  const double scale = 0.044194173824159220275;  // sqrt(2/1024)
  warp_dst1024([&](int j) { return __ldcg(zr + (j - 1)); }, xs, t, twb, scale);
  if constexpr (MODE != 0) {
    const double2 l = __ldg(lam + row);
    double sv[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) sv[r] = __ldg(sigma + min(t + 32 * r, NSR - 1));
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int i = t + 32 * r;
      if (i < NSR) xs[dst32_slot(i)] = shift_apply<MODE>(xs[dst32_slot(i)], l.x - dt * sv[r], l.y);
    }
    __syncwarp();
    warp_dst1024([&](int j) { return xs[dst32_slot(j - 1)]; }, xs, t, twb, scale);
  }
#pragma unroll 8
  for (int r = 0; r < 32; ++r) {
    const int i = t + 32 * r;
    if (i < NSR) zr[i] = xs[dst32_slot(i)];
  }
}

cudaError_t launch_dst_rows_w32(double2* Z, int n, int n_rows, const double2* lambda, const double* sigma,
                                double dt, const double2* tw_base, cudaStream_t st, int mode) {
  if (n != 1023) return cudaErrorNotSupported;
  const size_t smem = size_t(kW32DstWarps) * kDst32Tile * sizeof(double2);
  const unsigned grid = unsigned((n_rows + kW32DstWarps - 1) / kW32DstWarps);
  cudaError_t e = cudaSuccess;
#define FPC_DSTW32(MODE)                                                                               \
  {                                                                                                    \
    if ((e = prep_w32((const void*)k_dst_rows_w32<MODE>, smem, kW32DstWarps)) != cudaSuccess) return e;              \
    k_dst_rows_w32<MODE><<<grid, 32 * kW32DstWarps, smem, st>>>(Z, n_rows, lambda, sigma, dt, tw_base);   \
    note_launch();                                                                                     \
  }
  if (mode == 0)
    FPC_DSTW32(0)
  else if (mode == 1)
    FPC_DSTW32(1)
  else
    FPC_DSTW32(2)
#undef FPC_DSTW32
  return cudaGetLastError();
}

// 2D tau solve, column pass (tau.hpp:79-119 along ix) for n = 1023: for frequency plane rp and column
// iy, DST over ix, divide (MODE 1) / multiply (MODE 2) by lambda_rp - dt sigma[ix n + iy], DST over ix,
// in place.  A CTA owns kW32Warps adjacent columns, one per warp; the columns are staged through the
// warps' tiles (row segments of kW32Warps complex values: 8 rows per warp instruction) in the DST's
// own slot layout, each tile shifted by 2 c slots so a staging instruction's 4 columns x 2 rows per
// quarter warp hit 8 different 16-byte banks.  sigma = the plan's table [ix][iy] followed by its
// transpose [iy][ix] (read here: contiguous in ix).
template <int MODE>
__global__ void __launch_bounds__(32 * kW32TauColWarps, 8 / kW32TauColWarps)
    k_tau_cols_w32(double2* __restrict__ Z, const double2* __restrict__ lam, const double* __restrict__ sigma,
                   double dt, const double2* __restrict__ twb) {
  constexpr int NSR = 1023, C = kW32TauColWarps, NT = 32 * kW32TauColWarps, RS = NT / C, SK = 8 / C;
  extern __shared__ double2 wsm[];
  constexpr int ntile = (NSR + C - 1) / C;
  const int rp = int(blockIdx.x) / ntile;
  const int iy0 = (int(blockIdx.x) - rp * ntile) * C;
  const int ncol = min(C, NSR - iy0);
  double2* zb = Z + size_t(rp) * NSR * NSR + iy0;
  const int t = int(threadIdx.x) & 31;
  const int w = int(threadIdx.x) >> 5;
  const int c = int(threadIdx.x) % C, ix0 = int(threadIdx.x) / C;
  const bool okc = c < ncol;
  {
    double2* dst = wsm + c * kDst32Tile + SK * c;
    const double2* zc = zb + (okc ? c : 0);
#pragma unroll 8
    for (int ix = ix0; ix < NSR; ix += RS) cp_async16_zfill(dst + dst32_slot(ix), zc + size_t(ix) * NSR, okc);
    cp_async_wait_all();
  }
  __syncthreads();
  double2* xs = wsm + w * kDst32Tile + SK * w;
  const double scale = 0.044194173824159220275;  // sqrt(2/1024)
  // DST, shift, DST: one copy of the transform code (the unrolled DST is ~10K instructions)
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    warp_dst1024([&](int j) { return xs[dst32_slot(j - 1)]; }, xs, t, twb, scale);
    if (pass == 0) {
      const double2 l = __ldg(lam + rp);
      const int iy = min(iy0 + w, NSR - 1);
      const double* sg = sigma + size_t(NSR) * NSR + size_t(iy) * NSR;  // transposed table: row iy
      // the column's 32 sigma values per lane in flight together (L2 latency paid once)
      double sv[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) sv[r] = __ldg(sg + min(t + 32 * r, NSR - 1));
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int i = t + 32 * r;
        if (i < NSR) xs[dst32_slot(i)] = shift_apply<MODE>(xs[dst32_slot(i)], l.x - dt * sv[r], l.y);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (okc) {
    const double2* src = wsm + c * kDst32Tile + SK * c;
#pragma unroll 8
    for (int ix = ix0; ix < NSR; ix += RS) zb[size_t(ix) * NSR + c] = src[dst32_slot(ix)];
  }
}

cudaError_t launch_tau_cols_w32(double2* Z, int n, int n_planes, const double2* lambda, const double* sigma,
                                double dt, const double2* tw_base, cudaStream_t st, bool forward) {
  if (n != 1023) return cudaErrorNotSupported;
  const size_t smem = size_t(kW32TauColWarps) * kDst32Tile * sizeof(double2);
  const unsigned grid = unsigned(n_planes) * unsigned((1023 + kW32TauColWarps - 1) / kW32TauColWarps);
  cudaError_t e = cudaSuccess;
  if (forward) {
    if ((e = prep_w32((const void*)k_tau_cols_w32<2>, smem, kW32TauColWarps)) != cudaSuccess) return e;
    k_tau_cols_w32<2><<<grid, 32 * kW32TauColWarps, smem, st>>>(Z, lambda, sigma, dt, tw_base);
  } else {
    if ((e = prep_w32((const void*)k_tau_cols_w32<1>, smem, kW32TauColWarps)) != cudaSuccess) return e;
    k_tau_cols_w32<1><<<grid, 32 * kW32TauColWarps, smem, st>>>(Z, lambda, sigma, dt, tw_base);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace fpc
