// warp_dst.cuh -- orthonormal DST-I of one complex row of n = 255 points (N = n + 1 = 256) owned by
// a group of 16 lanes (warp_fft.cuh), for the 2D lattice rows of config 2 (tau.hpp:79-96 row pass)
// and the 1D tau solves at n = 255 (tau.hpp:98-119).
//
// Same split as dst_block.cuh (no recurrences; the reference's accuracy): with M = N/2,
//   y_0 = 0, y_j = sin(pi j/N)(f_j + f_{N-j}) + (f_j - f_{N-j})/2,    Y = FFT_N^+(y)
//     F_{2k} = -(i/2)(Y_k - Y_{N-k})                                   k = 1..M-1
//   s_j = f_j + f_{N-j} (j < M), s_M = f_M, t_k = s_{M-k},
//   V_0 = t_0, V_k = (1/2) e^{i pi k/N} (t_k - i t_{M-k}),            v = FFT_M^+(V)
//     F_{2k+1} = (-1)^k x_k, x_{2m} = v_m, x_{2m+1} = v_{M-1-m}        k = 0..M-1
//   DST(f)_i = sqrt(2/N) F_{i+1}
// Layouts: the 256-point transform is warp_fft_sq<16> (lane t holds y_{t+16r}, 16 registers); the
// 128-point one is warp_fft_8x16 below (lane t holds V_{t+16r}, 8 registers).  Every f the lane
// needs is read from the source functor in the pre-phase (global row or the group's tile), so the
// tile is free for the transposes; the outputs are assembled in natural order in the tile.
#pragma once
#include "warp_fft.cuh"

#ifndef FPC_DST_SHFL
#define FPC_DST_SHFL 1
#endif

namespace fpc {

// 128-point transform by 16 lanes, 8 values each: lane t holds x[t + 16 r] (r < 8) on entry and
// X[t + 16 p] (p < 8) on exit.  k = q + 8 p' (q < 8, p' < 16): pass A = DFT_8 over r + twiddle
// w_128^{t q}, transpose (tile row q = the 16 lanes' values), pass B = DFT_16 over t split into its
// even/odd output halves: lane L = q + 8h forms (B_{t0} +- B_{t0+8}) (x w_16^{t0} for h = 1) and runs
// one DFT_8, giving X_{q + 8(2p'' + h)} = X_{L + 16 p''}.
template <int S>
__device__ __forceinline__ void warp_fft_8x16(double2 (&v)[8], double2* __restrict__ xs, int t,
                                              const double2* __restrict__ twb) {
  constexpr int LD = WarpFftTile<16>::LD;
  Dft<8, S>::run(v);
  apply_twiddles<8, S>(v, twb + 128, twb + 32, t);  // v[q] *= w_128^{S t q}
#pragma unroll
  for (int q = 0; q < 8; ++q) xs[q * LD + t] = v[q];
  __syncwarp();
  const int q = t & 7, h = t >> 3;
  double2 b[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) b[u] = xs[q * LD + u];
  __syncwarp();
#pragma unroll
  for (int t0 = 0; t0 < 8; ++t0) {
    const double2 d = h ? csub(b[t0], b[t0 + 8]) : cadd(b[t0], b[t0 + 8]);
    if (h == 0 || t0 == 0) {
      v[t0] = d;
    } else {  // d * w_16^{S t0}
      const double c = kC16[t0], sn = S * kC16[(t0 + 12) & 15];
      v[t0] = make_double2(fma(d.x, c, -d.y * sn), fma(d.x, sn, d.y * c));
    }
  }
  Dft<8, S>::run(v);
}

// Output slot of DST index i in the group's tile: i + i/8, so the stride-2 and stride-4 scatter
// of the assembly and the unit-stride read-back are all free of 16-byte bank conflicts.  The tile
// needs kDstTileSize >= dst_slot(254) + 1 double2.
__device__ __forceinline__ int dst_slot(int i) { return i + (i >> 3); }
constexpr int kDstTileSize = 288;

// DST of one row: f(j) returns f_j (j = 1..255, complex).  On return the group's tile holds
// DST(f)_i * scale at tile slot dst_slot(i) (i = 0..254); the caller reads it back after a
// __syncwarp (index t + 16 r is lane t's r-th coalesced output).  A tile-backed source may use the
// same layout (f(j) = xs[dst_slot(j - 1)]): every f is read before the first transpose.
template <class Src>
__device__ __forceinline__ void warp_dst256(Src f, double2* __restrict__ xs, int t, const double2* __restrict__ twb,
                                            double scale) {
  constexpr int N = 256, M = 128;
  const double2* tw2N = twb + 2 * N;  // e^{-i pi j/N}
  double2 y[16], V[8], slo[8];
  // pre-phase: y_j (j = t + 16 r) and V_k (k = t + 16 r, r < 8).  s_k = f_k + f_{N-k} is this lane's
  // s at r, and s_{M-k} = f_{M-k} + f_{M+k} is its s at r + 8 (M + k = t + 16(r + 8)), so V needs no
  // further loads; V_0 = s_M = f_M = (2 f_M)/2 with the j = M term.
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int j = t + 16 * r;
    double2 sj = make_double2(0.0, 0.0);
    if (j == 0) {
      y[r] = sj;
    } else {
      const double2 f1 = f(j), f2 = f(N - j);
      sj = cadd(f1, f2);
      const double2 dj = csub(f1, f2);
      const double sinj = -__ldg(tw2N + j).y;
      y[r] = make_double2(fma(sinj, sj.x, 0.5 * dj.x), fma(sinj, sj.y, 0.5 * dj.y));
    }
    if (r < 8) {
      slo[r] = sj;
    } else {
      const int k = j - M;  // = t + 16 (r - 8)
      if (k == 0) {
        V[r - 8] = cscale(sj, 0.5);
      } else {
        const double2 wk = __ldg(tw2N + k);  // e^{-i pi k/N}
        V[r - 8] = cscale(cmul(cconj(wk), csub(sj, mul_si<1>(slo[r - 8]))), 0.5);
      }
    }
  }
  __syncwarp();  // a tile-backed source has been read completely
  warp_fft_sq<16, 1>(y, xs, t, twb);  // lane t: Y_{t + 16 p}
  // even outputs F_{2k} = -(i/2)(Y_k - Y_{N-k}), k = t + 16 p (p < 8, k >= 1): the mirror N - k sits
  // in lane (16 - t) mod 16, register 15 - p (t != 0), or this lane's register 16 - p (t = 0)
  double2 ev[8];
#if FPC_DST_SHFL
  {
    double2 ym[8];
    ym[0] = warp_fft_mirror<16, 0>(y, t); ym[1] = warp_fft_mirror<16, 1>(y, t);
    ym[2] = warp_fft_mirror<16, 2>(y, t); ym[3] = warp_fft_mirror<16, 3>(y, t);
    ym[4] = warp_fft_mirror<16, 4>(y, t); ym[5] = warp_fft_mirror<16, 5>(y, t);
    ym[6] = warp_fft_mirror<16, 6>(y, t); ym[7] = warp_fft_mirror<16, 7>(y, t);
#pragma unroll
    for (int p = 0; p < 8; ++p) ev[p] = make_double2(0.5 * (y[p].y - ym[p].y), -0.5 * (y[p].x - ym[p].x));
  }
#else
  constexpr int LD = WarpFftTile<16>::LD;
#pragma unroll
  for (int p = 0; p < 16; ++p) xs[p * LD + t] = y[p];
  __syncwarp();
  const int tm = (16 - t) & 15;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int pm = t == 0 ? ((16 - p) & 15) : (15 - p);
    const double2 ym = xs[pm * LD + tm];
    ev[p] = make_double2(0.5 * (y[p].y - ym.y), -0.5 * (y[p].x - ym.x));
  }
  __syncwarp();
#endif
  warp_fft_8x16<1>(V, xs, t, twb);  // lane t: v_{t + 16 p}
  // assemble DST(f)_i = scale F_{i+1} in natural order: F_{2k} -> i = 2k - 1; v_m -> i = 4m (m < 64)
  // or -v_m -> i = 510 - 4m (m >= 64)
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int k = t + 16 * p;
    if (k >= 1) xs[dst_slot(2 * k - 1)] = cscale(ev[p], scale);
    const int m = k;
    if (m < M / 2)
      xs[dst_slot(4 * m)] = cscale(V[p], scale);
    else
      xs[dst_slot(510 - 4 * m)] = cscale(V[p], -scale);
  }
  __syncwarp();
}

}  // namespace fpc
