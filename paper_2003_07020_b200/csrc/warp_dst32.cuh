// warp_dst32.cuh -- orthonormal DST-I of one complex row of n = 1023 points (N = 1024) owned by one
// warp (warp_fft32.cuh), for the 2D lattice rows and columns of config 3 (tau.hpp:79-96) and the 1D
// tau solves at n = 1023 (tau.hpp:98-119).
//
// The split of dst_block.cuh / warp_dst.cuh (no recurrences; the reference's accuracy), M = N/2:
//   y_0 = 0, y_j = sin(pi j/N)(f_j + f_{N-j}) + (f_j - f_{N-j})/2,    Y = FFT_N^+(y)
//     F_{2k} = -(i/2)(Y_k - Y_{N-k})                                   k = 1..M-1
//   s_j = f_j + f_{N-j} (j < M), s_M = f_M,
//   V_0 = s_M, V_k = (1/2) e^{i pi k/N} (s_{M-k} - i s_k),             v = FFT_M^+(V)
//     F_{4m+1} = v_m (m < M/2), F_{4M-4m-1} = -v_m (m >= M/2)
//   DST(f)_i = sqrt(2/N) F_{i+1}
// Lane t holds y_{t+32r} (32 registers) and V_{t+32r} (r < 16): the pair (r, r + 16) of y needs
// f_j, f_{N-j} at j = t + 32 r and j + M, whose sums are exactly s_k and s_{M-k} of V_k, k = j.
// The 512-point transform of V is a 16 x 32 scheme on the same tile.
#pragma once
#include "warp_fft32.cuh"

namespace fpc {

// 512-point transform by 32 lanes, 16 values each: lane t holds x[t + 32 r] (r < 16) on entry and
// X[t + 32 p] (p < 16) on exit.  k = q + 16 p' (q < 16, p' < 32): pass A = DFT_16 over r + twiddle
// w_512^{t q}, transpose (tile row q = the 32 lanes' values), pass B = DFT_32 over t split by output
// parity: lane L = q + 16 h forms b_{t0} +- b_{t0+16} (x w_32^{t0} for h = 1) and runs one DFT_16,
// giving X_{q + 16 (2 p'' + h)} = X_{L + 32 p''}.
template <int S>
__device__ __forceinline__ void warp_fft_16x32(double2 (&v)[16], double2* __restrict__ xs, int t,
                                               const double2* __restrict__ twb) {
  constexpr int LD = kW32LD;
  Dft<16, S>::run(v);
  apply_twiddles<16, S>(v, twb + 512, twb + 128, t);  // v[q] *= w_512^{S t q}
#pragma unroll
  for (int q = 0; q < 16; ++q) xs[q * LD + t] = v[q];
  __syncwarp();
  const int q = t & 15;
  const bool h = t >= 16;
#pragma unroll
  for (int t0 = 0; t0 < 16; ++t0) {
    const double2 b0 = xs[q * LD + t0], b1 = xs[q * LD + t0 + 16];
    const double2 d = h ? csub(b0, b1) : cadd(b0, b1);
    const double2 dr = rot32<S>(d, t0);
    v[t0] = h ? dr : d;
  }
  __syncwarp();
  Dft<16, S>::run(v);
}

// Output slot of DST index i in the warp's tile: i + i/8 (the stride-2 and stride-4 scatters of the
// assembly and the unit-stride read-back are free of 16-byte bank conflicts).
__device__ __forceinline__ int dst32_slot(int i) { return i + (i >> 3); }
constexpr int kDst32Tile = 1160;  // >= dst32_slot(1022) + 1 = 1150, and >= kW32Tile = 1056; + skew room

// DST of one row: f(j) returns f_j (j = 1..1023).  On return the warp's tile holds DST(f)_i * scale
// at slot dst32_slot(i); the caller reads it back after the trailing __syncwarp.  A tile-backed
// source may use the same layout: every f is read before the first transpose.
template <class Src>
__device__ __forceinline__ void warp_dst1024(Src f, double2* __restrict__ xs, int t, const double2* __restrict__ twb,
                                             double scale) {
  constexpr int N = 1024, M = 512;
  const double2* tw2N = twb + 2 * N;  // e^{-i pi j/N}
  double2 y[32], V[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int j = t + 32 * r;  // < M
    const int j2 = j + M;
    double2 slo = make_double2(0.0, 0.0);
    if (j == 0) {
      y[r] = slo;
    } else {
      const double2 f1 = f(j), f2 = f(N - j);
      slo = cadd(f1, f2);
      const double2 dj = csub(f1, f2);
      const double sinj = -__ldg(tw2N + j).y;
      y[r] = make_double2(fma(sinj, slo.x, 0.5 * dj.x), fma(sinj, slo.y, 0.5 * dj.y));
    }
    const double2 g1 = f(j2), g2 = f(N - j2);
    const double2 shi = cadd(g1, g2), dh = csub(g1, g2);
    const double sinh_ = -__ldg(tw2N + j2).y;
    y[r + 16] = make_double2(fma(sinh_, shi.x, 0.5 * dh.x), fma(sinh_, shi.y, 0.5 * dh.y));
    if (j == 0) {
      V[r] = cscale(shi, 0.5);
    } else {
      const double2 wk = __ldg(tw2N + j);  // e^{-i pi k/N}
      V[r] = cscale(cmul(cconj(wk), csub(shi, mul_si<1>(slo))), 0.5);
    }
  }
  __syncwarp();  // a tile-backed source has been read completely
  warp_fft_1024<1>(y, xs, t, twb);  // lane t: Y_{t + 32 p}
  // even outputs F_{2k} = -(i/2)(Y_k - Y_{N-k}), k = t + 32 p (p < 16): the mirror N - k sits in lane
  // (32 - t) mod 32, register 31 - p (t != 0), or this lane's register 32 - p (t = 0)
  double2 ev[16];
  {
    const int src = (32 - t) & 31;
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      double2 ym;
      ym.x = __shfl_sync(0xffffffffu, y[31 - p].x, src);
      ym.y = __shfl_sync(0xffffffffu, y[31 - p].y, src);
      if (t == 0) ym = y[(32 - p) & 31];
      ev[p] = make_double2(0.5 * (y[p].y - ym.y), -0.5 * (y[p].x - ym.x));
    }
  }
  warp_fft_16x32<1>(V, xs, t, twb);  // lane t: v_{t + 32 p}
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    const int k = t + 32 * p;
    if (k >= 1) xs[dst32_slot(2 * k - 1)] = cscale(ev[p], scale);
    if (k < M / 2)
      xs[dst32_slot(4 * k)] = cscale(V[p], scale);
    else
      xs[dst32_slot(2 * N - 2 - 4 * k)] = cscale(V[p], -scale);
  }
  __syncwarp();
}

}  // namespace fpc
