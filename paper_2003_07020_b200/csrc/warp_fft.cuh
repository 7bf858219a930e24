// warp_fft.cuh -- register-resident fp64 FFTs owned by a group of R lanes of one warp (sm_100a).
//
// The CTA-level Stockham engine (fft_block.cuh) moves every value through shared memory twice per
// radix-16 pass and synchronises the whole CTA between passes.  For the short transforms of the 2D
// lattice (M = 256 points for n = 255: rows of config 2) that leaves the kernels latency bound on
// barriers and shared-memory round trips (ncu, profiles/r2_summary.md).  Here a transform of
// M = R*R points is owned by R lanes:
//   lane t holds x[t + R r] in v[r]                      (input layout, r = 0..R-1)
//   pass A: DFT_R over r in registers, twiddle w_M^{t q}
//   one transpose through a private (R x (R+1)) shared-memory tile, ordered by __syncwarp
//   pass B: DFT_R over t in registers
//   lane q holds X[q + R p] in v[p]                      (output layout)
// The output layout is the input layout of the same routine (X[q + R p] <-> x[t + R r]), so an
// inverse transform runs straight from a forward's output, and returns values in the forward's input
// layout: a Toeplitz product (FFT, pointwise, inverse FFT) ends with every lane holding exactly the
// positions it loaded.  No CTA barrier anywhere: warps run independently and overlap each other's
// global-memory latency.
//
// Twiddle tables as in fft_block.cuh: tw_N[t] = e^{-2 pi i t/N} at tw_base + N (reference polar()
// values, fft.hpp:36-37).  Sign convention: S = +1 computes X[k] = sum_j x[j] e^{+2 pi i jk/M}.
#pragma once
#include "fft_block.cuh"

namespace fpc {

// Stride of a group's transpose tile row (double2 units): R + 1 keeps both the row-wise writes
// (lane t, fixed q) and the column-wise reads (lane q, fixed t) conflict free for 16-byte accesses.
template <int R>
struct WarpFftTile {
  static constexpr int LD = R + 1;
  static constexpr int SIZE = R * LD;  // double2 per group
};

// v *= w^{S r} with w = e^{2 pi i/16}, r < 8 (the constants of Dft<16>)
template <int S>
__device__ __forceinline__ double2 rot16(double2 x, int r) {
  if (r == 0) return x;
  if (r == 4) return mul_si<S>(x);
  const double c = kC16[r], sn = S * kC16[(r + 12) & 15];
  return make_double2(fma(x.x, c, -x.y * sn), fma(x.x, sn, x.y * c));
}

// DFT_16 of v[0..7] with v[8..15] = 0 (the zero-padded half of a packed circulant embedding):
// X_{2q} = DFT_8(v)_q, X_{2q+1} = DFT_8(v_r w^r)_q -- a quarter fewer operations than the full
// transform, and no arithmetic on the zeros (x + 0.0 cannot be folded by the compiler: -0.0).
template <int S>
__device__ __forceinline__ void dft16_half_in(double2 (&v)[16]) {
  double2 e[8], o[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    e[r] = v[r];
    o[r] = rot16<S>(v[r], r);
  }
  Dft<8, S>::run(e);
  Dft<8, S>::run(o);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[2 * q] = e[q];
    v[2 * q + 1] = o[q];
  }
}

// outputs 0..7 of DFT_16 only (the packed inverse's first half: the truncated Toeplitz product);
// v[8..15] are left unspecified
template <int S>
__device__ __forceinline__ void dft16_low_out(double2 (&v)[16]) {
  double2 e[8], o[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    e[r] = v[2 * r];
    o[r] = v[2 * r + 1];
  }
  Dft<8, S>::run(e);
  Dft<8, S>::run(o);
#pragma unroll
  for (int b = 0; b < 8; ++b) v[b] = cadd(e[b], rot16<S>(o[b], b));
}

// M = R*R point transform by the R lanes of a group (t = lane index within the group).
// `xs` = the group's private tile (WarpFftTile<R>::SIZE double2).  `twb` = tw_base.
// All groups of a warp call this together (twiddles: two table loads and their powers, as the
// Stockham passes -- 15 table loads per pass measured slower).  IN_HALF (R = 16): inputs v[8..15] are zero;
// OUT_HALF (R = 16): only outputs v[0..7] are needed.
template <int R, int S, bool IN_HALF = false, bool OUT_HALF = false>
__device__ __forceinline__ void warp_fft_sq(double2 (&v)[R], double2* __restrict__ xs, int t,
                                            const double2* __restrict__ twb) {
  constexpr int M = R * R;
  constexpr int LD = WarpFftTile<R>::LD;
  if constexpr (IN_HALF) {
    static_assert(R == 16, "half-input pass: R = 16");
    dft16_half_in<S>(v);
  } else {
    Dft<R, S>::run(v);
  }
  apply_twiddles<R, S>(v, twb + M, twb + M / 4, t);  // v[q] *= w_M^{S t q}
#pragma unroll
  for (int q = 0; q < R; ++q) xs[q * LD + t] = v[q];
  __syncwarp();
#pragma unroll
  for (int u = 0; u < R; ++u) v[u] = xs[t * LD + u];
  __syncwarp();  // the tile is free again when any lane of the group reuses it
  if constexpr (OUT_HALF) {
    static_assert(R == 16, "half-output pass: R = 16");
    dft16_low_out<S>(v);
  } else {
    Dft<R, S>::run(v);
  }
}

// Value held by the lane that owns bin M - k, for the lane owning k = q + R p (output layout):
// lane (R - q) mod R, register R-1-p (q != 0), or this lane's register (R - p) mod R (q == 0).
// Every lane of the warp must call it with the same p (width-R shuffle segments).
template <int R, int P>
__device__ __forceinline__ double2 warp_fft_mirror(const double2 (&v)[R], int q) {
  const int src = (R - q) & (R - 1);
  double2 m;
  m.x = __shfl_sync(0xffffffffu, v[R - 1 - P].x, src, R);
  m.y = __shfl_sync(0xffffffffu, v[R - 1 - P].y, src, R);
  if (q == 0) m = v[(R - P) & (R - 1)];
  return m;
}

}  // namespace fpc
