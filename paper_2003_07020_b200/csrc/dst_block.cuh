// dst_block.cuh -- CTA-level orthonormal DST-I of complex rows in shared memory.
//
// Replaces the reference's dst1 (dst.hpp:21-43), which runs one complex FFT of the length-2(n+1)
// odd extension, by the half-length sine-transform algorithm (pre-twiddle + one N-point FFT +
// a prefix sum; N = n + 1 = 2^LOGN):
//   y_0 = 0,  y_j = sin(pi j/N) (f_j + f_{N-j}) + (f_j - f_{N-j})/2          (j = 1..N-1)
//   Y_k = sum_j y_j e^{+2 pi i jk/N}
//   F_{2k}   = -(i/2) (Y_k - Y_{N-k})                                         (k = 1..N/2-1)
//   F_{2k+1} = Y_0/2 + sum_{m=1..k} (Y_m + Y_{N-m})/2                           (k = 0..N/2-1)
// with F_m = sum_j f_j sin(pi j m/N) and DST(f)_i = sqrt(2/N) F_{i+1}.  The identity holds for
// complex f directly (it is real-linear with real coefficients), so a complex row costs one
// N-point complex FFT -- a quarter of the reference's 2N-point transform per component pair.
// The prefix sum is a fixed-shape (deterministic) per-thread / warp-shuffle / per-warp scan.
#pragma once
#include "fft_block.cuh"

namespace fpc {

__device__ __forceinline__ double2 shfl_up2(double2 v, int d, int width) {
  double2 r;
  r.x = __shfl_up_sync(0xffffffffu, v.x, d, width);
  r.y = __shfl_up_sync(0xffffffffu, v.y, d, width);
  return r;
}

// Scratch: (blockDim.x / 32) double2 in shared memory.
// Buffers: B = blockDim.x * E / N buffers of stride BS; input f_j at slot j (slot 0 ignored).
// Output: DST(f)_i * scale written at slot i + OUT_SHIFT (i = 0..N-2); slot 0 zeroed when
// OUT_SHIFT = 1 so the buffer is again a valid input.
template <int LOGN, int BS, int E, int OUT_SHIFT>
__device__ __forceinline__ void block_dst(double2* s, const double2* __restrict__ twb, double scale,
                                          double2* scratch) {
  constexpr int N = 1 << LOGN;
  constexpr int TPB = N / E;    // threads per buffer
  constexpr int KP = E / 2;     // k values per thread (N/2 per buffer)
  const int nthr = blockDim.x;
  const double2* tw2N = twb + 2 * N;  // e^{-i pi j/N}
  // 1. pre-twiddle, in place on (j, N-j) pairs
  for (int t = threadIdx.x; t < (nthr / TPB) * (N / 2); t += nthr) {
    const int b = t / (N / 2), j = 1 + (t & (N / 2 - 1));
    double2* r = s + b * BS;
    const double sj = -__ldg(tw2N + j).y;  // sin(pi j/N)
    const double2 fj = r[pad16(j)], fm = r[pad16(N - j)];
    const double2 sum = cadd(fj, fm), dif = csub(fj, fm);
    r[pad16(j)] = make_double2(fma(sj, sum.x, 0.5 * dif.x), fma(sj, sum.y, 0.5 * dif.y));
    if (j != N / 2) r[pad16(N - j)] = make_double2(fma(sj, sum.x, -0.5 * dif.x), fma(sj, sum.y, -0.5 * dif.y));
    if (j == 1) r[0] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  block_fft<LOGN, 1, BS, E>(s, twb + N, 0);

  // 2. post: thread handles k = tb*KP .. tb*KP + KP-1 of its buffer
  const int b = threadIdx.x / TPB, tb = threadIdx.x - b * TPB;
  const double2* r = s + b * BS;
  double2 ev[KP], od[KP];
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const int k = tb * KP + u;
    const double2 yk = r[pad16(k)], ym = r[pad16((N - k) & (N - 1))];
    ev[u] = make_double2(0.5 * (yk.y - ym.y), -0.5 * (yk.x - ym.x));  // -(i/2)(Yk - Ym)
    od[u] = k == 0 ? cscale(yk, 0.5) : cscale(cadd(yk, ym), 0.5);
  }
#pragma unroll
  for (int u = 1; u < KP; ++u) od[u] = cadd(od[u - 1], od[u]);  // in-thread inclusive prefix
  // segmented (per buffer) exclusive scan of thread totals
  constexpr int W = TPB < 32 ? TPB : 32;
  double2 incl = od[KP - 1];
  const int lane = threadIdx.x & 31;
  const int lw = lane & (W - 1);
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    const double2 o = shfl_up2(incl, d, W);
    if (lw >= d) incl = cadd(incl, o);
  }
  double2 excl = shfl_up2(incl, 1, W);
  if (lw == 0) excl = make_double2(0.0, 0.0);
  if constexpr (TPB > 32) {
    const int warp = threadIdx.x >> 5;
    if (lane == 31) scratch[warp] = incl;
    __syncthreads();
    const int w0 = (b * TPB) >> 5;
    double2 off = make_double2(0.0, 0.0);
    for (int w = w0; w < warp; ++w) off = cadd(off, scratch[w]);
    excl = cadd(off, excl);
  }
  __syncthreads();  // every read of Y is done before the buffer is overwritten
  double2* rw = s + b * BS;
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const int k = tb * KP + u;
    const double2 o = cadd(excl, od[u]);
    if (k > 0) rw[pad16(2 * k - 1 + OUT_SHIFT)] = cscale(ev[u], scale);
    rw[pad16(2 * k + OUT_SHIFT)] = cscale(o, scale);
  }
  if (OUT_SHIFT == 1 && tb == 0) rw[0] = make_double2(0.0, 0.0);
  __syncthreads();
}

}  // namespace fpc
