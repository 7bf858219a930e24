// fft_block.cuh -- CTA-level fp64 complex FFT engine in shared memory (sm_100a).
//
// Replaces the reference's scalar radix-2 `fft_pow2` (fft.hpp:49-67) on the hot path.  Design:
//   * Stockham autosort, radix 16/8/4/2 passes; each thread owns E = 16 complex values per pass
//     (one radix-16 butterfly, two radix-8, ...), reads them from smem, __syncthreads, applies
//     twiddles + the in-register DFT, writes them to their autosorted slots, __syncthreads.
//     In-place in one buffer: every read of a pass completes before any write.
//   * Buffers are padded one complex per 16 (pad(i) = i + i/16) so the radix-R strided writes of
//     the first pass and the unit-stride reads of every pass are bank-conflict free for 16-byte
//     (double2) accesses.
//   * Twiddles: two loads per butterfly from a per-size table tw_N[t] = e^{-2 pi i t/N}
//     (built on the host with the reference's polar() formula, fft.hpp:36-37), the remaining
//     powers by <=3 complex products.
//   * Batched: a CTA runs B independent transforms of size N = 2^LOGN (buffers at stride
//     padded(N)), NT = B*N/16 threads.
// Kernel sign convention: SIGN = +1 computes x[k] = sum_j x[j] e^{+2 pi i jk/N} (fft.hpp:93-95).
#pragma once
#include <cuda_runtime.h>

namespace fpc {

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 4); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by S*i (S = +-1)
template <int S>
__device__ __forceinline__ double2 mul_si(double2 a) {
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// cos/sin(2 pi k / 16), k = 0..15
__device__ __constant__ double kC16[16] = {
    1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
    0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
    -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977,
    0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674};

// In-register DFT of size R with kernel e^{S 2 pi i jk/R}: natural order in and out.
// Recursive radix-2 DIT; all indices compile-time after unrolling.
template <int R, int S>
struct Dft {
  __device__ __forceinline__ static void run(double2* v) {
    double2 e[R / 2], o[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    Dft<R / 2, S>::run(e);
    Dft<R / 2, S>::run(o);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      // w^k = e^{S 2 pi i k / R}; index into the 16-point table
      constexpr int step = 16 / R;
      double2 t;
      const int idx = k * step;
      if (idx == 0) {
        t = o[k];
      } else if (idx == 4) {
        t = mul_si<S>(o[k]);
      } else if (idx == 8) {
        t = make_double2(-o[k].x, -o[k].y);
      } else if (idx == 12) {
        t = mul_si<-S>(o[k]);
      } else {
        const double c = kC16[idx];
        const double s = S * kC16[(idx + 12) & 15];  // sin(2 pi idx/16) = cos(2 pi (idx-4)/16)
        t = make_double2(fma(o[k].x, c, -o[k].y * s), fma(o[k].x, s, o[k].y * c));
      }
      v[k] = cadd(e[k], t);
      v[k + R / 2] = csub(e[k], t);
    }
  }
};
template <int S>
struct Dft<2, S> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};
template <int S>
struct Dft<4, S> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    const double2 s13 = cadd(v[1], v[3]), d13 = mul_si<S>(csub(v[1], v[3]));
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13);
    v[3] = csub(d02, d13);
  }
};

// Twiddle table access: tw points at the size-N table, tw[t] = e^{-2 pi i t / N}, 0 <= t < N.
template <int S>
__device__ __forceinline__ double2 twid(const double2* __restrict__ tw, int t) {
  const double2 w = __ldg(tw + t);
  return S > 0 ? cconj(w) : w;
}

// Multiply v[r] (r = 1..R-1) by w^r, w = tw[t1] (w4 = tw[4 t1] when R > 4).
template <int R, int S>
__device__ __forceinline__ void apply_twiddles(double2* v, const double2* __restrict__ tw, int t1) {
  if (t1 == 0) return;
  const double2 w1 = twid<S>(tw, t1);
  if constexpr (R == 2) {
    v[1] = cmul(v[1], w1);
  } else if constexpr (R == 4) {
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
  } else {
    const double2 w4 = twid<S>(tw, 4 * t1);
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    double2 w[R];
    w[1] = w1;
    w[2] = w2;
    w[3] = w3;
    w[4] = w4;
    w[5] = cmul(w4, w1);
    w[6] = cmul(w4, w2);
    w[7] = cmul(w4, w3);
    if constexpr (R == 16) {
      const double2 w8 = cmul(w4, w4);
      w[8] = w8;
#pragma unroll
      for (int r = 1; r < 8; ++r) w[8 + r] = cmul(w8, w[r]);
    }
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
  }
}

// One Stockham pass of radix R over B buffers of size N held in smem (padded, stride padded(N)).
// Each thread processes 16/R butterflies (16 complex values).  Ns = current sub-transform length.
template <int LOGN, int R, int S>
__device__ __forceinline__ void stockham_pass(double2* s, const double2* __restrict__ tw, int Ns,
                                              int nbuf) {
  constexpr int N = 1 << LOGN;
  constexpr int NB = N / R;          // butterflies per buffer
  constexpr int PER = 16 / R;        // butterflies per thread
  double2 v[PER][R];
  int dst_b[PER], dst_off[PER];
  const int nthr = blockDim.x;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int g = threadIdx.x + q * nthr;  // global butterfly index across buffers
    const int b = g / NB;
    const int j = g - b * NB;
    dst_b[q] = -1;
    if (b < nbuf) {
      const double2* base = s + b * padded(N);
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = base[pad16(j + r * NB)];
      const int jm = j & (Ns - 1);
      apply_twiddles<R, S>(v[q], tw, jm * (N / (Ns * R)));
      Dft<R, S>::run(v[q]);
      dst_b[q] = b;
      dst_off[q] = (j - jm) * R + jm;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (dst_b[q] >= 0) {
      double2* base = s + dst_b[q] * padded(N);
#pragma unroll
      for (int r = 0; r < R; ++r) base[pad16(dst_off[q] + r * Ns)] = v[q][r];
    }
  }
  __syncthreads();
}

// Full transform of B = nbuf buffers; requires blockDim.x * 16 == nbuf * N (or more threads
// than needed: extra butterflies are masked).  The caller must __syncthreads() before the call
// (data written to smem) and may read the result after it returns.
template <int LOGN, int S>
__device__ __forceinline__ void block_fft(double2* s, const double2* __restrict__ tw, int nbuf) {
  constexpr int N = 1 << LOGN;
  int Ns = 1;
  // radix-16 passes first, then the remainder (8, 4 or 2)
  if constexpr (LOGN >= 4) {
#pragma unroll
    for (int p = 0; p < LOGN / 4; ++p) {
      stockham_pass<LOGN, 16, S>(s, tw, Ns, nbuf);
      Ns *= 16;
    }
  }
  constexpr int rem = LOGN % 4;
  if constexpr (rem == 3) stockham_pass<LOGN, 8, S>(s, tw, Ns, nbuf);
  if constexpr (rem == 2) stockham_pass<LOGN, 4, S>(s, tw, Ns, nbuf);
  if constexpr (rem == 1) stockham_pass<LOGN, 2, S>(s, tw, Ns, nbuf);
  (void)N;
}

}  // namespace fpc
