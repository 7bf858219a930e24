// warp_fft32.cuh -- 1024-point fp64 transforms owned by ONE warp: 32 lanes x 32 registers (sm_100a).
//
// The n = 1023 lattice rows / columns of BASELINE config 3 (2D 1023^2 x 1024) ran on the CTA-level
// Stockham engine (fft_block.cuh): three shared-memory passes per 1024-point transform and a CTA
// barrier after each.  Here the scheme of warp_fft.cuh is carried to R = 32:
//   lane t holds x[t + 32 r] in v[r]                     (r = 0..31: 128 registers of data)
//   pass A: DFT_32 over r in registers, twiddle w_1024^{t q}
//   one transpose through the warp's private 32 x 33 tile (16.9 KB), ordered by __syncwarp
//   pass B: DFT_32 over t in registers
//   lane q holds X[q + 32 p] in v[p]
// One shared-memory round trip per transform instead of three, no CTA barrier.  The register
// budget (255 per thread at 8 warps per SM) is what shapes the callers: nothing else that is wide
// may be live across a transform.
#pragma once
#include "warp_fft.cuh"

namespace fpc {

// cos(2 pi k / 32), k = 0..31
__device__ __constant__ double kC32[32] = {
    1.0, 0.98078528040323045, 0.92387953251128676, 0.83146961230254524,
    0.70710678118654752, 0.55557023301960222, 0.38268343236508977, 0.19509032201612827,
    0.0, -0.19509032201612827, -0.38268343236508977, -0.55557023301960222,
    -0.70710678118654752, -0.83146961230254524, -0.92387953251128676, -0.98078528040323045,
    -1.0, -0.98078528040323045, -0.92387953251128676, -0.83146961230254524,
    -0.70710678118654752, -0.55557023301960222, -0.38268343236508977, -0.19509032201612827,
    0.0, 0.19509032201612827, 0.38268343236508977, 0.55557023301960222,
    0.70710678118654752, 0.83146961230254524, 0.92387953251128676, 0.98078528040323045};

// x * w^{S r}, w = e^{2 pi i/32}, 0 <= r < 16 (compile-time r after unrolling)
template <int S>
__device__ __forceinline__ double2 rot32(double2 x, int r) {
  if (r == 0) return x;
  if (r == 8) return mul_si<S>(x);
  const double c = kC32[r], sn = S * kC32[(r + 24) & 31];  // sin(2 pi r/32) = cos(2 pi (r - 8)/32)
  return make_double2(fma(x.x, c, -x.y * sn), fma(x.x, sn, x.y * c));
}

// the radix-2 step on top of two DFT_16 (fft_block.cuh Dft<R>: its constant table stops at 16)
template <int S>
struct Dft<32, S> {
  __device__ __forceinline__ static void run(double2* v) {
    double2 e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    Dft<16, S>::run(e);
    Dft<16, S>::run(o);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 tt = rot32<S>(o[k], k);
      v[k] = cadd(e[k], tt);
      v[k + 16] = csub(e[k], tt);
    }
  }
};

// DFT_32 of v[0..15] with v[16..31] = 0 (the zero-padded half of the packed circulant embedding)
template <int S>
__device__ __forceinline__ void dft32_half_in(double2 (&v)[32]) {
  double2 e[16], o[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    e[r] = v[r];
    o[r] = rot32<S>(v[r], r);
  }
  Dft<16, S>::run(e);
  Dft<16, S>::run(o);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    v[2 * q] = e[q];
    v[2 * q + 1] = o[q];
  }
}

// outputs 0..15 of DFT_32 only (the truncated Toeplitz product); v[16..31] are left unspecified
template <int S>
__device__ __forceinline__ void dft32_low_out(double2 (&v)[32]) {
  double2 e[16], o[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    e[r] = v[2 * r];
    o[r] = v[2 * r + 1];
  }
  Dft<16, S>::run(e);
  Dft<16, S>::run(o);
#pragma unroll
  for (int b = 0; b < 16; ++b) v[b] = cadd(e[b], rot32<S>(o[b], b));
}

// v[q] *= w^{q}, q = 1..31, w = tw[t1]; w^4 and w^16 from the tables a quarter / a sixteenth the
// size (the same doubles as tw[4 t1], tw[16 t1]); the other powers by at most three products
template <int S>
__device__ __forceinline__ void apply_twiddles32(double2 (&v)[32], const double2* __restrict__ tw,
                                                 const double2* __restrict__ tw4, const double2* __restrict__ tw16,
                                                 int t1) {
  const double2 w1 = twid<S>(tw, t1);
  const double2 w4 = twid<S>(tw4, t1);
  const double2 w16 = twid<S>(tw16, t1);
  const double2 w2 = cmul(w1, w1);
  const double2 w3 = cmul(w2, w1);
  const double2 w8 = cmul(w4, w4);
  const double2 w12 = cmul(w8, w4);
#pragma unroll
  for (int hi = 0; hi < 2; ++hi) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 wa = a == 0 ? make_double2(1.0, 0.0) : (a == 1 ? w4 : (a == 2 ? w8 : w12));
      if (hi) wa = a == 0 ? w16 : cmul(w16, wa);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = 16 * hi + 4 * a + b;
        if (q == 0) continue;
        const double2 wb = b == 1 ? w1 : (b == 2 ? w2 : w3);
        const double2 w = b == 0 ? wa : ((a == 0 && hi == 0) ? wb : cmul(wa, wb));
        v[q] = cmul(v[q], w);
      }
    }
  }
}

constexpr int kW32LD = 33;                  // tile row stride (double2): conflict-free both ways
constexpr int kW32Tile = 32 * kW32LD;       // double2 per warp

// 1024-point transform by the 32 lanes of a warp.  xs = the warp's tile (kW32Tile double2).
// IN_HALF: v[16..31] are zero on entry; OUT_HALF: only v[0..15] are needed on exit.
template <int S, bool IN_HALF = false, bool OUT_HALF = false>
__device__ __forceinline__ void warp_fft_1024(double2 (&v)[32], double2* __restrict__ xs, int t,
                                              const double2* __restrict__ twb) {
  constexpr int M = 1024, LD = kW32LD;
  if constexpr (IN_HALF)
    dft32_half_in<S>(v);
  else
    Dft<32, S>::run(v);
  apply_twiddles32<S>(v, twb + M, twb + M / 4, twb + M / 16, t);  // v[q] *= w_M^{S t q}
#pragma unroll
  for (int q = 0; q < 32; ++q) xs[q * LD + t] = v[q];
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 32; ++u) v[u] = xs[t * LD + u];
  __syncwarp();
  if constexpr (OUT_HALF)
    dft32_low_out<S>(v);
  else
    Dft<32, S>::run(v);
}

// Packed circulant product on the warp's spectrum (lane t holds Z_{t + 32 p} in z[p]); the
// arithmetic per mirror pair (k, M - k) is warp_packed_product_shfl's / k_matvec_1d's.  Lane t
// forms the pairs of its bins k = t + 32 p, p < 16; the mirror operand Z_{M-k} comes from lane
// 32 - t, register 31 - p, by shuffle (lane 0: its own register 32 - p), and the partner's result
// U_{M-k} goes back the same way straight into the register the operand came from -- dead from that
// point on -- so no second array is live.
__device__ __forceinline__ void warp_packed_product_1024(double2 (&z)[32], int t, const double* __restrict__ eig,
                                                         const double2* __restrict__ twL) {
  constexpr int R = 32, M = 1024, H = 16;
  const int src = (R - t) & (R - 1);
  {  // the self pair k = M/2 (lane 0, register 16; the other lanes compute on their own value and drop it)
    const double2 mid = z[H];
    const double2 w = __ldg(twL + M / 2);
    const double ek = __ldg(eig + M / 2);
    const double2 P = cadd(mid, cconj(mid)), Q = csub(mid, cconj(mid));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), ek);
    const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
    const double2 zmid = cadd(A, mul_si<1>(cmul(D, cconj(w))));
    if (t == 0) z[H] = zmid;
  }
#pragma unroll
  for (int p = 0; p < H; ++p) {
    const int k = t + R * p;
    const double2 a = z[p];
    double2 bq;
    bq.x = __shfl_sync(0xffffffffu, z[R - 1 - p].x, src);
    bq.y = __shfl_sync(0xffffffffu, z[R - 1 - p].y, src);
    if (t == 0) bq = z[(R - p) & (R - 1)];
    const double2 w = __ldg(twL + k);  // e^{-2 pi i k/L}
    const double ek = __ldg(eig + k), em = __ldg(eig + M - k);
    const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), em);
    const double2 A = cadd(Yk, cconj(Ym)), D = csub(Yk, cconj(Ym));
    double2 uk = cadd(A, mul_si<1>(cmul(D, cconj(w))));
    const double2 um = cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
    if (p == 0 && t == 0) {  // bin 0 carries the DC and Nyquist values of the real embedding
      const double y0 = __ldg(eig) * (2.0 * (a.x + a.y));
      const double ym = __ldg(eig + M) * (2.0 * (a.x - a.y));
      uk = make_double2(y0 + ym, y0 - ym);
    }
    z[p] = uk;
    double2 u;
    u.x = __shfl_sync(0xffffffffu, um.x, src);
    u.y = __shfl_sync(0xffffffffu, um.y, src);
    if (t != 0)
      z[R - 1 - p] = u;
    else if (p >= 1)
      z[(R - p) & (R - 1)] = um;
  }
}

}  // namespace fpc
