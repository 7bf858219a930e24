// dst_block.cuh -- CTA-level orthonormal DST-I of complex rows in shared memory.
//
// Replaces the reference's dst1 (dst.hpp:21-43: one complex FFT of the length-2(n+1) odd
// extension) by a split that needs 1.5 FFTs of length N = n + 1 per complex row and keeps the
// reference's accuracy (no recurrences):  with F_m = sum_j f_j sin(pi j m/N) and
// DST(f)_i = sqrt(2/N) F_{i+1},
//   even outputs (sine-transform pre-twiddle + one N-point FFT):
//     y_0 = 0, y_j = sin(pi j/N)(f_j + f_{N-j}) + (f_j - f_{N-j})/2,  Y = FFT_N^{+}(y)
//     F_{2k} = -(i/2) (Y_k - Y_{N-k})                                    k = 1..M-1, M = N/2
//   odd outputs (a DCT-III of length M through one M-point FFT, Makhoul's reordering):
//     s_j = f_j + f_{N-j} (j < M), s_M = f_M,  t_k = s_{M-k}
//     V_0 = t_0, V_k = (1/2) e^{i pi k/(2M)} (t_k - i t_{M-k}),  v = FFT_M^{+}(V)
//     x_{2m} = v_m, x_{2m+1} = v_{M-1-m},  F_{2k+1} = (-1)^k x_k          k = 0..M-1
// (The classic single-FFT sine transform recovers the odd outputs by a running sum, whose error
// grows like sqrt(N); that is measurably worse than the reference at large N, so it is not used.)
// The identities are real-linear with real coefficients, so they hold for complex rows directly.
#pragma once
#include <type_traits>

#include "fft_block.cuh"

#ifndef FPC_DST_PH
#define FPC_DST_PH(i) \
  do {                \
  } while (0)
#endif

#ifndef FPC_DCT_HALF_GROUP
#define FPC_DCT_HALF_GROUP 1
#endif
#ifndef FPC_DST_PRE_SEL
#define FPC_DST_PRE_SEL 1
#endif
#ifndef FPC_DST_DUAL
#define FPC_DST_DUAL 0  // measured slower (config-1 tau 3.18 -> 3.35 ms per solve), kept for A/B
#endif
#ifndef FPC_DCT_HALF_MAXLOG
#define FPC_DCT_HALF_MAXLOG 9
#endif

namespace fpc {

// Buffers: B = blockDim.x * 16 / N rows; row b has an N-slot buffer at s + b*BS (input f_j at
// slot j, slot 0 ignored) and an M-slot scratch buffer at h + b*BH.  Output: DST(f)_i * scale at
// slot i + OUT_SHIFT of the N-slot buffer (slot 0 zeroed when OUT_SHIFT = 1, so the buffer is
// again a valid input).
// One row per CTA with the N-point FFT's radix-2 remainder pass (N = 2^(4k+1)) folded into the
// pre-twiddle: the quadruple (j, N-j, M-j, M+j) holds both radix-2 pairs (j, j+M) and (M-j, N-j),
// so the pre-phase writes the first Stockham pass's outputs directly (one shared-memory pass and
// two barriers less per DST).
// gsrc != nullptr: the row is read straight from global memory (f_j = gsrc[j-1]) instead of the
// buffer (saves the staging pass of the first DST of a tau solve)
// Src: f(j) -> f_j, j = 1..N-1 (the buffer, a global row, or a gather of two real rows)
template <int LOGN, int BH, class Src>
__device__ __forceinline__ void dst_pre_folded(double2* r, double2* hv, const double2* __restrict__ tw2N,
                                               Src f) {
  constexpr int N = 1 << LOGN, M = N / 2, NT = N / 16;
  constexpr int KQ = (M / 2) / NT;  // quadruples j < M/2 per thread; j = M/2 goes to thread 0
  static_assert(KQ * NT == M / 2, "quadruple count must divide the thread count");
  double2 o[KQ][4], mid[2];
#pragma unroll
  for (int u = 0; u < KQ; ++u) {
    const int j = int(threadIdx.x) + u * NT;
    if (j == 0) {  // y_0 = 0, y_M = 2 f_M, V_0 = f_M
      const double2 fm = f(M);
      o[u][0] = cscale(fm, 2.0);
      o[u][1] = cscale(fm, -2.0);
      hv[0] = fm;
      continue;
    }
    const double2 wj = __ldg(tw2N + j);
    const double2 wm = make_double2(-wj.y, -wj.x);  // e^{-i pi (M-j)/N} = -i conj(e^{-i pi j/N}), M = N/2
    const double2 f1 = f(j), f2 = f(N - j);
    const double2 g1 = f(M - j), g2 = f(M + j);
    const double2 sj = cadd(f1, f2), dj = csub(f1, f2), sm = cadd(g1, g2), dm = csub(g1, g2);
    const double sinj = -wj.y, sinm = -wm.y;
    const double2 yj = make_double2(fma(sinj, sj.x, 0.5 * dj.x), fma(sinj, sj.y, 0.5 * dj.y));
    const double2 yNj = make_double2(fma(sinj, sj.x, -0.5 * dj.x), fma(sinj, sj.y, -0.5 * dj.y));
    const double2 yMj = make_double2(fma(sinm, sm.x, 0.5 * dm.x), fma(sinm, sm.y, 0.5 * dm.y));
    const double2 yPj = make_double2(fma(sinm, sm.x, -0.5 * dm.x), fma(sinm, sm.y, -0.5 * dm.y));
    o[u][0] = cadd(yj, yPj);  // pair (j, j+M)
    o[u][1] = csub(yj, yPj);
    o[u][2] = cadd(yMj, yNj);  // pair (M-j, N-j)
    o[u][3] = csub(yMj, yNj);
    hv[pad16(j)] = cscale(cmul(cconj(wj), csub(sm, mul_si<1>(sj))), 0.5);
    hv[pad16(M - j)] = cscale(cmul(cconj(wm), csub(sj, mul_si<1>(sm))), 0.5);
  }
  if (threadIdx.x == 0) {  // j = M/2: its own mirror, pair (M/2, 3M/2)
    constexpr int j = M / 2;
    const double2 wj = __ldg(tw2N + j);
    const double2 f1 = f(j), f2 = f(N - j);
    const double2 sj = cadd(f1, f2), dj = csub(f1, f2);
    const double sinj = -wj.y;
    const double2 yj = make_double2(fma(sinj, sj.x, 0.5 * dj.x), fma(sinj, sj.y, 0.5 * dj.y));
    const double2 yNj = make_double2(fma(sinj, sj.x, -0.5 * dj.x), fma(sinj, sj.y, -0.5 * dj.y));
    mid[0] = cadd(yj, yNj);
    mid[1] = csub(yj, yNj);
    hv[pad16(j)] = cscale(cmul(cconj(wj), csub(sj, mul_si<1>(sj))), 0.5);
  }
  __syncthreads();  // every f has been read before the pass outputs overwrite the row
  // the pair (2j, 2j+1) is written as two stores whose slot parity alternates with lane bit 2: each
  // store then covers eight bank groups per quarter warp (2j alone hits four, twice)
  const int sel = FPC_DST_PRE_SEL ? (int(threadIdx.x) >> 2) & 1 : 0;
#pragma unroll
  for (int u = 0; u < KQ; ++u) {
    const int j = int(threadIdx.x) + u * NT;
    r[pad16(2 * j + sel)] = sel ? o[u][1] : o[u][0];
    r[pad16(2 * j + 1 - sel)] = sel ? o[u][0] : o[u][1];
    if (j != 0) {
      r[pad16(2 * (M - j))] = o[u][2];
      r[pad16(2 * (M - j) + 1)] = o[u][3];
    }
  }
  if (threadIdx.x == 0) {
    r[pad16(M)] = mid[0];
    r[pad16(M + 1)] = mid[1];
  }
}

template <int LOGN, int BS, int BH, int OUT_SHIFT, bool FOLD = false, class Src = void*>
__device__ __forceinline__ void block_dst(double2* s, double2* h, const double2* __restrict__ twb,
                                          double scale, const double2* gsrc = nullptr, Src src = nullptr) {
  constexpr int N = 1 << LOGN, M = N / 2;
  constexpr int E = N < 16 ? N : 16;  // complex values per thread in the N-point FFT
  constexpr int TPB = N / E;          // threads per row
  constexpr int KP = M / TPB;         // k values per thread in the post-processing
  const int nthr = blockDim.x;
  const int nrow = nthr / TPB;
  const double2* tw2N = twb + 2 * N;  // e^{-i pi j/N}
  if constexpr (FOLD) {
    static_assert(LOGN % 4 == 1 && LOGN >= 5, "fold needs N = 2 * 16^k");
    if constexpr (!std::is_same<Src, void*>::value)
      dst_pre_folded<LOGN, BH>(s, h, tw2N, src);
    else if (gsrc)
      dst_pre_folded<LOGN, BH>(s, h, tw2N, [&](int j) { return gsrc[j - 1]; });
    else
      dst_pre_folded<LOGN, BH>(s, h, tw2N, [&](int j) { return s[pad16(j)]; });
    __syncthreads();
    FPC_DST_PH(0);
    if constexpr (FPC_DST_DUAL && E == 16) {
      // the N-point FFT (after the folded radix-2 pass) and the M-point DCT FFT, both k radix-16
      // passes, pipelined against each other (fft_block.cuh dual_fft_passes)
      dual_fft_passes<LOGN, BS, 2, LOGN - 1, BH, 1, 1>(s, twb + N, h, twb + M, int(threadIdx.x), nthr, nthr / 2);
    } else {
    fft_passes<LOGN, 1, BS, E, 2, CtaSync>(s, twb + N, int(threadIdx.x), nthr);
    FPC_DST_PH(1);
    if constexpr (FPC_DCT_HALF_GROUP && E == 16) {
      // the M-point DCT FFT in radix-16 passes by half the CTA (named barrier): fewer passes, i.e.
      // less shared-memory traffic, than radix-8 passes over all threads -- these kernels are
      // bound by the shared-memory pipe
      constexpr int NH = (N / 2) / 16;
      if (int(threadIdx.x) < NH) group_fft<LOGN - 1, 1, BH, 16, NH, 1>(h, twb + M, int(threadIdx.x));
      __syncthreads();
    } else {
      block_fft<LOGN - 1, 1, BH, E / 2>(h, twb + M, 0);
    }
    }
    FPC_DST_PH(2);
  } else {
  // 1. pre: quadruples (j, N-j, M-j, M+j), j = 1..M/2 (degenerate at j = M/2 and for j = M)
  for (int t = threadIdx.x; t < nrow * (M / 2 + 1); t += nthr) {
    const int b = t / (M / 2 + 1), j = t - b * (M / 2 + 1);
    double2* r = s + b * BS;
    double2* hv = h + b * BH;
    if (j == 0) {  // centre f_M: y_M = 2 f_M, V_0 = t_0 = f_M; y_0 = 0
      const double2 fm = r[pad16(M)];
      r[pad16(M)] = cscale(fm, 2.0);
      r[0] = make_double2(0.0, 0.0);
      hv[0] = fm;
      continue;
    }
    const double2 wj = __ldg(tw2N + j);            // e^{-i pi j/N}: sin(pi j/N) = -wj.y
    const double2 wm = make_double2(-wj.y, -wj.x);  // e^{-i pi (M-j)/N} = -i conj(wj)
    const double2 f1 = r[pad16(j)], f2 = r[pad16(N - j)];
    const double2 sj = cadd(f1, f2), dj = csub(f1, f2);
    const double sinj = -wj.y, sinm = -wm.y;
    r[pad16(j)] = make_double2(fma(sinj, sj.x, 0.5 * dj.x), fma(sinj, sj.y, 0.5 * dj.y));
    r[pad16(N - j)] = make_double2(fma(sinj, sj.x, -0.5 * dj.x), fma(sinj, sj.y, -0.5 * dj.y));
    // s_{M-j} from the mirrored pair (M-j, M+j); for j = M/2 it is the same pair
    double2 sm;
    if (j != M / 2) {
      const double2 g1 = r[pad16(M - j)], g2 = r[pad16(M + j)];
      sm = cadd(g1, g2);
      const double2 dm = csub(g1, g2);
      r[pad16(M - j)] = make_double2(fma(sinm, sm.x, 0.5 * dm.x), fma(sinm, sm.y, 0.5 * dm.y));
      r[pad16(M + j)] = make_double2(fma(sinm, sm.x, -0.5 * dm.x), fma(sinm, sm.y, -0.5 * dm.y));
    } else {
      sm = sj;
    }
    // V_k = 1/2 e^{i pi k/N} (t_k - i t_{M-k}) with t_k = s_{M-k}:
    //   k = j:     1/2 e^{i pi j/N}     (s_{M-j} - i s_j)
    //   k = M - j: 1/2 e^{i pi (M-j)/N} (s_j - i s_{M-j})
    hv[pad16(j)] = cscale(cmul(cconj(wj), csub(sm, mul_si<1>(sj))), 0.5);
    if (j != M / 2) hv[pad16(M - j)] = cscale(cmul(cconj(wm), csub(sj, mul_si<1>(sm))), 0.5);
  }
  __syncthreads();
  FPC_DST_PH(0);
  block_fft<LOGN, 1, BS, E>(s, twb + N, 0);
  FPC_DST_PH(1);
  // the M-point DCT FFTs of all rows: radix-16 passes on half the CTA when the CTA size allows
  // (fewer shared-memory passes, as in the folded path; N <= 512: the larger-N small grids are
  // latency bound and lose more to the idle half), else radix-8 passes on all threads
  if (FPC_DCT_HALF_GROUP && E == 16 && LOGN >= 5 && LOGN <= FPC_DCT_HALF_MAXLOG && nthr == 256) {
    if (int(threadIdx.x) < 128) group_fft<LOGN - 1, 1, BH, 16, 128, 1>(h, twb + M, int(threadIdx.x));
    __syncthreads();
  } else if (FPC_DCT_HALF_GROUP && E == 16 && LOGN >= 5 && LOGN <= FPC_DCT_HALF_MAXLOG && nthr == 512) {
    if (int(threadIdx.x) < 256) group_fft<LOGN - 1, 1, BH, 16, 256, 1>(h, twb + M, int(threadIdx.x));
    __syncthreads();
  } else {
    block_fft<LOGN - 1, 1, BH, E / 2>(h, twb + M, 0);
  }
  FPC_DST_PH(2);
  }

  // 2. post: thread handles k = tb*KP .. tb*KP + KP-1 of its row
  const int b = threadIdx.x / TPB, tb = threadIdx.x - b * TPB;
  const double2* r = s + b * BS;
  const double2* hv = h + b * BH;
  double2 ev[KP], od[KP];
  // thread tb owns k = tb*KP .. tb*KP + KP-1, visited in a per-thread rotated order: at step u the
  // eight lanes of a quarter warp then hit eight different bank groups in the reads of Y_k, Y_{N-k},
  // the DCT slot and the two output writes (1.05 wavefronts per access against 1.6 unrotated,
  // KP = 8)
#ifndef FPC_DST_POST_ROT
#define FPC_DST_POST_ROT 1
#endif
  // (rows of TPB < 32 threads share a warp at skewed buffer strides: same rotation for TPB >= 8,
  // (4 tb + 5 floor(tb/2)) for TPB = 4: 2.8 -> 1.6 wavefronts)
  const int rot = !FPC_DST_POST_ROT ? 0
                  : TPB >= 8        ? 4 * tb + 4 * (tb >> 1)
                  : TPB == 4        ? 4 * tb + 5 * (tb >> 1)
                                    : 0;
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const int k = tb * KP + ((u + rot) & (KP - 1));
    const double2 yk = r[pad16(k)], ym = r[pad16((N - k) & (N - 1))];
    ev[u] = make_double2(0.5 * (yk.y - ym.y), -0.5 * (yk.x - ym.x));  // -(i/2)(Yk - Y_{N-k})
    const double2 x = hv[pad16((k & 1) ? (M - 1 - (k >> 1)) : (k >> 1))];
    od[u] = (k & 1) ? make_double2(-x.x, -x.y) : x;
  }
  __syncthreads();  // every read of Y is done before the buffer is overwritten
  double2* rw = s + b * BS;
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const int k = tb * KP + ((u + rot) & (KP - 1));
    if (k > 0) rw[pad16(2 * k - 1 + OUT_SHIFT)] = cscale(ev[u], scale);
    rw[pad16(2 * k + OUT_SHIFT)] = cscale(od[u], scale);
  }
  if (OUT_SHIFT == 1 && tb == 0) rw[0] = make_double2(0.0, 0.0);
  __syncthreads();
  FPC_DST_PH(3);
}

}  // namespace fpc
