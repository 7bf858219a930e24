// kernels_commuted.cu -- the commuted ordering of the alpha-circulant preconditioner (SURVEY
// §8(f)1), 1D.  The reference applies (alpha_circulant.hpp:137-199, tau.hpp:98-119)
//   P^{-1} = (D^{-1} F^* (x) I) blockdiag_n[ S (lambda_n - dt Sigma)^{-1} S ] (F D (x) I)
// with S the orthonormal DST-I (S = S^T = S^{-1}, dst.hpp:15-20) and F the time DFT.  Because
// (F D (x) I) and (I (x) S) act on different axes they commute, so
//   P^{-1} = (I (x) S) (D^{-1} F^* (x) I) diag_{n,i}[ 1/(lambda_n - dt sigma_i) ] (F D (x) I) (I (x) S):
//   1. a DST of every time level (contiguous rows of the time-major vector; real rows, so two
//      levels k and k + Nt/2 ride in one complex row),
//   2. per spatial mode i, ONE column kernel: scale, real time FFT, divide by
//      (lambda_n - dt sigma_i), inverse FFT, unscale (the reference's K2 + K4 without the half
//      spectrum's HBM round trip),
//   3. the DST of every time level again.
// Same 48 B/DoF of compulsory traffic; rounding-level difference from the reference ordering;
// in the time-sharded multi-GPU layout it needs 2 all-to-alls per apply instead of 4.
#include <cstdint>

#include "dst_block.cuh"
#include "fft_block.cuh"
#include "kernels.cuh"

namespace fpc {

__host__ __device__ constexpr int skewed_c(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}
__host__ __device__ constexpr int minb_c(int nt) { return nt <= 128 ? 4 : nt <= 256 ? 2 : 1; }

template <int LOGM, int TOT, int E_ = 16>
struct CGeo {
  static constexpr int E = E_;
  static constexpr int M = 1 << LOGM;
  static constexpr int B = (TOT / M) > 0 ? (TOT / M) : 1;
  static constexpr int NT = (B * M) / E;
  static constexpr int BS = B > 1 ? skewed_c(M) : padded(M);
  static constexpr size_t SMEM = size_t(B) * BS * sizeof(double2);
};

__device__ __forceinline__ double& ccomp(double2* s, int slot_padded, int c) {
  return reinterpret_cast<double*>(s + slot_padded)[c];
}

__device__ __forceinline__ void l2_prefetch_tile(const void* base, size_t stride, int nrows, int width, int nthr) {
  const char* b = static_cast<const char*>(base);
  for (int r = threadIdx.x; r < nrows; r += nthr) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(b + size_t(r) * stride);
    const uintptr_t l0 = a0 & ~uintptr_t(127), l1 = (a0 + uintptr_t(width) - 1) & ~uintptr_t(127);
    for (uintptr_t l = l0; l <= l1; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
  }
}

// ---------------------------------------------------------------------------------------------
// 1. DST of time-level pairs: complex row r = v_r + i v_{r+H} (H = Nt/2), out_r = Re S(row),
//    out_{r+H} = Im S(row), scaled by `scale` (= sqrt(2/N) * input scale).  N = Ns + 1 = 2^LOGN.
// ---------------------------------------------------------------------------------------------
constexpr int kTotPairs = 4096;
template <int LOGN>
struct PairGeo {
  static constexpr int EE = (1 << LOGN) < 16 ? (1 << LOGN) : 16;
  using G = CGeo<LOGN, (LOGN >= 13 ? (1 << LOGN) : kTotPairs), EE>;
  static constexpr int BH = G::B > 1 ? skewed_c(G::M / 2) : padded(G::M / 2);
  static constexpr size_t SMEM = G::SMEM + size_t(G::B) * BH * sizeof(double2);
};

template <int LOGN>
__global__ void __launch_bounds__(PairGeo<LOGN>::G::NT, minb_c(PairGeo<LOGN>::G::NT))
    k_dst_pairs(const double* __restrict__ v, double* __restrict__ out, int n_pairs, double scale,
                const double2* __restrict__ twb) {
  using G = typename PairGeo<LOGN>::G;
  constexpr int N = G::M, B = G::B, BS = G::BS, NT = G::NT;
  constexpr int NS = N - 1;
  constexpr int BH = PairGeo<LOGN>::BH;
  constexpr int U = 4;
  extern __shared__ double2 smem[];
  double2* hbuf = smem + B * BS;
  const int r0 = blockIdx.x * B;
  const int nb = min(B, n_pairs - r0);
  const size_t half = size_t(n_pairs) * NS;  // offset of level r + H
  // both source rows into L2 up front
  for (int b = 0; b < nb; ++b)
    for (int h = 0; h < 2; ++h) {
      const char* zr = reinterpret_cast<const char*>(v + size_t(r0 + b) * NS + h * half);
      const uintptr_t l0 = reinterpret_cast<uintptr_t>(zr) & ~uintptr_t(127);
      const uintptr_t l1 = (reinterpret_cast<uintptr_t>(zr) + size_t(NS) * 8 - 1) & ~uintptr_t(127);
      for (uintptr_t l = l0 + uintptr_t(threadIdx.x) * 128; l <= l1; l += uintptr_t(NT) * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
    }
  constexpr bool kDirect = (LOGN == 13 && B == 1);
  if constexpr (kDirect) {
    const double* re = v + size_t(r0) * NS;
    const double* im = re + half;
    block_dst<LOGN, BS, BH, 0, true>(smem, hbuf, twb, scale, nullptr,
                                     [&](int j) { return make_double2(__ldg(re + j - 1), __ldg(im + j - 1)); });
  } else {
    for (int b = 0; b < B; ++b) {
      const double* re = v + size_t(r0 + b) * NS;
      double2* s = smem + b * BS;
      for (int i0 = threadIdx.x; i0 < NS; i0 += U * NT) {
        double xr[U], xi[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * NT;
          const bool ok = i < NS && b < nb;
          xr[u] = ok ? re[i] : 0.0;
          xi[u] = ok ? re[half + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * NT;
          if (i < NS) s[pad16(i + 1)] = make_double2(xr[u], xi[u]);
        }
      }
    }
    __syncthreads();
    block_dst<LOGN, BS, BH, 0>(smem, hbuf, twb, scale);
  }
  for (int b = 0; b < nb; ++b) {
    double* o = out + size_t(r0 + b) * NS;
    const double2* s = smem + b * BS;
    for (int i = threadIdx.x; i < NS; i += NT) {
      const double2 y = s[pad16(i)];
      o[i] = y.x;
      o[half + i] = y.y;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// 2. Column solve: for each spatial mode p of B columns, x_k = s_in * sf_k * u[k*Ns + p],
//    Z = FFT^{+}(x) (Hermitian half by real packing, as K2), Y_n = Z_n / (lambda_n - dt sigma_p)
//    (MODE 1; MODE 2 multiplies: apply_forward), z_k = sb_k / Nt * Re IFFT(Y) (as K4, mirror folded).
//    In place is allowed (a CTA reads its whole column tile before it writes).
// ---------------------------------------------------------------------------------------------
template <int LOGM>
constexpr int tot_c() { return LOGM >= 10 ? 8192 : 4096; }

template <int LOGM, int MODE>
__global__ void __launch_bounds__(CGeo<LOGM, tot_c<LOGM>()>::NT, minb_c(CGeo<LOGM, tot_c<LOGM>()>::NT))
    k_time_solve(const double* __restrict__ u, double* __restrict__ z, int ns, const double* __restrict__ sf,
                 const double* __restrict__ sb, double s_in, const double2* __restrict__ lam,
                 const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  using G = CGeo<LOGM, tot_c<LOGM>()>;
  constexpr int M = G::M, B = G::B, NTIME = 2 * M, BS = G::BS, NT = G::NT;
  constexpr int U = 16;
  extern __shared__ double2 smem[];
  const int p0 = blockIdx.x * B;
  l2_prefetch_tile(u + p0, size_t(ns) * 8, NTIME, B * 8, NT);

#ifndef FPC_TF_FUSED
#define FPC_TF_FUSED 1
#endif
  if (FPC_TF_FUSED) {
    block_fft_columns_from<LOGM, 1, B, BS, G::E>(smem, twb + M, [&](int c, int kk) {
      const int p = p0 + c;
      return p < ns ? __ldg(sf + kk) * (s_in * u[size_t(kk) * ns + p]) : 0.0;
    });
  } else {
  for (int e0 = threadIdx.x; e0 < B * NTIME; e0 += U * NT) {
    double x[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = e0 + q * NT;
      const int c = e % B, kk = e / B;
      const int p = p0 + c;
      x[q] = (e < B * NTIME && p < ns) ? u[size_t(kk) * ns + p] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = e0 + q * NT;
      if (e < B * NTIME) {
        const int c = e % B, kk = e / B;
        ccomp(smem, c * BS + pad16(kk >> 1), kk & 1) = __ldg(sf + kk) * (s_in * x[q]);
      }
    }
  }
  __syncthreads();
  block_fft<LOGM, 1, BS, G::E>(smem, twb + M, B);
  }

  // unpack (n, M-n) -> Z_n, Z_{M-n}; divide; repack for the inverse (K2 / K4 formulas)
  const double2* twT = twb + NTIME;  // e^{-2 pi i n/Nt}
  for (int t = threadIdx.x; t < B * (M / 2 + 1); t += NT) {
    const int c = t % B, n = t / B;
    const int p = p0 + c;
    double2* s = smem + c * BS;
    const double sg = p < ns ? __ldg(sigma + p) : 0.0;
    if (n == 0) {
      const double2 zz = s[0];
      const double2 l0 = __ldg(lam), lm = __ldg(lam + M);
      const double2 ya = shift_apply<MODE>(make_double2(zz.x + zz.y, 0.0), l0.x - dt * sg, l0.y);
      const double2 yb = shift_apply<MODE>(make_double2(zz.x - zz.y, 0.0), lm.x - dt * sg, lm.y);
      const double2 A = cadd(ya, yb), Bv = csub(ya, yb);
      s[0] = cadd(A, mul_si<1>(Bv));
    } else {
      const double2 a = s[pad16(n)], bq = s[pad16(M - n)];
      const double2 wc = __ldg(twT + n);  // e^{-2 pi i n/Nt}
      const double2 w = cconj(wc);
      const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
      const double2 iwQ = mul_si<1>(cmul(w, Q));
      const double2 ln = __ldg(lam + n), lmn = __ldg(lam + M - n);
      const double2 ya = shift_apply<MODE>(cscale(csub(P, iwQ), 0.5), ln.x - dt * sg, ln.y);
      const double2 yb = shift_apply<MODE>(cscale(cconj(cadd(P, iwQ)), 0.5), lmn.x - dt * sg, lmn.y);
      const double2 A = cadd(ya, cconj(yb));
      const double2 Bn = cmul(csub(ya, cconj(yb)), wc);
      s[pad16(n)] = cadd(A, mul_si<1>(Bn));
      if (n != M - n) s[pad16(M - n)] = cadd(cconj(A), mul_si<1>(cconj(Bn)));
    }
  }
  __syncthreads();
  block_fft<LOGM, -1, BS, G::E>(smem, twb + M, B);

  const double inv_nt = 1.0 / double(NTIME);
  for (int e = threadIdx.x; e < B * NTIME; e += NT) {
    const int c = e % B, kk = e / B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const double val = ccomp(smem, c * BS + pad16(kk >> 1), kk & 1);
    z[size_t(kk) * ns + p] = (__ldg(sb + kk) * inv_nt) * val;
  }
}

// ---------------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------------
template <class K>
static cudaError_t prep_c(K kernel, size_t smem, int threads = 1024) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct(smem, threads));
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaSuccess;
}

static int ilog2_c(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

#define FPC_DISPATCH_C(logm, CALL)         \
  switch (logm) {                          \
    case 1: CALL(1); break;                \
    case 2: CALL(2); break;                \
    case 3: CALL(3); break;                \
    case 4: CALL(4); break;                \
    case 5: CALL(5); break;                \
    case 6: CALL(6); break;                \
    case 7: CALL(7); break;                \
    case 8: CALL(8); break;                \
    case 9: CALL(9); break;                \
    case 10: CALL(10); break;              \
    case 11: CALL(11); break;              \
    case 12: CALL(12); break;              \
    case 13: CALL(13); break;              \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_dst_pairs(const double* v, double* out, int n_space, int n_time, double s_in,
                             const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int ln = ilog2_c(n_space + 1);
  const int n_pairs = n_time / 2;
  const double scale = s_in * sqrt(2.0 / double(n_space + 1));
#define CALL(LN)                                                                              \
  {                                                                                           \
    using PG = PairGeo<LN>;                                                                   \
    if ((err = prep_c(k_dst_pairs<LN>, PG::SMEM, PG::G::NT)) != cudaSuccess) return err;                 \
    k_dst_pairs<LN><<<(n_pairs + PG::G::B - 1) / PG::G::B, PG::G::NT, PG::SMEM, st>>>(v, out, n_pairs, \
                                                                                    scale, tw_base); note_launch(); \
  }
  FPC_DISPATCH_C(ln, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_time_solve(const double* u, double* z, int n_space, int n_time, const double* scale_fwd,
                              const double* scale_bwd, double s_in, const double2* lambda, const double* sigma,
                              double dt, const double2* tw_base, cudaStream_t st, bool forward) {
  cudaError_t err = cudaSuccess;
  if (time_split_supported(n_time))
    return launch_time_solve_split(u, z, n_space, n_time, scale_fwd, scale_bwd, s_in, lambda, sigma, dt, tw_base, st,
                                   forward);
  const int lm = ilog2_c(n_time) - 1;
#define CALL(LM)                                                                                      \
  {                                                                                                   \
    using G = CGeo<LM, tot_c<LM>()>;                                                                  \
    auto kern = forward ? k_time_solve<LM, 2> : k_time_solve<LM, 1>;                                  \
    if ((err = prep_c(kern, G::SMEM, G::NT)) != cudaSuccess) return err;                                     \
    kern<<<(n_space + G::B - 1) / G::B, G::NT, G::SMEM, st>>>(u, z, n_space, scale_fwd, scale_bwd, s_in, \
                                                              lambda, sigma, dt, tw_base); note_launch();            \
  }
  FPC_DISPATCH_C(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

}  // namespace fpc
