// kernels_1d.cu -- sm_100a kernels of the 1D hot path: all-at-once matvec (K1), the
// alpha-circulant preconditioner's time FFTs (K2/K4) and the tau shifted solves (K3).
//
// Data layout in HBM (matches the reference's time-major vectors, all_at_once.hpp:18-22):
//   v[k*Ns + p]            real fp64, k = time level, p = spatial index
//   Z[n*Ns + p]            complex128 half spectrum, n = 0..Nt/2 (frequency-major rows, so the
//                          tau solves of K3 read contiguous rows; alpha_circulant.hpp:153-156)
// Every transform is a power-of-two complex FFT run in shared memory by fft_block.cuh; the
// real-input transforms use the standard half-length packing (two reals per complex).
#include <cooperative_groups.h>

#include "fft_block.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fpc {

// Elements per CTA for a kernel family; B = buffers per CTA, NT = threads.
template <int LOGM, int TOT>
struct Geo {
  static constexpr int M = 1 << LOGM;
  static constexpr int B = (TOT / M) > 0 ? (TOT / M) : 1;
  static constexpr int NT = (B * M) / 16;
  static constexpr size_t SMEM = size_t(B) * padded(M) * sizeof(double2);
};

__device__ __forceinline__ double& comp(double2* s, int slot_padded, int c) {
  return reinterpret_cast<double*>(s + slot_padded)[c];
}

// =====================================================================================
// K1: 1D all-at-once matvec.  One buffer per time block k; real packing of the length-L
// circulant embedding (L = 2M = next_pow2(2 Ns), toeplitz.hpp:26) into an M-point FFT.
// eig'[k] = -dt * eig[k] / (2L), k = 0..M  (eig real & even: the circulant column is
// symmetric, toeplitz.hpp:27-33).
// =====================================================================================
constexpr int kTotMv = 4096;

template <int LOGM>
__global__ void __launch_bounds__(Geo<LOGM, kTotMv>::NT)
    k_matvec_1d(const double* __restrict__ v, double* __restrict__ y, int ns, int nt,
                const double* __restrict__ eig, const double2* __restrict__ twb) {
  using G = Geo<LOGM, kTotMv>;
  constexpr int M = G::M, B = G::B, L = 2 * M;
  extern __shared__ double2 smem[];
  const int k0 = blockIdx.x * B;
  const int nb = min(B, nt - k0);

  for (int e = threadIdx.x; e < B * L; e += blockDim.x) {
    const int b = e / L, idx = e - b * L;
    double x = 0.0;
    if (b < nb && idx < ns) x = v[size_t(k0 + b) * ns + idx];
    comp(smem, b * padded(M) + pad16(idx >> 1), idx & 1) = x;
  }
  __syncthreads();
  block_fft<LOGM, -1>(smem, twb + M, B);

  // pointwise product with the circulant eigenvalues, done on (k, M-k) pairs of the packed
  // spectrum: unpack -> X_k, X_{M-k}; Y = eig' X; repack for the inverse.
  const double2* twL = twb + L;
  for (int t = threadIdx.x; t < B * (M / 2 + 1); t += blockDim.x) {
    const int b = t / (M / 2 + 1), kk = t - b * (M / 2 + 1);
    double2* s = smem + b * padded(M);
    if (kk == 0) {
      const double2 z = s[0];
      const double y0 = eig[0] * (2.0 * (z.x + z.y));
      const double ym = eig[M] * (2.0 * (z.x - z.y));
      s[0] = make_double2(y0 + ym, y0 - ym);
    } else {
      const int i1 = pad16(kk), i2 = pad16(M - kk);
      const double2 a = s[i1], bq = s[i2];
      const double2 w = __ldg(twL + kk);  // e^{-2 pi i k/L}
      const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
      const double2 iwQ = mul_si<1>(cmul(w, Q));
      const double2 Xk = csub(P, iwQ);
      const double2 Xm = cconj(cadd(P, iwQ));
      const double2 Yk = cscale(Xk, eig[kk]);
      const double2 Ym = cscale(Xm, eig[M - kk]);
      const double2 A = cadd(Yk, cconj(Ym));
      const double2 D = csub(Yk, cconj(Ym));
      const double2 Bk = cmul(D, cconj(w));
      const double2 Bm = cmul(cconj(D), w);
      s[i1] = cadd(A, mul_si<1>(Bk));
      if (kk != M - kk) s[i2] = cadd(cconj(A), mul_si<1>(Bm));
    }
  }
  __syncthreads();
  block_fft<LOGM, 1>(smem, twb + M, B);

  // epilogue: BDF2 stencil (time_stencil.hpp:16-26) + the spatial term
  for (int e = threadIdx.x; e < B * ns; e += blockDim.x) {
    const int b = e / ns, idx = e - b * ns;
    if (b >= nb) continue;
    const int k = k0 + b;
    const double tv = comp(smem, b * padded(M) + pad16(idx >> 1), idx & 1);
    const size_t o = size_t(k) * ns + idx;
    double c;
    if (k == 0)
      c = v[o];
    else if (k == 1)
      c = 1.5 * v[o] + -2.0 * v[o - ns];
    else
      c = 1.5 * v[o] + -2.0 * v[o - ns] + 0.5 * v[o - 2 * size_t(ns)];
    y[o] = c + tv;
  }
}

// =====================================================================================
// K2: time FFT forward over spatial columns (alpha_circulant.hpp:146-156), Hermitian half.
// CTA = B columns; M = Nt/2.
// =====================================================================================
constexpr int kTotT = 8192;

template <int LOGM>
__global__ void __launch_bounds__(Geo<LOGM, kTotT>::NT)
    k_time_fwd(const double* __restrict__ v, double2* __restrict__ Z, int ns,
               const double* __restrict__ sf, double s_in, const double2* __restrict__ twb) {
  using G = Geo<LOGM, kTotT>;
  constexpr int M = G::M, B = G::B, NTIME = 2 * M;
  extern __shared__ double2 smem[];
  const int p0 = blockIdx.x * B;

  for (int e = threadIdx.x; e < B * NTIME; e += blockDim.x) {
    const int c = e % B, kk = e / B;
    const int p = p0 + c;
    double x = 0.0;
    if (p < ns) x = sf[kk] * (s_in * v[size_t(kk) * ns + p]);
    comp(smem, c * padded(M) + pad16(kk >> 1), kk & 1) = x;
  }
  __syncthreads();
  block_fft<LOGM, 1>(smem, twb + M, B);

  const double2* twT = twb + NTIME;  // e^{-2 pi i n/Nt}; the forward kernel here is e^{+...}
  for (int t = threadIdx.x; t < B * (M / 2 + 1); t += blockDim.x) {
    const int c = t % B, n = t / B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const double2* s = smem + c * padded(M);
    if (n == 0) {
      const double2 z = s[0];
      Z[p] = make_double2(z.x + z.y, 0.0);
      Z[size_t(M) * ns + p] = make_double2(z.x - z.y, 0.0);
    } else {
      const double2 a = s[pad16(n)], bq = s[pad16(M - n)];
      const double2 w = cconj(__ldg(twT + n));  // e^{+2 pi i n/Nt}
      const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
      const double2 iwQ = mul_si<1>(cmul(w, Q));
      Z[size_t(n) * ns + p] = cscale(csub(P, iwQ), 0.5);
      if (n != M - n) Z[size_t(M - n) * ns + p] = cscale(cconj(cadd(P, iwQ)), 0.5);
    }
  }
}

// =====================================================================================
// K4: inverse time FFT (alpha_circulant.hpp:167-198) from the half spectrum; the mirror
// Z_{Nt-n} = conj(Z_n) (alpha_circulant.hpp:167-175) is folded into the real-output packing.
// =====================================================================================
template <int LOGM>
__global__ void __launch_bounds__(Geo<LOGM, kTotT>::NT)
    k_time_inv(const double2* __restrict__ Z, double* __restrict__ z, int ns,
               const double* __restrict__ sb, const double2* __restrict__ twb) {
  using G = Geo<LOGM, kTotT>;
  constexpr int M = G::M, B = G::B, NTIME = 2 * M;
  extern __shared__ double2 smem[];
  const int p0 = blockIdx.x * B;
  const double2* twT = twb + NTIME;

  for (int t = threadIdx.x; t < B * (M / 2 + 1); t += blockDim.x) {
    const int c = t % B, n = t / B;
    const int p = p0 + c;
    double2* s = smem + c * padded(M);
    if (p >= ns) {  // padding column: keep its buffer finite
      s[pad16(n)] = make_double2(0.0, 0.0);
      if (n != 0) s[pad16(M - n)] = make_double2(0.0, 0.0);
      continue;
    }
    if (n == 0) {
      const double2 y0 = Z[p], ym = Z[size_t(M) * ns + p];
      const double2 A = cadd(y0, ym), Bv = csub(y0, ym);
      s[0] = cadd(A, mul_si<1>(Bv));
    } else {
      const double2 a = Z[size_t(n) * ns + p], bq = Z[size_t(M - n) * ns + p];
      const double2 w = __ldg(twT + n);  // e^{-2 pi i n/Nt}
      const double2 A = cadd(a, cconj(bq));
      const double2 Bn = cmul(csub(a, cconj(bq)), w);
      s[pad16(n)] = cadd(A, mul_si<1>(Bn));
      if (n != M - n) s[pad16(M - n)] = cadd(cconj(A), mul_si<1>(cconj(Bn)));
    }
  }
  __syncthreads();
  block_fft<LOGM, -1>(smem, twb + M, B);

  const double inv_nt = 1.0 / double(NTIME);
  for (int e = threadIdx.x; e < B * NTIME; e += blockDim.x) {
    const int c = e % B, kk = e / B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const double val = comp(smem, c * padded(M) + pad16(kk >> 1), kk & 1);
    z[size_t(kk) * ns + p] = (sb[kk] * inv_nt) * val;
  }
}

// =====================================================================================
// K3 (1D): tau shifted solves (tau.hpp:98-119), one frequency row of Ns complex per CTA pair.
// A 2-CTA cluster splits the row by component: rank 0 transforms Re, rank 1 transforms Im
// (the DST is real-linear, dst.hpp:14-20), each with one packed M-point FFT (M = Ns + 1) of the
// length-2M odd extension (dst.hpp:26-32).  The complex division (tau.hpp:109-114) needs both
// components, exchanged through distributed shared memory.
// =====================================================================================
constexpr int kTotTau = 4096;

template <int LOGM>
struct TauGeo {
  using G = Geo<LOGM, (LOGM >= 13 ? (1 << LOGM) : kTotTau)>;
  static constexpr size_t SMEM = G::SMEM + size_t(G::B) * G::M * sizeof(double);
};

// Pack +-x into the odd extension w (length 2M): w[i+1] = x_i, w[2M-1-i] = -x_i.
template <int M>
__device__ __forceinline__ void pack_odd(double2* s, int i, double x) {
  const int p1 = i + 1, p2 = 2 * M - 1 - i;
  comp(s, pad16(p1 >> 1), p1 & 1) = x;
  comp(s, pad16(p2 >> 1), p2 & 1) = -x;
}

// DST post-processing for pair (k, M-k): returns the two DST outputs y_{k-1}, y_{M-k-1}.
template <int M>
__device__ __forceinline__ void dst_post(const double2* s, const double2* __restrict__ tw2M, int k,
                                         double scale, double& yk, double& ym) {
  const double2 a = s[pad16(k)], bq = s[pad16(M - k)];
  const double2 w = __ldg(tw2M + k);  // e^{-2 pi i k/(2M)}
  const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
  const double2 iwQ = mul_si<1>(cmul(w, Q));
  // V_k = (P - iwQ)/2, V_{M-k} = conj(P + iwQ)/2; y = -scale*Im(V)  (dst.hpp:33-41)
  yk = -scale * 0.5 * (P.y - iwQ.y);
  ym = scale * 0.5 * (P.y + iwQ.y);
}

template <int LOGM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TauGeo<LOGM>::G::NT)
    k_tau_solve_1d(double2* __restrict__ Z, int ns, int n_rows, const double2* __restrict__ lam,
                   const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  using G = typename TauGeo<LOGM>::G;
  constexpr int M = G::M, B = G::B;
  extern __shared__ double2 smem[];
  double2* F = smem;
  double* D = reinterpret_cast<double*>(smem + B * padded(M));
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int g = blockIdx.x >> 1;
  const int r0 = g * B;
  const int nb = min(B, n_rows - r0);
  const double scale = sqrt(2.0 / double(M)) * 0.5;
  const double2* tw2M = twb + 2 * M;
  double* Zd = reinterpret_cast<double*>(Z);

  // 1. load my component of each row into the odd-extension packing
  for (int e = threadIdx.x; e < B * ns; e += blockDim.x) {
    const int b = e / ns, i = e - b * ns;
    const double x = b < nb ? Zd[2 * (size_t(r0 + b) * ns + i) + rank] : 0.0;
    pack_odd<M>(F + b * padded(M), i, x);
  }
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    comp(F + b * padded(M), 0, 0) = 0.0;
    comp(F + b * padded(M), pad16(M >> 1), 0) = 0.0;
  }
  __syncthreads();
  block_fft<LOGM, -1>(F, twb + M, B);
  // 2. first DST -> D
  for (int t = threadIdx.x; t < B * (M / 2); t += blockDim.x) {
    const int b = t / (M / 2), k = 1 + (t - b * (M / 2));
    double yk, ym;
    dst_post<M>(F + b * padded(M), tw2M, k, scale, yk, ym);
    D[b * M + k - 1] = yk;
    D[b * M + M - k - 1] = ym;
  }
  cluster.sync();
  // 3. divide by (lambda_n - dt sigma_i) with both components; repack my component
  const double* Dre = cluster.map_shared_rank(D, 0);
  const double* Dim = cluster.map_shared_rank(D, 1);
  for (int e = threadIdx.x; e < B * ns; e += blockDim.x) {
    const int b = e / ns, i = e - b * ns;
    double q = 0.0;
    if (b < nb) {
      const double2 l = lam[r0 + b];
      const double cr = l.x - dt * sigma[i], ci = l.y;
      const double ar = Dre[b * M + i], ai = Dim[b * M + i];
      // Smith's division (a)/(c)
      double qr, qi;
      if (fabs(cr) >= fabs(ci)) {
        const double rr = ci / cr, den = cr + ci * rr;
        qr = (ar + ai * rr) / den;
        qi = (ai - ar * rr) / den;
      } else {
        const double rr = cr / ci, den = cr * rr + ci;
        qr = (ar * rr + ai) / den;
        qi = (ai * rr - ar) / den;
      }
      q = rank == 0 ? qr : qi;
    }
    pack_odd<M>(F + b * padded(M), i, q);
  }
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    comp(F + b * padded(M), 0, 0) = 0.0;
    comp(F + b * padded(M), pad16(M >> 1), 0) = 0.0;
  }
  __syncthreads();
  block_fft<LOGM, -1>(F, twb + M, B);
  // 4. second DST -> my component of the row, in place in Z
  for (int t = threadIdx.x; t < B * (M / 2); t += blockDim.x) {
    const int b = t / (M / 2), k = 1 + (t - b * (M / 2));
    if (b >= nb) continue;
    double yk, ym;
    dst_post<M>(F + b * padded(M), tw2M, k, scale, yk, ym);
    const size_t base = size_t(r0 + b) * ns;
    Zd[2 * (base + k - 1) + rank] = yk;
    Zd[2 * (base + M - k - 1) + rank] = ym;
  }
  cluster.sync();  // keep D alive until the peer CTA has read it
}

// =====================================================================================
// launchers
// =====================================================================================
template <class K>
static cudaError_t prep(K kernel, size_t smem) {
  if (smem > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaSuccess;
}

#define FPC_DISPATCH_LOGM(logm, MAXLOG, CALL) \
  switch (logm) {                             \
    case 1: CALL(1); break;                   \
    case 2: CALL(2); break;                   \
    case 3: CALL(3); break;                   \
    case 4: CALL(4); break;                   \
    case 5: CALL(5); break;                   \
    case 6: CALL(6); break;                   \
    case 7: CALL(7); break;                   \
    case 8: CALL(8); break;                   \
    case 9: CALL(9); break;                   \
    case 10: CALL(10); break;                 \
    case 11: CALL(11); break;                 \
    case 12: CALL(12); break;                 \
    case 13: CALL(13); break;                 \
    default: return cudaErrorInvalidValue;    \
  }

cudaError_t launch_matvec_1d(const double* v, double* y, int n_space, int n_time, int log_m,
                             const double* eig_scaled, const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
#define CALL(LM)                                                                          \
  {                                                                                       \
    using G = Geo<LM, kTotMv>;                                                            \
    if ((err = prep(k_matvec_1d<LM>, G::SMEM)) != cudaSuccess) return err;                \
    k_matvec_1d<LM><<<(n_time + G::B - 1) / G::B, G::NT, G::SMEM, st>>>(                  \
        v, y, n_space, n_time, eig_scaled, tw_base);                                      \
  }
  if (log_m == 0) return cudaErrorInvalidValue;
  FPC_DISPATCH_LOGM(log_m, 13, CALL)
#undef CALL
  return cudaGetLastError();
}

static int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

cudaError_t launch_time_fwd(const double* v, double2* Z, int n_space, int n_time,
                            const double* scale_fwd, double s_in, const double2* tw_base,
                            cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2(n_time) - 1;
#define CALL(LM)                                                                          \
  {                                                                                       \
    using G = Geo<LM, kTotT>;                                                             \
    if ((err = prep(k_time_fwd<LM>, G::SMEM)) != cudaSuccess) return err;                 \
    k_time_fwd<LM><<<(n_space + G::B - 1) / G::B, G::NT, G::SMEM, st>>>(                  \
        v, Z, n_space, scale_fwd, s_in, tw_base);                                         \
  }
  FPC_DISPATCH_LOGM(lm, 13, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_time_inv(const double2* Z, double* z, int n_space, int n_time,
                            const double* scale_bwd, const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2(n_time) - 1;
#define CALL(LM)                                                                          \
  {                                                                                       \
    using G = Geo<LM, kTotT>;                                                             \
    if ((err = prep(k_time_inv<LM>, G::SMEM)) != cudaSuccess) return err;                 \
    k_time_inv<LM><<<(n_space + G::B - 1) / G::B, G::NT, G::SMEM, st>>>(Z, z, n_space,     \
                                                                        scale_bwd, tw_base); \
  }
  FPC_DISPATCH_LOGM(lm, 13, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_tau_solve_1d(double2* Z, int n_space, int n_rows, const double2* lambda,
                                const double* sigma, double dt, const double2* tw_base,
                                cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2(n_space + 1);
#define CALL(LM)                                                                          \
  {                                                                                       \
    using TG = TauGeo<LM>;                                                                \
    if ((err = prep(k_tau_solve_1d<LM>, TG::SMEM)) != cudaSuccess) return err;            \
    const int groups = (n_rows + TG::G::B - 1) / TG::G::B;                                \
    k_tau_solve_1d<LM><<<2 * groups, TG::G::NT, TG::SMEM, st>>>(Z, n_space, n_rows, lambda, \
                                                                 sigma, dt, tw_base);     \
  }
  FPC_DISPATCH_LOGM(lm, 13, CALL)
#undef CALL
  return cudaGetLastError();
}

}  // namespace fpc
