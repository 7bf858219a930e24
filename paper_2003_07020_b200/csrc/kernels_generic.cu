// kernels_generic.cu -- the PC apply for sizes the power-of-two kernels do not cover: any n_time
// (time FFT of length N_t) and any n_space (DST-I of length n, i.e. an FFT of length 2(n+1)).
//
// The reference's fft_inplace falls back to Bluestein's chirp-z for a non-power-of-two length
// (fft.hpp:69-101); this is that algorithm on the device: one CTA per sequence runs
//   a_j = x_j c_j (zero-padded to L = next_pow2(2 len - 1)),  A = FFT_L^-(a),  A *= B,
//   a = FFT_L^+(A),  x_k = c_k a_k / L,
// with the chirp c_m = e^{sign i pi (m^2 mod 2 len)/len} and B = FFT_L^-(b), b_m = conj(c_|m|)
// circularly, both built on the host exactly as fft.hpp:71-89 builds them.  The transforms of
// length L are the CTA-level Stockham engine of fft_block.cuh.  Around it, element-wise kernels
// restate the rest of the apply (alpha_circulant.hpp:137-199 with InnerSweep and the dst1 odd
// extension dst.hpp:21-43): the scaled time input, the odd extension / extraction of each DST
// sequence (with the shifted-eigenvalue step of tau.hpp:98-136 fused into the extraction) and the
// real output with the inverse scaling.  It keeps a full [N_t][N_s] complex spectrum and one
// odd-extension buffer: general, not fast -- the BASELINE configurations never take this path.
#include <algorithm>

#include "fft_block.cuh"
#include "kernels.cuh"

namespace fpc {

namespace {

template <int LOGL>
struct BlueGeo {
  static constexpr int L = 1 << LOGL;
  static constexpr int E = L < 16 ? L : 16;
  static constexpr int NT = L / E;
  static constexpr size_t SMEM = size_t(padded(L)) * sizeof(double2);
};

// sequence s, element j of a strided batch: data + base(s) + j * es with
// base(s) = (s / inner) * outer_stride + (s % inner) * inner_stride
struct SeqMap {
  long long inner, outer_stride, inner_stride, es;
  __device__ __forceinline__ size_t base(long long s) const {
    return size_t((s / inner) * outer_stride + (s % inner) * inner_stride);
  }
};

template <int LOGL>
__global__ void __launch_bounds__(BlueGeo<LOGL>::NT)
    k_bluestein(double2* __restrict__ data, int len, SeqMap map, const double2* __restrict__ chirp,
                const double2* __restrict__ bhat, double inv_l, const double2* __restrict__ twb) {
  using G = BlueGeo<LOGL>;
  constexpr int L = G::L;
  extern __shared__ double2 smem[];
  double2* x = data + map.base(blockIdx.x);
  for (int j = threadIdx.x; j < L; j += G::NT)
    smem[pad16(j)] = j < len ? cmul(x[size_t(j) * map.es], __ldg(chirp + j)) : make_double2(0.0, 0.0);
  __syncthreads();
  block_fft<LOGL, -1, padded(L), G::E>(smem, twb + L, 1);
  for (int j = threadIdx.x; j < L; j += G::NT) smem[pad16(j)] = cmul(smem[pad16(j)], __ldg(bhat + j));
  __syncthreads();
  block_fft<LOGL, 1, padded(L), G::E>(smem, twb + L, 1);
  for (int k = threadIdx.x; k < len; k += G::NT)
    x[size_t(k) * map.es] = cscale(cmul(__ldg(chirp + k), smem[pad16(k)]), inv_l);
}

// power-of-two length: the plain transform (fft_pow2's role in fft_inplace, fft.hpp:95-101)
template <int LOGL, int S>
__global__ void __launch_bounds__(BlueGeo<LOGL>::NT)
    k_dft_pow2(double2* __restrict__ data, SeqMap map, const double2* __restrict__ twb) {
  using G = BlueGeo<LOGL>;
  constexpr int L = G::L;
  extern __shared__ double2 smem[];
  double2* x = data + map.base(blockIdx.x);
  for (int j = threadIdx.x; j < L; j += G::NT) smem[pad16(j)] = x[size_t(j) * map.es];
  __syncthreads();
  block_fft<LOGL, S, padded(L), G::E>(smem, twb + L, 1);
  for (int k = threadIdx.x; k < L; k += G::NT) x[size_t(k) * map.es] = smem[pad16(k)];
}

// U[k][p] = s_in scale_fwd[k] v[k][p] as complex (alpha_circulant.hpp:146-152)
__global__ void k_gen_time_in(const double* __restrict__ v, double2* __restrict__ U, size_t n, int ns,
                              const double* __restrict__ sf, double s_in) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    const int k = int(e / size_t(ns));
    U[e] = make_double2(__ldg(sf + k) * (s_in * v[e]), 0.0);
  }
}

// z[k][p] = Re((scale_bwd[k] / N_t) U[k][p])  (alpha_circulant.hpp:187-198)
__global__ void k_gen_time_out(const double2* __restrict__ U, double* __restrict__ z, size_t n, int ns,
                               const double* __restrict__ sb, double inv_nt) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    const int k = int(e / size_t(ns));
    z[e] = (__ldg(sb + k) * inv_nt) * U[e].x;
  }
}

// the same with the imaginary-residue guard's partial sums (alpha_circulant.hpp:188-198):
// partial[blk * 2 + {0, 1}] = {sum Im^2, sum |.|^2} of the scaled complex output
constexpr int kGuardThreads = 256;
__global__ void __launch_bounds__(kGuardThreads)
    k_gen_time_out_guard(const double2* __restrict__ U, double* __restrict__ z, size_t n, int ns,
                         const double* __restrict__ sb, double inv_nt, double* __restrict__ partial) {
  double im2 = 0.0, tot2 = 0.0;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    const int k = int(e / size_t(ns));
    const double sc = __ldg(sb + k) * inv_nt;
    const double2 u = cscale(U[e], sc);
    z[e] = u.x;
    im2 = fma(u.y, u.y, im2);
    tot2 = fma(u.x, u.x, fma(u.y, u.y, tot2));
  }
  __shared__ double red[kGuardThreads / 32][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) {
    im2 += __shfl_xor_sync(0xffffffffu, im2, off);
    tot2 += __shfl_xor_sync(0xffffffffu, tot2, off);
  }
  if (lane == 0) {
    red[warp][0] = im2;
    red[warp][1] = tot2;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double a = 0.0;
    for (int w = 0; w < kGuardThreads / 32; ++w) a += red[w][threadIdx.x];
    partial[blockIdx.x * 2 + threadIdx.x] = a;
  }
}

// the frequencies N_t/2 < q < N_t as conj of N_t - q (alpha_circulant.hpp:167-175)
__global__ void k_gen_mirror(double2* __restrict__ U, int nt, int ns, int h) {
  const size_t n = size_t(nt - h) * size_t(ns);
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    const int q = h + int(e / size_t(ns));
    const int p = int(e % size_t(ns));
    U[size_t(q) * ns + p] = cconj(U[size_t(nt - q) * ns + p]);
  }
}

// odd extension of every sequence (dst.hpp:27-31): D[s][0] = 0, D[s][j+1] = u_j,
// D[s][n+1] = 0, D[s][P-1-j] = -u_j, P = 2(n+1)
__global__ void k_gen_odd_ext(const double2* __restrict__ U, SeqMap map, int n, long long count,
                              double2* __restrict__ D) {
  const int P = 2 * (n + 1);
  const size_t tot = size_t(count) * size_t(P);
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += size_t(gridDim.x) * blockDim.x) {
    const long long s = (long long)(e / size_t(P));
    const int m = int(e % size_t(P));
    double2 val = make_double2(0.0, 0.0);
    if (m >= 1 && m <= n) val = U[map.base(s) + size_t(m - 1) * map.es];
    else if (m >= n + 2) {
      const double2 u = U[map.base(s) + size_t(P - 1 - m) * map.es];
      val = make_double2(-u.x, -u.y);
    }
    D[e] = val;
  }
}

// y_i = scale * (i * D[s][i+1]) (dst.hpp:34-40), then MODE 1: y_i /= (lambda_f - dt sigma_i),
// MODE 2: y_i *= (lambda_f - dt sigma_i) (tau.hpp:109-118); f = s / per_freq, sigma index =
// in-plane offset of the element
template <int MODE>
__global__ void k_gen_dst_out(const double2* __restrict__ D, SeqMap map, int n, long long count,
                              double2* __restrict__ U, double scale, long long per_freq, long long plane,
                              const double2* __restrict__ lam, const double* __restrict__ sigma, double dt) {
  const int P = 2 * (n + 1);
  const size_t tot = size_t(count) * size_t(n);
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += size_t(gridDim.x) * blockDim.x) {
    const long long s = (long long)(e / size_t(n));
    const int i = int(e % size_t(n));
    const double2 d = D[size_t(s) * P + i + 1];
    double2 y = cscale(make_double2(-d.y, d.x), scale);
    const size_t off = map.base(s) + size_t(i) * map.es;
    if constexpr (MODE != 0) {
      const long long f = s / per_freq;
      const double2 l = __ldg(lam + f);
      y = shift_apply<MODE>(y, l.x - dt * __ldg(sigma + (off - size_t(f * plane))), l.y);
    }
    U[off] = y;
  }
}

int ilog2c(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

unsigned ew_grid(size_t n) { return unsigned(std::min<size_t>((n + 255) / 256, size_t(148) * 16)); }

}  // namespace

cudaError_t launch_bluestein(double2* data, int len, long long count, long long inner, long long outer_stride,
                             long long inner_stride, long long es, const double2* chirp, const double2* bhat,
                             const double2* tw_base, cudaStream_t st, int sign) {
  if (len >= 2 && (len & (len - 1)) == 0) {  // power of two: no chirp (as the reference's fft_inplace)
    const int lg = ilog2c(len);
    if (lg > 13 || count <= 0) return cudaErrorInvalidValue;
    const SeqMap m{inner, outer_stride, inner_stride, es};
    cudaError_t e = cudaSuccess;
#define FPC_DFT2(LL)                                                                                       \
  case LL: {                                                                                               \
    using G = BlueGeo<LL>;                                                                                 \
    if (sign > 0) {                                                                                        \
      if (G::SMEM > 48 * 1024 && (e = cudaFuncSetAttribute(k_dft_pow2<LL, 1>,                                \
                                                           cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                                           int(G::SMEM))) != cudaSuccess)                 \
        return e;                                                                                          \
      k_dft_pow2<LL, 1><<<unsigned(count), G::NT, G::SMEM, st>>>(data, m, tw_base);                        \
    } else {                                                                                               \
      if (G::SMEM > 48 * 1024 && (e = cudaFuncSetAttribute(k_dft_pow2<LL, -1>,                               \
                                                           cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                                           int(G::SMEM))) != cudaSuccess)                 \
        return e;                                                                                          \
      k_dft_pow2<LL, -1><<<unsigned(count), G::NT, G::SMEM, st>>>(data, m, tw_base);                       \
    }                                                                                                      \
    note_launch();                                                                                         \
  } break;
    switch (lg) {
      FPC_DFT2(1) FPC_DFT2(2) FPC_DFT2(3) FPC_DFT2(4) FPC_DFT2(5) FPC_DFT2(6) FPC_DFT2(7) FPC_DFT2(8)
      FPC_DFT2(9) FPC_DFT2(10) FPC_DFT2(11) FPC_DFT2(12) FPC_DFT2(13)
      default:
        return cudaErrorInvalidValue;
    }
#undef FPC_DFT2
    return cudaGetLastError();
  }
  const int logl = ilog2c(2LL * len - 1);
  if (logl > 13 || count <= 0) return cudaErrorInvalidValue;
  const SeqMap map{inner, outer_stride, inner_stride, es};
  const double inv_l = 1.0 / double(1LL << logl);
  cudaError_t e = cudaSuccess;
#define FPC_BLUE(LL)                                                                                    \
  case LL: {                                                                                            \
    using G = BlueGeo<LL>;                                                                              \
    if (G::SMEM > 48 * 1024 &&                                                                          \
        (e = cudaFuncSetAttribute(k_bluestein<LL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::SMEM))) != \
            cudaSuccess)                                                                                \
      return e;                                                                                         \
    k_bluestein<LL><<<unsigned(count), G::NT, G::SMEM, st>>>(data, len, map, chirp, bhat, inv_l, tw_base); \
    note_launch();                                                                                      \
  } break;
  switch (logl) {
    FPC_BLUE(2) FPC_BLUE(3) FPC_BLUE(4) FPC_BLUE(5) FPC_BLUE(6) FPC_BLUE(7) FPC_BLUE(8) FPC_BLUE(9)
    FPC_BLUE(10) FPC_BLUE(11) FPC_BLUE(12) FPC_BLUE(13)
    default:
      return cudaErrorInvalidValue;
  }
#undef FPC_BLUE
  return cudaGetLastError();
}

cudaError_t launch_gen_time_in(const double* v, double2* U, int ns, int nt, const double* sf, double s_in,
                               cudaStream_t st) {
  const size_t n = size_t(ns) * size_t(nt);
  k_gen_time_in<<<ew_grid(n), 256, 0, st>>>(v, U, n, ns, sf, s_in);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_time_out(const double2* U, double* z, int ns, int nt, const double* sb, cudaStream_t st) {
  const size_t n = size_t(ns) * size_t(nt);
  k_gen_time_out<<<ew_grid(n), 256, 0, st>>>(U, z, n, ns, sb, 1.0 / double(nt));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_time_out_guard(const double2* U, double* z, int ns, int nt, const double* sb, double* partial,
                                      cudaStream_t st) {
  const size_t n = size_t(ns) * size_t(nt);
  k_gen_time_out_guard<<<dots_grid(), kGuardThreads, 0, st>>>(U, z, n, ns, sb, 1.0 / double(nt), partial);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_mirror(double2* U, int nt, int ns, int h, cudaStream_t st) {
  if (h >= nt) return cudaSuccess;
  const size_t n = size_t(nt - h) * size_t(ns);
  k_gen_mirror<<<ew_grid(n), 256, 0, st>>>(U, nt, ns, h);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_dst(double2* U, double2* D, int n, long long count, long long inner, long long outer_stride,
                           long long inner_stride, long long es, const double2* chirp, const double2* bhat,
                           const double2* tw_base, int mode, long long per_freq, long long plane, const double2* lam,
                           const double* sigma, double dt, cudaStream_t st) {
  const SeqMap map{inner, outer_stride, inner_stride, es};
  const int P = 2 * (n + 1);
  k_gen_odd_ext<<<ew_grid(size_t(count) * P), 256, 0, st>>>(U, map, n, count, D);
  note_launch();
  // the odd extensions are contiguous rows of P: FFT_P^- of each (dst.hpp:32)
  cudaError_t e = launch_bluestein(D, P, count, 1, P, 0, 1, chirp, bhat, tw_base, st, -1);
  if (e != cudaSuccess) return e;
  const double scale = std::sqrt(2.0 / double(n + 1)) * 0.5;
  const unsigned g = ew_grid(size_t(count) * n);
  if (mode == 0)
    k_gen_dst_out<0><<<g, 256, 0, st>>>(D, map, n, count, U, scale, per_freq, plane, lam, sigma, dt);
  else if (mode == 1)
    k_gen_dst_out<1><<<g, 256, 0, st>>>(D, map, n, count, U, scale, per_freq, plane, lam, sigma, dt);
  else
    k_gen_dst_out<2><<<g, 256, 0, st>>>(D, map, n, count, U, scale, per_freq, plane, lam, sigma, dt);
  note_launch();
  return cudaGetLastError();
}

}  // namespace fpc
