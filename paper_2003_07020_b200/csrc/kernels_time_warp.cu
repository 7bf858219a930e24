// kernels_time_warp.cu -- the preconditioner's time FFTs (alpha_circulant.hpp:146-156 forward,
// 167-198 inverse) for n_time = 1024 on warp-owned transforms: one column per warp.
//
// The 2-CTA split kernels (kernels_tsplit.cu) move a column tile through three shared-memory
// Stockham passes with CTA and cluster barriers between them (config 3: 33-36% of the HBM roof,
// stalls: long scoreboard 32-39%, barrier 11-19%, membar 7-12%).  Here the packed 512-point
// transform of a column is held by one warp (16 registers per lane, the 16 x 32 scheme of
// warp_dst32.cuh: one transpose), the Hermitian pre/post-processing exchanges mirrors by shuffles,
// and the only CTA-wide steps are the two staging phases: a CTA owns 8 adjacent columns, reads
// their row segments (64 bytes forward, 128 bytes inverse) with asynchronous copies straight into
// the warps' buffers, and writes the results back through the same buffers in whole row segments.
// 16 warps per SM (two CTAs), 8.4 KB of shared memory per warp: the buffer is the staging area,
// then the transpose tile, then the output area.
#include <cstdlib>

#include "bulk_copy.cuh"
#include "kernels.cuh"
#include "warp_dst32.cuh"

namespace fpc {

namespace {

#ifndef FPC_TW_COLS
#define FPC_TW_COLS 8
#endif
constexpr int kTwCols = FPC_TW_COLS;  // columns (= warps) per CTA: 8 (two CTAs per SM) or 16 (one)
constexpr int kTwBuf = 8592;    // bytes per warp buffer: >= the 16 x 33 tile (8448) and the 513-row
                                // spectrum (8208); = 16 mod 128, so the 8 buffers' equal offsets
                                // fall in 8 different 16-byte banks
constexpr int kTwSkew = kTwCols == 8 ? 16 : 0;  // extra bytes per column for the 8-byte phases (4 rows x 8 columns of
                                // a warp instruction then cover all sixteen 8-byte banks twice)
static_assert(kTwBuf % 16 == 0 && kTwBuf % 128 == 16, "buffer stride");
static_assert(16 * kW32LD * 16 <= kTwBuf && (kTwCols - 1) * kTwSkew + 8192 <= kTwBuf && 513 * 16 <= kTwBuf, "buffer");

}  // namespace

// K2: Z[n][p] = sum_k s_in scale_fwd[k] v[k][p] e^{+2 pi i kn/Nt}, n = 0..Nt/2, Nt = 1024: the real
// series packed into M = 512 complex points c_m = (x_{2m}, x_{2m+1}), X = FFT_M^+(c), and
//   Z_n = (1/2) [ (X_n + conj X_{M-n}) - i e^{+2 pi i n/Nt} (X_n - conj X_{M-n}) ],  Z_M = Re X_0 - Im X_0
// (the per-bin arithmetic of k_time_fwd, kernels_1d.cu; every lane forms its own 16 bins, the mirror
// X_{M-n} of bin n = t + 32 p coming from lane 32 - t, register 15 - p).
__global__ void __launch_bounds__(32 * kTwCols, 16 / kTwCols)
    k_time_fwd_w512(const double* __restrict__ v, double2* __restrict__ Z, int ns, const double* __restrict__ sf,
                    double s_in, const double2* __restrict__ twb) {
  constexpr int M = 512, NTIME = 1024, C = kTwCols, RS = 32;
  extern __shared__ __align__(128) unsigned char tsm[];
  const int tid = int(threadIdx.x);
  const int p0 = int(blockIdx.x) * C;
  const int ncol = min(C, ns - p0);
  const int c = tid % C, k0 = tid / C;
  const bool okc = c < ncol;
  {
    double* dst = reinterpret_cast<double*>(tsm + c * kTwBuf + c * kTwSkew);
    const double* src = v + p0 + (okc ? c : 0);
#pragma unroll 8
    for (int k = k0; k < NTIME; k += RS) cp_async8_zfill(dst + k, src + size_t(k) * ns, okc);
    cp_async_wait_all();
  }
  __syncthreads();
  const int w = tid >> 5, t = tid & 31;
  double2 z[16];
  {
    const double2* in = reinterpret_cast<const double2*>(tsm + w * kTwBuf + w * kTwSkew);
    const double2* sf2 = reinterpret_cast<const double2*>(sf);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int m = t + 32 * r;
      const double2 x = in[m], s = __ldg(sf2 + m);
      z[r] = make_double2(s.x * (s_in * x.x), s.y * (s_in * x.y));
    }
  }
  __syncwarp();
  double2* xs = reinterpret_cast<double2*>(tsm + w * kTwBuf);
  warp_fft_16x32<1>(z, xs, t, twb);  // lane t: X_{t + 32 p}
  const double2* twT = twb + NTIME;
  const int src = (32 - t) & 31;
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    const int n = t + 32 * p;
    const double2 a = z[p];
    double2 bq;
    bq.x = __shfl_sync(0xffffffffu, z[15 - p].x, src);
    bq.y = __shfl_sync(0xffffffffu, z[15 - p].y, src);
    if (t == 0) bq = z[(16 - p) & 15];
    const double2 wn = cconj(__ldg(twT + n));  // e^{+2 pi i n/Nt}
    const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
    const double2 iwQ = mul_si<1>(cmul(wn, Q));
    double2 o = cscale(csub(P, iwQ), 0.5);
    if (p == 0 && t == 0) {
      o = make_double2(a.x + a.y, 0.0);
      xs[M] = make_double2(a.x - a.y, 0.0);
    }
    xs[n] = o;
  }
  __syncthreads();
  if (okc) {
    const double2* ob = reinterpret_cast<const double2*>(tsm + c * kTwBuf);
    double2* zc = Z + p0 + c;
#pragma unroll 8
    for (int n = k0; n <= M; n += RS) zc[size_t(n) * ns] = ob[n];
  }
}

// K4: z[k][p] = (scale_bwd[k] / Nt) sum_n Z_n e^{-2 pi i kn/Nt} over the Hermitian extension of the
// half spectrum Z_0..Z_M: s_m = (Z_m + conj Z_{M-m}) + i e^{-2 pi i m/Nt} (Z_m - conj Z_{M-m})
// (m = 0: (Z_0 + Z_M) + i (Z_0 - Z_M), as k_time_inv), c = FFT_M^-(s), z_{2m} = Re c_m, z_{2m+1} = Im c_m.
__global__ void __launch_bounds__(32 * kTwCols, 16 / kTwCols)
    k_time_inv_w512(const double2* __restrict__ Z, double* __restrict__ z, int ns, const double* __restrict__ sb,
                    const double2* __restrict__ twb) {
  constexpr int M = 512, NTIME = 1024, C = kTwCols, RS = 32;
  extern __shared__ __align__(128) unsigned char tsm[];
  const int tid = int(threadIdx.x);
  const int p0 = int(blockIdx.x) * C;
  const int ncol = min(C, ns - p0);
  const int c = tid % C, k0 = tid / C;
  const bool okc = c < ncol;
  {
    double2* dst = reinterpret_cast<double2*>(tsm + c * kTwBuf);
    const double2* src = Z + p0 + (okc ? c : 0);
#pragma unroll 8
    for (int n = k0; n <= M; n += RS) cp_async16_zfill(dst + n, src + size_t(n) * ns, okc);
    cp_async_wait_all();
  }
  __syncthreads();
  const int w = tid >> 5, t = tid & 31;
  double2* xs = reinterpret_cast<double2*>(tsm + w * kTwBuf);
  const double2* twT = twb + NTIME;
  double2 s[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int m = t + 32 * r;
    const double2 ya = xs[m], yb = xs[M - m];
    if (r == 0 && t == 0) {
      const double2 A = cadd(ya, yb), Bv = csub(ya, yb);
      s[r] = cadd(A, mul_si<1>(Bv));
    } else {
      const double2 wn = __ldg(twT + m);  // e^{-2 pi i m/Nt}
      const double2 A = cadd(ya, cconj(yb));
      const double2 Bn = cmul(csub(ya, cconj(yb)), wn);
      s[r] = cadd(A, mul_si<1>(Bn));
    }
  }
  __syncwarp();
  warp_fft_16x32<-1>(s, xs, t, twb);  // lane t: c_{t + 32 p}
  {
    double2* ob = reinterpret_cast<double2*>(tsm + w * kTwBuf + w * kTwSkew);
    const double2* sb2 = reinterpret_cast<const double2*>(sb);
    const double inv_nt = 1.0 / double(NTIME);
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const int m = t + 32 * p;
      const double2 q = __ldg(sb2 + m);
      ob[m] = make_double2((q.x * inv_nt) * s[p].x, (q.y * inv_nt) * s[p].y);
    }
  }
  __syncthreads();
  if (okc) {
    const double* ob = reinterpret_cast<const double*>(tsm + c * kTwBuf + c * kTwSkew);
    double* zc = z + p0 + c;
#pragma unroll 8
    for (int k = k0; k < NTIME; k += RS) zc[size_t(k) * ns] = ob[k];
  }
}

// n_time = 1024 with at least a wave of column tiles; FPC_TIME_WARP=0 keeps the split kernels (A/B)
bool time_warp_supported(int n_space, int n_time) {
  static const int min_cols = [] {
    const char* e = std::getenv("FPC_TIME_WARP");
    if (e && e[0] == '0') return -1;
    const char* m = std::getenv("FPC_TIME_WARP_MIN_COLS");
    return (m && m[0]) ? std::atoi(m) : 2 * 148 * kTwCols;
  }();
  return min_cols >= 0 && n_time == 1024 && n_space >= min_cols;
}

static cudaError_t prep_tw(const void* kernel, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                              carveout_pct(smem, 32 * kTwCols));
}

cudaError_t launch_time_fwd_warp(const double* v, double2* Z, int n_space, int n_time, const double* scale_fwd,
                                 double s_in, const double2* tw_base, cudaStream_t st) {
  if (n_time != 1024) return cudaErrorNotSupported;
  const size_t smem = size_t(kTwCols) * kTwBuf;
  cudaError_t e = prep_tw((const void*)k_time_fwd_w512, smem);
  if (e != cudaSuccess) return e;
  k_time_fwd_w512<<<(n_space + kTwCols - 1) / kTwCols, 32 * kTwCols, smem, st>>>(v, Z, n_space, scale_fwd, s_in,
                                                                               tw_base);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_time_inv_warp(const double2* Z, double* z, int n_space, int n_time, const double* scale_bwd,
                                 const double2* tw_base, cudaStream_t st) {
  if (n_time != 1024) return cudaErrorNotSupported;
  const size_t smem = size_t(kTwCols) * kTwBuf;
  cudaError_t e = prep_tw((const void*)k_time_inv_w512, smem);
  if (e != cudaSuccess) return e;
  k_time_inv_w512<<<(n_space + kTwCols - 1) / kTwCols, 32 * kTwCols, smem, st>>>(Z, z, n_space, scale_bwd, tw_base);
  note_launch();
  return cudaGetLastError();
}

}  // namespace fpc
