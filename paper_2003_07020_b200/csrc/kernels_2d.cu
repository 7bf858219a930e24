// kernels_2d.cu -- 2D lattice kernels: the x-direction half of RieszJacobian2D::apply
// (jacobian.hpp:88-93, strided columns) and the column passes of the 2D tau solves
// (tau.hpp:79-96 dst_lattice_inplace, columns after rows).  The contiguous-row halves reuse the
// 1D kernels (launch_matvec_rows / launch_dst_rows in kernels_1d.cu).
//
// Lattice p = ix*n + iy (x slow, problems.hpp:164-165).  A CTA owns C consecutive iy columns of one
// time block (matvec) or one frequency row (tau): each lattice row ix contributes C contiguous
// values (coalesced), and each column becomes one smem FFT buffer.
#include <algorithm>
#include <cstdlib>

#include "dst_block.cuh"
#include "fft_block.cuh"
#include "kernels.cuh"

namespace fpc {

namespace {

__host__ __device__ constexpr int skew2(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}
// Column-buffer stride for the column-fastest phases (loads, eigenvalue product, divide, stores:
// lane = column c fastest, then the slot).  A quarter warp of 16-byte accesses covers 8/C slots of
// each of C buffers (C <= 8), so the buffers must start 8/C bank groups apart (stride = 8/C mod 8):
// C = 4 -> 2, C = 2 -> 4.  The 8-byte halves of the loads/epilogue then also land in distinct banks
// (C = 4: 8 banks apart).  C >= 8 keeps the one-group skew (same slot, 8 consecutive buffers).
__host__ __device__ constexpr int skew_cols(int m, int c) {
  return m < 16 ? padded(m)
                : padded(m) + (((c == 4 ? 2 : c == 2 ? 4 : 1) - padded(m) % 8 + 8) % 8);
}
__device__ __forceinline__ double& comp2(double2* s, int slot_padded, int c) {
  return reinterpret_cast<double*>(s + slot_padded)[c];
}

template <class K>
cudaError_t prep2(K kernel, size_t smem, int threads = 1024) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct(smem, threads));
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaSuccess;
}

int ilog2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

constexpr int kTot2 = 4096;
#ifndef FPC_COLS_RED
#define FPC_COLS_RED 1
#endif

template <int LOGM>
struct ColGeo {
  static constexpr int M = 1 << LOGM;
  static constexpr int E = M < 16 ? M : 16;
  static constexpr int C = kTot2 / M > 0 ? kTot2 / M : 1;  // columns per CTA
  static constexpr int NT = C * M / E;
  static constexpr int BS = C > 1 ? skew_cols(M, C) : padded(M);
  static constexpr int BH = C > 1 ? skew2(M / 2) : padded(M / 2);  // DCT-III scratch (tau)
  static constexpr size_t SMEM = size_t(C) * (BS + BH) * sizeof(double2);  // tau: FFT + DCT-III buffers
  static constexpr size_t SMEM_MV = size_t(C) * BS * sizeof(double2);      // matvec: FFT buffers only
};

}  // namespace

// ------------------------------------------------------------------------------------------
// y[k][ix][iy] += (dt sx / (2L)) * (T_x v[k][.][iy])[ix]  for C columns iy of time block k.
// eig = dt*sx*eig(Tx)/(2L) pre-folded (the sign: y = c - dt*A v, A = -sx Tx (x) I - ...).
// ------------------------------------------------------------------------------------------
template <int LOGM>
__global__ void __launch_bounds__(ColGeo<LOGM>::NT, (ColGeo<LOGM>::NT <= 256 ? 2 : 1))
    k_matvec_2d_cols(const double* __restrict__ v, double* __restrict__ y, int n,
                     const double* __restrict__ eig, const double2* __restrict__ twb) {
  using G = ColGeo<LOGM>;
  constexpr int M = G::M, C = G::C, NT = G::NT, BS = G::BS, L = 2 * M, E = G::E;
  constexpr int U = 8;
  extern __shared__ double2 smem[];
  const int tiles = (n + C - 1) / C;
  const int k = blockIdx.x / tiles;
  const int iy0 = (blockIdx.x - k * tiles) * C;
  const size_t base = size_t(k) * n * n;

  // load columns: element (ix, c) -> buffer c, packed slot ix/2 (real packing of length L); only
  // the n real rows are read (16 loads in flight per thread), the padding is zero-filled apart
  constexpr int UL = 16;
  for (int e0 = threadIdx.x; e0 < C * n; e0 += UL * NT) {
    double x[UL];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int e = e0 + u * NT;
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      x[u] = (e < C * n && iy < n) ? v[base + size_t(ix) * n + iy] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int e = e0 + u * NT;
      if (e < C * n) {
        const int c = e % C, ix = e / C;
        comp2(smem, c * BS + pad16(ix >> 1), ix & 1) = x[u];
      }
    }
  }
  {
    const int s0 = (n + 1) >> 1;  // first slot with both entries at ix >= n
    for (int t = threadIdx.x; t < C * M; t += NT) {
      const int c = t / M, m = t - c * M;
      if (m >= s0) smem[c * BS + pad16(m)] = make_double2(0.0, 0.0);
      else if ((n & 1) && m == s0 - 1) comp2(smem, c * BS + pad16(m), 1) = 0.0;
    }
  }
  __syncthreads();
  block_fft<LOGM, -1, BS, E>(smem, twb + M, C);
  const double2* twL = twb + L;
  for (int t = threadIdx.x; t < C * (M / 2 + 1); t += NT) {
    const int c = t % C, kk = t / C;
    double2* s = smem + c * BS;
    if (kk == 0) {
      const double2 z = s[0];
      const double y0 = eig[0] * (2.0 * (z.x + z.y));
      const double ym = eig[M] * (2.0 * (z.x - z.y));
      s[0] = make_double2(y0 + ym, y0 - ym);
    } else {
      const int i1 = pad16(kk), i2 = pad16(M - kk);
      const double2 w = __ldg(twL + kk);
      const double ek = __ldg(eig + kk), em = __ldg(eig + M - kk);
      const double2 a = s[i1], bq = s[i2];
      const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
      const double2 iwQ = mul_si<1>(cmul(w, Q));
      const double2 Yk = cscale(csub(P, iwQ), ek);
      const double2 Ym = cscale(cconj(cadd(P, iwQ)), em);
      const double2 A = cadd(Yk, cconj(Ym));
      const double2 D = csub(Yk, cconj(Ym));
      s[i1] = cadd(A, mul_si<1>(cmul(D, cconj(w))));
      if (kk != M - kk) s[i2] = cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
    }
  }
  __syncthreads();
  block_fft<LOGM, 1, BS, E>(smem, twb + M, C);
#if FPC_COLS_RED
  // y += x-direction term as reductions performed at the L2 (RED.ADD.F64, no return value): every
  // element receives exactly one add -- the same double as load-add-store -- without the strided
  // read of y or the wait for it (B200 config 2: matvec 667 -> 592 us; kernels_warp.cu)
  for (int e = threadIdx.x; e < C * n; e += NT) {
    const int c = e % C, ix = e / C;
    const int iy = iy0 + c;
    if (iy < n) atomicAdd(y + base + size_t(ix) * n + iy, comp2(smem, c * BS + pad16(ix >> 1), ix & 1));
  }
  return;
#endif
  // y += x-direction term: the read-modify-write batched 8 deep (latency bound otherwise)
  constexpr int UE = 8;
  for (int e0 = threadIdx.x; e0 < C * n; e0 += UE * NT) {
    double yo[UE];
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      const int e = e0 + u * NT;
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      yo[u] = (e < C * n && iy < n) ? y[base + size_t(ix) * n + iy] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      const int e = e0 + u * NT;
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      if (e < C * n && iy < n) y[base + size_t(ix) * n + iy] = yo[u] + comp2(smem, c * BS + pad16(ix >> 1), ix & 1);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Column pass of the 2D tau solve for frequency row r: DST over ix of C columns, divide by
// (lambda_r - dt sigma[ix*n + iy]), DST over ix again.  Rows (iy) are done before and after by
// launch_dst_rows.
// ------------------------------------------------------------------------------------------
template <int LOGM, int MODE>  // MODE 1: solve (divide), 2: forward action (multiply), 0: one DST only
__global__ void __launch_bounds__(ColGeo<LOGM>::NT, (ColGeo<LOGM>::NT <= 256 ? 2 : 1))
    k_tau_2d_cols(double2* __restrict__ Z, int n, const double2* __restrict__ lam,
                  const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  using G = ColGeo<LOGM>;
  constexpr int M = G::M, C = G::C, NT = G::NT, BS = G::BS, E = G::E;
  constexpr int NSR = M - 1;  // column length n
  constexpr int U = 16;       // loads in flight per thread (these phases are latency bound)
  extern __shared__ double2 smem[];
  double2* hbuf = smem + C * BS;  // DCT-III scratch columns (dst_block.cuh)
  constexpr int BH = G::BH;
  const int tiles = (NSR + C - 1) / C;
  const int r = blockIdx.x / tiles;
  const int iy0 = (blockIdx.x - r * tiles) * C;
  double2* Zr = Z + size_t(r) * NSR * NSR;
  const double scale = sqrt(2.0 / double(M));
  (void)n;

  for (int e0 = threadIdx.x; e0 < C * NSR; e0 += U * NT) {
    double2 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      x[u] = (e < C * NSR && iy < NSR) ? Zr[size_t(ix) * NSR + iy] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      if (e < C * NSR) {
        const int c = e % C, ix = e / C;
        smem[c * BS + pad16(ix + 1)] = x[u];
      }
    }
  }
  __syncthreads();
  if constexpr (MODE == 0) {  // the column DST of the 2D lattice transform (commuted ordering)
    block_dst<LOGM, BS, BH, 0>(smem, hbuf, twb, scale);
    for (int e = threadIdx.x; e < C * NSR; e += NT) {
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      if (iy >= NSR) continue;
      Zr[size_t(ix) * NSR + iy] = smem[c * BS + pad16(ix)];
    }
    return;
  }
  block_dst<LOGM, BS, BH, 1>(smem, hbuf, twb, scale);
  const double2 l = __ldg(lam + r);
  for (int e0 = threadIdx.x; e0 < C * NSR; e0 += U * NT) {
    double sg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      sg[u] = (e < C * NSR && iy < NSR) ? __ldg(sigma + size_t(ix) * NSR + iy) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int c = e % C, ix = e / C;
      const int iy = iy0 + c;
      if (e >= C * NSR || iy >= NSR) continue;
      double2* s = smem + c * BS + pad16(ix + 1);
      *s = shift_apply<MODE>(*s, l.x - dt * sg[u], l.y);
    }
  }
  __syncthreads();
  block_dst<LOGM, BS, BH, 0>(smem, hbuf, twb, scale);
  for (int e = threadIdx.x; e < C * NSR; e += NT) {
    const int c = e % C, ix = e / C;
    const int iy = iy0 + c;
    if (iy >= NSR) continue;
    Zr[size_t(ix) * NSR + iy] = smem[c * BS + pad16(ix)];
  }
}

// ------------------------------------------------------------------------------------------
// time levels (2j, 2j+1) as one complex level: U[j][p] = s (v[2j][p] + i v[2j+1][p]), and back.
// The spatial transforms are real-linear, so a complex transform of the pair is the pair of real
// transforms (the commuted ordering's DST per time level).
__global__ void k_pack_pairs(const double* __restrict__ v, double2* __restrict__ U, int ns, size_t npairs_ns,
                             double s) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < npairs_ns; e += size_t(gridDim.x) * blockDim.x) {
    const size_t j = e / size_t(ns), p = e - j * size_t(ns);
    U[e] = make_double2(s * v[(2 * j) * size_t(ns) + p], s * v[(2 * j + 1) * size_t(ns) + p]);
  }
}
__global__ void k_unpack_pairs(const double2* __restrict__ U, double* __restrict__ v, int ns, size_t npairs_ns) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < npairs_ns; e += size_t(gridDim.x) * blockDim.x) {
    const size_t j = e / size_t(ns), p = e - j * size_t(ns);
    const double2 u = U[e];
    v[(2 * j) * size_t(ns) + p] = u.x;
    v[(2 * j + 1) * size_t(ns) + p] = u.y;
  }
}
cudaError_t launch_pack_pairs(const double* v, double2* U, int ns, int n_levels, double s, cudaStream_t st) {
  const size_t n = size_t(n_levels / 2) * size_t(ns);
  k_pack_pairs<<<unsigned(std::min<size_t>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(v, U, ns, n, s);
  note_launch();
  return cudaGetLastError();
}
cudaError_t launch_unpack_pairs(const double2* U, double* v, int ns, int n_levels, cudaStream_t st) {
  const size_t n = size_t(n_levels / 2) * size_t(ns);
  k_unpack_pairs<<<unsigned(std::min<size_t>((n + 255) / 256, 148 * 16)), 256, 0, st>>>(U, v, ns, n);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
#define FPC_DISPATCH_2D(logm, CALL)        \
  switch (logm) {                          \
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
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_matvec_2d(const double* v, double* y, int n, int n_time, int log_m,
                             const double* eig_y_scaled, const double* eig_x_scaled,
                             const double2* tw_base, cudaStream_t st, int koff) {
  // y-direction on contiguous rows + BDF2 stencil (writes y), then x-direction columns (adds)
  cudaError_t err =
      launch_matvec_rows(v, y, n, n_time * n, n, n * n, log_m, eig_y_scaled, tw_base, st, koff);
  if (err != cudaSuccess) return err;
  if (log_m == 8 && warp_kernels_enabled())
    return launch_matvec_cols_warp(v, y, n, n_time, log_m, eig_x_scaled, tw_base, st);
  if (log_m == 10 && warp32_kernels_enabled())
    return launch_matvec_cols_w32(v, y, n, n_time, eig_x_scaled, tw_base, st);
#define CALL(LM)                                                                          \
  {                                                                                       \
    using G = ColGeo<LM>;                                                                 \
    if ((err = prep2(k_matvec_2d_cols<LM>, G::SMEM_MV, G::NT)) != cudaSuccess) return err;       \
    const int tiles = (n + G::C - 1) / G::C;                                              \
    k_matvec_2d_cols<LM><<<n_time * tiles, G::NT, G::SMEM_MV, st>>>(v, y, n, eig_x_scaled, tw_base); note_launch(); \
  }
  FPC_DISPATCH_2D(log_m, CALL)
#undef CALL
  return cudaGetLastError();
}

template <int LM, int MODE>
static cudaError_t tau2d_cols(double2* Z, int n, int n_rows, const double2* lambda,
                              const double* sigma, double dt, const double2* tw_base,
                              cudaStream_t st) {
  using G = ColGeo<LM>;
  cudaError_t err = prep2(k_tau_2d_cols<LM, MODE>, G::SMEM, G::NT);
  if (err != cudaSuccess) return err;
  const int tiles = (n + G::C - 1) / G::C;
  k_tau_2d_cols<LM, MODE><<<n_rows * tiles, G::NT, G::SMEM, st>>>(Z, n, lambda, sigma, dt, tw_base); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_dst_cols_2d(double2* Z, int n, int n_planes, const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2i(n + 1);
#define CALL(LM)                                                                            \
  err = tau2d_cols<LM, 0>(Z, n, n_planes, nullptr, nullptr, 0.0, tw_base, st);             \
  if (err != cudaSuccess) return err;
  FPC_DISPATCH_2D(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_tau_solve_2d(double2* Z, int n, int n_rows, const double2* lambda,
                                const double* sigma, double dt, const double2* tw_base,
                                cudaStream_t st, bool forward, double2* scratch) {
  // rows (iy) DST, columns (ix) DST-divide-DST, rows DST again (tau.hpp:79-96, 98-119)
  cudaError_t err = cudaSuccess;
  static const bool transposed = [] {  // FPC_TAU_T=0: the strided column pass (A/B)
    const char* e = std::getenv("FPC_TAU_T");
    return !(e && e[0] == '0');
  }();
  if (n == 255 && scratch && transposed && warp_kernels_enabled()) {
    if ((err = launch_dst_rows_T(Z, scratch, n, n_rows, nullptr, nullptr, 0.0, tw_base, st, 0)) != cudaSuccess)
      return err;
    if ((err = launch_dst_rows_T(scratch, Z, n, n_rows, lambda, sigma, dt, tw_base, st, forward ? 2 : 1)) !=
        cudaSuccess)
      return err;
    return launch_dst_rows(Z, n, n_rows * n, tw_base, st);
  }
  err = launch_dst_rows(Z, n, n_rows * n, tw_base, st);
  if (err != cudaSuccess) return err;
  const int lm = ilog2i(n + 1);
  if (n == 255 && warp_kernels_enabled()) {
    if ((err = launch_tau_cols_warp(Z, n, n_rows, lambda, sigma, dt, tw_base, st, forward)) != cudaSuccess)
      return err;
    return launch_dst_rows(Z, n, n_rows * n, tw_base, st);
  }
  if (n == 1023 && warp32_kernels_enabled()) {
    if ((err = launch_tau_cols_w32(Z, n, n_rows, lambda, sigma, dt, tw_base, st, forward)) != cudaSuccess)
      return err;
    return launch_dst_rows(Z, n, n_rows * n, tw_base, st);
  }
#define CALL(LM)                                                                            \
  err = forward ? tau2d_cols<LM, 2>(Z, n, n_rows, lambda, sigma, dt, tw_base, st)           \
                : tau2d_cols<LM, 1>(Z, n, n_rows, lambda, sigma, dt, tw_base, st);          \
  if (err != cudaSuccess) return err;
  FPC_DISPATCH_2D(lm, CALL)
#undef CALL
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  return launch_dst_rows(Z, n, n_rows * n, tw_base, st);
}

}  // namespace fpc
