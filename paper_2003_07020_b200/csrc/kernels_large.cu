// kernels_large.cu -- K1 and K3 for long spatial rows (Ns + 1 = 16384 .. 65536, BASELINE config 4's
// upper range) on thread-block clusters of C CTAs that each own one 8192-point FFT in shared memory.
//
// A length-P transform (P = C * S, S = 8192) is split by residue classes of the output bins: with
// k = C k' + q,
//   X_k = sum_{m<S} [ w_P^{m q} * sum_{r<C} x_{m + r S} w_C^{r q} ] w_S^{m k'},
// so CTA q runs one S-point FFT on u^{(q)}_m = w_P^{mq} (C-point DFT over r of x_{m+rS})_q.  The
// C-point DFTs are computed once, by the CTA that owns m (m-slices of S/C), and scattered to the
// owners of q through distributed shared memory (DSMEM); after the local FFTs the inverse direction
// gathers the C values of one m (or k') from all CTAs and finishes with a C-point DFT in registers.
// Shared memory per CTA: 8192 complex (139 KB), 512 threads, one CTA per SM.
//
//  * matvec (all_at_once.hpp:33-55 + toeplitz.hpp:41-57): the length-L circulant embedding of one
//    time block (L = C*S, x real and zero past Ns) -> X = FFT_-(x) residue-split -> X_k * eig_k ->
//    per-CTA inverse FFT_+ -> gather y_m = Re sum_q e^{+2 pi i m q/L} P_q[m mod S] / L + BDF2 stencil.
//    (No real packing here: the pairing k <-> L-k of the packed form would cross CTAs.)
//  * tau shifted solve (tau.hpp:98-119), DST-I through the odd extension (dst.hpp:21-43):
//    g = (0, f_1..f_{N-1}, 0, -f_{N-1}..-f_1) of length 2N = C*S, G = FFT_-(g), F_k = (i/2) G_k,
//    DST(f)_{k-1} = sqrt(2/N) F_k; two DSTs with the shifted division between them, in place on the
//    frequency row (cluster barriers order every read of the row before its overwrite).
#include <cooperative_groups.h>

#include "fft_block.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fpc {

namespace {

constexpr int kLogS = 13, kS = 1 << kLogS, kThr = kS / 16;
constexpr int kBS = padded(kS);
constexpr size_t kSmemL = size_t(kBS) * sizeof(double2);

// ---------------------------------------------------------------------------------- matvec
template <int C>
__global__ void __launch_bounds__(kThr, 1)
    k_matvec_cl(const double* __restrict__ v, double* __restrict__ y, int ns, int koff,
                const double* __restrict__ eig, const double2* __restrict__ twb) {
  constexpr int L = C * kS;
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const size_t k = blockIdx.x / C;
  const long kg = long(k) + koff;
  const double* vk = v + k * ns;
  const double2* twL = twb + L;  // e^{-2 pi i t/L}
  cluster_sync_relaxed(cluster);  // every CTA of the cluster is running before its shared memory is written

  // 1. fold: for my m-slice, the C-point DFT over r of x_{m+rS} (x = 0 for index >= Ns, so only
  //    r < C/2 contribute), twiddled by w_L^{m q} and stored into CTA q's buffer
  for (int m = q * (kS / C) + int(threadIdx.x); m < (q + 1) * (kS / C); m += kThr) {
    double2 a[C];
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int j = m + r * kS;
      a[r] = make_double2(r < C / 2 && j < ns ? vk[j] : 0.0, 0.0);
    }
    Dft<C, -1>::run(a);
#pragma unroll
    for (int qq = 0; qq < C; ++qq) {
      double2* dst = cluster.map_shared_rank(smem, qq);
      dst[pad16(m)] = qq == 0 ? a[0] : cmul(a[qq], __ldg(twL + m * qq));
    }
  }
  cluster.sync();
  block_fft<kLogS, -1, kBS, 16>(smem, twb + kS, 1);

  // 2. X_k * eig'_k (k = C k' + q; eig real and even, table k = 0..L/2 holds -dt eig/(2L))
  for (int kp = threadIdx.x; kp < kS; kp += kThr) {
    const int kk = C * kp + q;
    const double e = 2.0 * __ldg(eig + (kk <= L / 2 ? kk : L - kk));
    smem[pad16(kp)] = cscale(smem[pad16(kp)], e);
  }
  __syncthreads();
  block_fft<kLogS, 1, kBS, 16>(smem, twb + kS, 1);
  cluster.sync();

  // 3. gather: y_{m0 + rS} = Re sum_q e^{+2 pi i (m0 + rS) q/L} P_q[m0], then + BDF2 stencil
  double* yk = y + k * ns;
  for (int m0 = q * (kS / C) + int(threadIdx.x); m0 < (q + 1) * (kS / C); m0 += kThr) {
    double2 t[C];
#pragma unroll
    for (int qq = 0; qq < C; ++qq) {
      const double2 p = cluster.map_shared_rank(smem, qq)[pad16(m0)];
      t[qq] = qq == 0 ? p : cmul(p, cconj(__ldg(twL + m0 * qq)));
    }
    Dft<C, 1>::run(t);
#pragma unroll
    for (int r = 0; r < C / 2; ++r) {
      const int j = m0 + r * kS;
      if (j >= ns) continue;
      const double c0 = vk[j];
      double c;  // time_stencil.hpp:16-26 (same association as all_at_once.hpp:44-53)
      if (kg == 0)
        c = c0;
      else if (kg == 1)
        c = 1.5 * c0 + -2.0 * vk[long(j) - ns];
      else
        c = 1.5 * c0 + -2.0 * vk[long(j) - ns] + 0.5 * vk[long(j) - 2 * long(ns)];
      yk[j] = c + t[r].x;
    }
  }
  cluster_sync_exit(cluster);  // partners have read this CTA's buffer (no wait on the y stores)
}

// ------------------------------------------------------------------ matvec, packed residue split
// The 2-CTA split of kernels_mv.cu generalised to C = M/S CTAs (C = 4: Ns = 32767, C = 8: Ns = 65535):
// the real length-L embedding is packed into M = L/2 complex points z_m = v_{2m} + i v_{2m+1}
// (z_m = 0 for m >= H = M/2), and the M-point transform is split by residue classes of the bins,
// k = C k' + q:
//   X_{Ck'+q} = sum_{m'<S} e^{-2 pi i m'k'/S} [ w_M^{m'q} sum_{j<C/2} z_{m'+jS} e^{-2 pi i jq/C} ],
// one S-point FFT per rank (only j < C/2 of the C-point DFT is non-zero: half the fold work of the
// unpacked k_matvec_cl, whose L-point transform is twice as long).  The spectral product pairs
// bins k and M-k: residues q and C-q, so ranks 0 and C/2 pair within themselves and rank q pairs
// with rank C-q through DSMEM (each rank of a pair handles the pairs whose own slot is < S/2, so
// no slot is touched by both).  Inverse: rank q inverts its residue class, then
//   y_{m'+jS} = sum_q e^{+2 pi i jq/C} [ w_M^{-m'q} a^{(q)}_{m'} ]   (j < C/2: the outputs needed),
// a C-point DFT over the ranks' values of one m', gathered through DSMEM.
template <int C>
__global__ void __launch_bounds__(kThr, 1)
    k_matvec_splitc(const double* __restrict__ v, double* __restrict__ y, int ns, int koff,
                    const double* __restrict__ eig, const double2* __restrict__ twb) {
  constexpr int S = kS, M = C * S, L = 2 * M;
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const size_t k = blockIdx.x / C;
  const long kg = long(k) + koff;
  const double* vk = v + k * ns;
  const double2* twM = twb + M;        // e^{-2 pi i t/M} = twMh[t >> 6] * twM[t & 63]
  const double2* twMh = twb + M / 64;
  auto wm = [&](int t) -> double2 { return cmul(__ldg(twMh + (t >> 6)), __ldg(twM + (t & 63))); };
  const double2* twC = twb + C;        // e^{-2 pi i t/C}
  cluster_sync_relaxed(cluster);       // every CTA of the cluster is running (DSMEM targets exist)

  // 1. forward: u_{m'} = w_M^{m'q} sum_{j<C/2} z_{m'+jS} e^{-2 pi i jq/C}, S-point FFT (-)
  auto load_u = [&](int mp) -> double2 {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < C / 2; ++j) {
      const int i = 2 * (mp + j * S);
      const double2 zm = make_double2(i < ns ? vk[i] : 0.0, i + 1 < ns ? vk[i + 1] : 0.0);
      acc = j == 0 ? zm : cadd(acc, q == 0 ? zm : cmul(zm, __ldg(twC + ((j * q) & (C - 1)))));
    }
    return q == 0 ? acc : cmul(acc, wm(mp * q));
  };
  block_fft_from<kLogS, -1, kBS, 16>(smem, twb + S, load_u);
  cluster.sync();  // both ranks of every pair have their spectra

  // 2. eigenvalue product on (kappa, M - kappa) pairs (kernels_mv.cu formulas)
  const double2* twL = twb + L;
  const double2* twLh = twb + L / 128;  // e^{-2 pi i kappa/L} = twLh[kappa >> 7] twL[kappa & 127]
  const int qp = (C - q) & (C - 1);      // partner rank (0 -> 0, C/2 -> C/2)
  double2* own = smem;
  double2* par = cluster.map_shared_rank(smem, qp);
  const int ntask = q == 0 ? S / 2 + 1 : S / 2;
  for (int t = int(threadIdx.x); t < ntask; t += kThr) {
    const int kap = C * t + q;
    if (kap == 0) {
      const double2 z = own[0];
      const double y0 = __ldg(eig) * (2.0 * (z.x + z.y));
      const double ym = __ldg(eig + M) * (2.0 * (z.x - z.y));
      own[0] = make_double2(y0 + ym, y0 - ym);
      continue;
    }
    // partner slot of M - kappa: rank 0 -> S - t, others -> S - 1 - t (in rank qp)
    const int s2 = q == 0 ? S - t : S - 1 - t;
    const double2 w = cmul(__ldg(twLh + (kap >> 7)), __ldg(twL + (kap & 127)));
    const double ek = __ldg(eig + kap), em = __ldg(eig + (M - kap));
    const double2 a = own[pad16(t)], bq = par[pad16(s2)];
    const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
    const double2 iwQ = mul_si<1>(cmul(w, Q));
    const double2 Yk = cscale(csub(P, iwQ), ek);
    const double2 Ym = cscale(cconj(cadd(P, iwQ)), em);
    const double2 A = cadd(Yk, cconj(Ym));
    const double2 D = csub(Yk, cconj(Ym));
    own[pad16(t)] = cadd(A, mul_si<1>(cmul(D, cconj(w))));
    if (!(q == 0 && s2 == t)) par[pad16(s2)] = cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
  }
  cluster.sync();  // the partner's writes into my slots >= S/2 are done
  block_fft<kLogS, 1, kBS, 16>(smem, twb + S, 1);
  cluster.sync();  // every rank's inverse is done

  // 3. y_{m'+jS} = sum_r e^{+2 pi i jr/C} w_M^{-m'r} a^{(r)}_{m'}, j < C/2; + BDF2 stencil
  double* yk = y + k * ns;
  for (int mp = q * (S / C) + int(threadIdx.x); mp < (q + 1) * (S / C); mp += kThr) {
    double2 b[C];
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const double2 p = cluster.map_shared_rank(smem, r)[pad16(mp)];
      b[r] = r == 0 ? p : cmul(p, cconj(wm(mp * r)));
    }
    Dft<C, 1>::run(b);
#pragma unroll
    for (int j = 0; j < C / 2; ++j) {
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const int i = 2 * (mp + j * S) + part;
        if (i >= ns) continue;
        const double c0 = vk[i];
        double c;  // time_stencil.hpp:16-26 (same association as all_at_once.hpp:44-53)
        if (kg == 0)
          c = c0;
        else if (kg == 1)
          c = 1.5 * c0 + -2.0 * vk[long(i) - ns];
        else
          c = 1.5 * c0 + -2.0 * vk[long(i) - ns] + 0.5 * vk[long(i) - 2 * long(ns)];
        yk[i] = c + (part ? b[j].y : b[j].x);
      }
    }
  }
  cluster_sync_exit(cluster);  // partners have read this CTA's buffer
}

// ---------------------------------------------------------------------------------- tau solve
// one DST-I of the row (in place), scaled by sqrt(2/N); MODE 1/2: divided/multiplied by the
// shifted eigenvalue (tau.hpp:109-118) on the way out
template <int C, int MODE, bool LAST = false>
__device__ __forceinline__ void dst_cl(double2* row, double2* smem, cg::cluster_group& cluster, int q,
                                       const double2* __restrict__ twb, double2 l,
                                       const double* __restrict__ sigma, double dt) {
  constexpr int P = C * kS, N = P / 2;  // 2N = P
  const double2* twP = twb + P;
  // fold over the odd extension g_j: f_j (1 <= j < N), -f_{2N-j} (N < j < 2N), 0 at j = 0, N
  for (int m = q * (kS / C) + int(threadIdx.x); m < (q + 1) * (kS / C); m += kThr) {
    double2 a[C];
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int j = m + r * kS;
      double2 g = make_double2(0.0, 0.0);
      if (j >= 1 && j < N) {
        g = row[j - 1];
      } else if (j > N) {
        const double2 f = row[P - j - 1];
        g = make_double2(-f.x, -f.y);
      }
      a[r] = g;
    }
    Dft<C, -1>::run(a);
#pragma unroll
    for (int qq = 0; qq < C; ++qq) {
      double2* dst = cluster.map_shared_rank(smem, qq);
      dst[pad16(m)] = qq == 0 ? a[0] : cmul(a[qq], __ldg(twP + m * qq));
    }
  }
  cluster.sync();  // every fold (and so every read of the row) is done
  block_fft<kLogS, -1, kBS, 16>(smem, twb + kS, 1);
  cluster.sync();
  // gather k' in my slice of [0, S/2): outputs k = C k' + q for all q, F_k = (i/2) G_k
  const double scale = sqrt(2.0 / double(N));
  for (int kp = q * (kS / (2 * C)) + int(threadIdx.x); kp < (q + 1) * (kS / (2 * C)); kp += kThr) {
#pragma unroll
    for (int qq = 0; qq < C; ++qq) {
      const int kk = C * kp + qq;
      if (kk < 1 || kk >= N) continue;
      const double2 gk = cluster.map_shared_rank(smem, qq)[pad16(kp)];
      double2 val = make_double2(-0.5 * gk.y * scale, 0.5 * gk.x * scale);
      if (MODE != 0) val = shift_apply<MODE>(val, l.x - dt * __ldg(sigma + kk - 1), l.y);
      row[kk - 1] = val;
    }
  }
  // row writes visible to the cluster (the next DST's fold reads them); after the last DST only
  // "partners are done with this buffer" is needed
  if constexpr (LAST)
    cluster_sync_exit(cluster);
  else
    cluster.sync();
}

template <int C, int MODE>
__global__ void __launch_bounds__(kThr, 1)
    k_tau_cl(double2* __restrict__ Z, int ns, const double2* __restrict__ lam, const double* __restrict__ sigma,
             double dt, const double2* __restrict__ twb) {
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const int rowi = blockIdx.x / C;
  double2* row = Z + size_t(rowi) * ns;
  const double2 l = MODE != 0 ? __ldg(lam + rowi) : make_double2(1.0, 0.0);
  cluster_sync_relaxed(cluster);  // every CTA of the cluster is running before its shared memory is written
  dst_cl<C, MODE>(row, smem, cluster, q, twb, l, sigma, dt);
  dst_cl<C, 0, true>(row, smem, cluster, q, twb, l, sigma, dt);
}

// one DST-I per row (the commuted ordering's per-level DST at n_space + 1 >= 16384)
template <int C>
__global__ void __launch_bounds__(kThr, 1)
    k_dst_cl(double2* __restrict__ Z, int ns, const double2* __restrict__ lam, const double* __restrict__ sigma,
             double dt, const double2* __restrict__ twb) {
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  double2* row = Z + size_t(blockIdx.x / C) * ns;
  cluster_sync_relaxed(cluster);  // every CTA of the cluster is running before its shared memory is written
  dst_cl<C, 0, true>(row, smem, cluster, q, twb, make_double2(1.0, 0.0), sigma, dt);
}

template <class K>
cudaError_t launch_cl(K kernel, int C, int nclusters, cudaStream_t st, void** args) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemL));
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(C) * unsigned(nclusters));
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = kSmemL;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(kernel), args);
}

}  // namespace

cudaError_t launch_matvec_large(const double* v, double* y, int n_space, int n_time, int log_m, int koff,
                                const double* eig_scaled, const double2* tw_base, cudaStream_t st) {
  void* args[] = {(void*)&v, (void*)&y, (void*)&n_space, (void*)&koff, (void*)&eig_scaled, (void*)&tw_base};
#ifndef FPC_MV_LARGE_SPLIT
#define FPC_MV_LARGE_SPLIT 1
#endif
  if (FPC_MV_LARGE_SPLIT) {  // packed residue split: M = C * 8192
    const int Cp = 1 << (log_m - kLogS);
    switch (Cp) {
      case 4: return launch_cl(k_matvec_splitc<4>, 4, n_time, st, args);
      case 8: return launch_cl(k_matvec_splitc<8>, 8, n_time, st, args);
      default: return cudaErrorInvalidValue;
    }
  }
  // unpacked: L = 2M = C * 8192 (M = 16384 runs on kernels_mv.cu's packed 2-CTA split instead)
  const int C = 1 << (log_m + 1 - kLogS);
  switch (C) {
    case 8: return launch_cl(k_matvec_cl<8>, 8, n_time, st, args);
    case 16: return launch_cl(k_matvec_cl<16>, 16, n_time, st, args);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tau_large(double2* Z, int n_space, int n_rows, const double2* lambda, const double* sigma,
                             double dt, const double2* tw_base, cudaStream_t st, bool forward) {
  // 2N = 2 (Ns + 1) = C * 8192
  const int C = 2 * (n_space + 1) / kS;
  void* args[] = {(void*)&Z, (void*)&n_space, (void*)&lambda, (void*)&sigma, (void*)&dt, (void*)&tw_base};
#define TAU_CASE(CC)                                                                    \
  case CC:                                                                              \
    return forward ? launch_cl(k_tau_cl<CC, 2>, CC, n_rows, st, args)                   \
                   : launch_cl(k_tau_cl<CC, 1>, CC, n_rows, st, args);
  switch (C) {
    TAU_CASE(4)
    TAU_CASE(8)
    TAU_CASE(16)
    default:
      return cudaErrorInvalidValue;
  }
#undef TAU_CASE
}

cudaError_t launch_dst_large(double2* Z, int n_space, int n_rows, const double2* tw_base, cudaStream_t st) {
  const int C = 2 * (n_space + 1) / kS;
  const double2* lam = nullptr;
  const double* sigma = nullptr;
  double dt = 0.0;
  void* args[] = {(void*)&Z, (void*)&n_space, (void*)&lam, (void*)&sigma, (void*)&dt, (void*)&tw_base};
  switch (C) {
    case 4: return launch_cl(k_dst_cl<4>, 4, n_rows, st, args);
    case 8: return launch_cl(k_dst_cl<8>, 8, n_rows, st, args);
    case 16: return launch_cl(k_dst_cl<16>, 16, n_rows, st, args);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fpc
