// kernels_mv.cu -- K1 for the large 1D case (M = 8192 packed points, Ns up to 8191): the
// all-at-once matvec (all_at_once.hpp:33-55 + toeplitz.hpp:41-57) on a 2-CTA cluster.
//
// The packed input z (real length-L embedding, L = 2M) has z_m = 0 for m >= H = M/2, so the first
// decimation-in-frequency stage of the M-point forward FFT is free: rank 0 transforms z (even
// bins), rank 1 transforms z_m e^{-2 pi i m/M} (odd bins), one H-point FFT each.  Spectral pairs
// (k, M-k) share parity, so the eigenvalue product stays CTA-local.  The inverse is split the same
// way (E = even bins, O = odd bins, y_m = E_m + e^{+2 pi i m/M} O_m); only y_m for m < H is needed
// and each rank assembles half of those, reading the partner's buffer through DSMEM.
//
// Memory phases are asynchronous or batched so their latency is paid once per CTA (measured with
// clock64 phase stamps: the first version spent ~60% of its cycles waiting on loads and the
// cluster barrier):
//   * the packed FFT input is read from global memory straight into the first radix-16 pass
//     (block_fft_from: no shared-memory staging pass);
//   * the post-twiddle of the odd half is applied by whichever rank assembles the output, so the
//     two ranks reach the cluster barrier with equal work;
//   * the BDF2 stencil inputs, both spectral halves and the twiddles of a thread's outputs are all
//     requested before any of them is used.
#include <cooperative_groups.h>

#include "fft_block.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fpc {

#ifdef FPC_PHASE_TIMING
__device__ long long g_phase_mv[1 << 16][8];
#define FPC_PHM(i) \
  do { if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) g_phase_mv[blockIdx.x][i] = clock64(); } while (0)
extern "C" int fpc_debug_phases_mv(long long* out, int nblocks) {
  return int(cudaMemcpyFromSymbol(out, g_phase_mv, size_t(nblocks) * 8 * sizeof(long long)));
}
#else
#define FPC_PHM(i) \
  do {             \
  } while (0)
#endif


// Fused middle of the split matvec for H = M/2 = 16^k (called after every forward pass but the
// last): thread j finishes the forward FFT's last radix-16 pass in registers -- it then holds the
// spectrum slots p_r = j + r H/16, r = 0..15 -- stores them, and reads the 16 mirror slots of its
// pairs (rank 0: H - p, rank 1: H - 1 - p; all held by one other thread).  Each own slot's output of
// the eigenvalue product is formed from (own, mirror) with the pair's canonical twiddle and
// eigenvalues, exactly the arithmetic of the unfused product (the pair's primary slot gets
// A + i D conj(w), the mirror slot conj(A) + i conj(D) w); the 16 outputs are exactly the operands
// of the inverse FFT's first radix-16 pass (no twiddles at NS = 1), which runs in registers too.
// Against the three separate phases: one shared-memory read and one write per element less, and one
// barrier less.
template <int LOGM>
__device__ __forceinline__ void mv_fused_product(double2* smem, int q, const double* __restrict__ eig,
                                                 const double2* __restrict__ twb) {
  constexpr int M = 1 << LOGM, H = M / 2, L = 2 * M, NB = H / 16, BS = padded(H);
  const int j = int(threadIdx.x);
  double2 v[1][16];
  int dst[1];
  stockham_load<LOGM - 1, 16, -1, BS, 16, NB>(smem, twb + H, j, NB, v, dst);
  __syncthreads();
  stockham_store<16, BS, 16, NB>(smem, v, dst);  // slot j + r NB <- v[0][r]
  __syncthreads();
  const double2* twL = twb + L;
  const double2* twLh = twb + L / 128;
  const double2* eigq = reinterpret_cast<const double2*>(eig + eigq_offset(M)) + q * (H / 2);
#ifndef FPC_MV_FG
#define FPC_MV_FG 4
#endif
  constexpr int G = FPC_MV_FG;  // slots whose mirror / table loads are in flight together
#pragma unroll
  for (int r0 = 0; r0 < 16; r0 += G) {
    double2 bm[G], wv[G], ee[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int s = j + (r0 + u) * NB;
      const int ms = q == 0 ? ((H - s) & (H - 1)) : H - 1 - s;  // mirror slot (rank 0 slot 0: itself)
      const bool prim = q == 0 ? s <= H / 2 : s < H / 2;
      const int s1 = prim ? s : ms;                             // the pair's primary slot
      const int t = q == 0 ? s1 - 1 : s1;                       // its task index
      const int kap = 2 * s1 + q;
      bm[u] = smem[pad16(ms)];
      const bool ok = !(q == 0 && s == 0);
      wv[u] = ok ? cmul(__ldg(twLh + (kap >> 7)), __ldg(twL + (kap & 127))) : make_double2(1.0, 0.0);
      ee[u] = ok ? __ldg(eigq + t) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int r = r0 + u;
      const int s = j + r * NB;
      if (q == 0 && s == 0) {  // bins 0 and M
        const double2 z = v[0][r];
        const double y0 = eig[0] * (2.0 * (z.x + z.y));
        const double ym = eig[M] * (2.0 * (z.x - z.y));
        v[0][r] = make_double2(y0 + ym, y0 - ym);
        continue;
      }
      const bool prim = q == 0 ? s <= H / 2 : s < H / 2;
      const double2 a = prim ? v[0][r] : bm[u], bq = prim ? bm[u] : v[0][r];
      const double2 w = wv[u];
      const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
      const double2 iwQ = mul_si<1>(cmul(w, Q));
      const double2 Yk = cscale(csub(P, iwQ), ee[u].x);
      const double2 Ym = cscale(cconj(cadd(P, iwQ)), ee[u].y);
      const double2 A = cadd(Yk, cconj(Ym));
      const double2 D = csub(Yk, cconj(Ym));
      v[0][r] = prim ? cadd(A, mul_si<1>(cmul(D, cconj(w)))) : cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
    }
  }
  Dft<16, 1>::run(v[0]);  // inverse FFT, first pass (NS = 1: no twiddles)
  __syncthreads();        // every mirror read is done before the pass outputs overwrite the buffer
  dst[0] = 16 * j;
  stockham_store<16, BS, 16, 1>(smem, v, dst);
  __syncthreads();
}

// two CTAs per SM for M = 8192 (4096-point halves); one for M = 16384 (8192-point halves)
template <int LOGM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((1 << (LOGM - 1)) / 16, LOGM <= 13 ? 2 : 1)
    k_matvec_split(const double* __restrict__ v, double* __restrict__ y, int ns, int koff,
                   const double* __restrict__ eig, const double2* __restrict__ twb) {
  constexpr int M = 1 << LOGM, H = M / 2, L = 2 * M, NT = H / 16, BS = padded(H);
  extern __shared__ double2 smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = int(cluster.block_rank());
  const size_t k = blockIdx.x >> 1;
  const long kg = long(k) + koff;  // global time level (time-sharded callers pass halo + offset)
  const double* vk = v + k * ns;
  const double2* twM = twb + M;
  FPC_PHM(0);

  // 1. forward FFT of the packed input z_m = v[2m] + i v[2m+1] (rank 1: b_m = z_m e^{-2 pi i m/M},
  //    the odd bins); the first radix pass takes its operands straight from global memory
  FPC_PHM(1);
  // e^{-2 pi i m/M} = tw_{M/64}[m >> 6] * tw_M[m & 63]: two small L1-resident tables instead of a
  // 64 KB stretch of the size-M table per row
  const double2* twMh = twb + M / 64;
  auto twm = [&](int m) -> double2 { return cmul(__ldg(twMh + (m >> 6)), __ldg(twM + (m & 63))); };
  auto load_z = [&](int m) -> double2 {
    const int i = 2 * m;
    const double2 zm = make_double2(i < ns ? vk[i] : 0.0, i + 1 < ns ? vk[i + 1] : 0.0);
    return q == 1 ? cmul(zm, twm(m)) : zm;
  };
#ifndef FPC_MV_FUSE
#define FPC_MV_FUSE 0  // measured slower (262 -> 269 us at config 1), kept for A/B
#endif
  // H = 16^k (M = 8192): the forward FFT's last pass, the eigenvalue product and the inverse FFT's
  // first pass share one register set (see mv_fused_product); otherwise three separate phases
  constexpr bool kFuse = FPC_MV_FUSE && (LOGM - 1) % 4 == 0;
  if constexpr (kFuse) {
    block_fft_from<LOGM - 1, -1, BS, 16, decltype(load_z), H / 16>(smem, twb + H, load_z);
    FPC_PHM(2);
    mv_fused_product<LOGM>(smem, q, eig, twb);
    FPC_PHM(3);
    fft_passes<LOGM - 1, 1, BS, 16, 16, CtaSync>(smem, twb + H, int(threadIdx.x), NT);
  } else {
  block_fft_from<LOGM - 1, -1, BS, 16>(smem, twb + H, load_z);
  FPC_PHM(2);

  // 2. eigenvalue product on (kappa, M - kappa) pairs; slot j of rank q holds bin 2j + q.
  //    task t: rank 0 -> (slot t+1, slot H-t-1, kappa 2t+2); rank 1 -> (t, H-1-t, 2t+1)
  const double2* twL = twb + L;
  const double2* twLh = twb + L / 128;  // e^{-2 pi i kappa/L} = tw_{L/128}[kappa >> 7] tw_L[kappa & 127]
  const double2* eigq = reinterpret_cast<const double2*>(eig + eigq_offset(M)) + q * (H / 2);
#ifndef FPC_MV_UP
#define FPC_MV_UP 4
#endif
  constexpr int UP = FPC_MV_UP;
  constexpr int ntask = H / 2;
  if (q == 0 && threadIdx.x == 0) {
    const double2 z = smem[0];
    const double y0 = eig[0] * (2.0 * (z.x + z.y));
    const double ym = eig[M] * (2.0 * (z.x - z.y));
    smem[0] = make_double2(y0 + ym, y0 - ym);
  }
  for (int t0 = threadIdx.x; t0 < ntask; t0 += UP * NT) {
    double2 wv[UP];
    double ek[UP], em[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int t = t0 + u * NT;
      const int kap = q == 0 ? 2 * (t + 1) : 2 * t + 1;
      const bool ok = t < ntask;
      wv[u] = ok ? cmul(__ldg(twLh + (kap >> 7)), __ldg(twL + (kap & 127))) : make_double2(1.0, 0.0);
      const double2 ee = ok ? __ldg(eigq + t) : make_double2(0.0, 0.0);
      ek[u] = ee.x;
      em[u] = ee.y;
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int t = t0 + u * NT;
      if (t >= ntask) continue;
      const int s1 = q == 0 ? t + 1 : t, s2 = q == 0 ? H - (t + 1) : H - 1 - t;
      const double2 w = wv[u];
      const double2 a = smem[pad16(s1)], bq = smem[pad16(s2)];
      const double2 P = cadd(a, cconj(bq)), Q = csub(a, cconj(bq));
      const double2 iwQ = mul_si<1>(cmul(w, Q));
      const double2 Yk = cscale(csub(P, iwQ), ek[u]);
      const double2 Ym = cscale(cconj(cadd(P, iwQ)), em[u]);
      const double2 A = cadd(Yk, cconj(Ym));
      const double2 D = csub(Yk, cconj(Ym));
      smem[pad16(s1)] = cadd(A, mul_si<1>(cmul(D, cconj(w))));
      if (s1 != s2) smem[pad16(s2)] = cadd(cconj(A), mul_si<1>(cmul(cconj(D), w)));
    }
  }
  __syncthreads();
  FPC_PHM(3);
  block_fft<LOGM - 1, 1, BS, 16>(smem, twb + H, 1);
  }
  FPC_PHM(4);
  cluster.sync();
  FPC_PHM(5);

  // 3. outputs 2m, 2m+1 for my half of m: y_m = E_m + e^{+2 pi i m/M} O_m, + the BDF2 stencil
  const double2* Eb = cluster.map_shared_rank(smem, 0);
  const double2* Ob = cluster.map_shared_rank(smem, 1);
  double* yk = y + k * ns;
  constexpr int PER = (H / 2) / NT;  // m values per thread
  static_assert(PER * NT == H / 2, "H/2 must be a multiple of the thread count");
#ifndef FPC_MV_UB
#define FPC_MV_UB 2
#endif
  constexpr int UB = FPC_MV_UB;      // m values whose loads are in flight together
#pragma unroll 1
  for (int u0 = 0; u0 < PER; u0 += UB) {
    double2 e[UB], o[UB], w[UB], c0[UB], c1[UB], c2[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int m = q * (H / 2) + threadIdx.x + (u0 + u) * NT;
      const int j0 = 2 * m;
      e[u] = Eb[pad16(m)];
      o[u] = Ob[pad16(m)];
      w[u] = twm(m);
      const bool ok0 = j0 < ns, ok1 = j0 + 1 < ns;
      c0[u] = make_double2(ok0 ? vk[j0] : 0.0, ok1 ? vk[j0 + 1] : 0.0);
      c1[u] = make_double2(ok0 && kg >= 1 ? vk[long(j0) - ns] : 0.0, ok1 && kg >= 1 ? vk[long(j0) + 1 - ns] : 0.0);
      c2[u] = make_double2(ok0 && kg >= 2 ? vk[long(j0) - 2 * long(ns)] : 0.0,
                           ok1 && kg >= 2 ? vk[long(j0) + 1 - 2 * long(ns)] : 0.0);
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int m = q * (H / 2) + threadIdx.x + (u0 + u) * NT;
      const int j0 = 2 * m;
      const double2 t = cadd(e[u], cmul(o[u], cconj(w[u])));
      double2 c;  // time_stencil.hpp:16-26 (same association as all_at_once.hpp:44-53)
      if (kg == 0)
        c = c0[u];
      else if (kg == 1)
        c = make_double2(1.5 * c0[u].x + -2.0 * c1[u].x, 1.5 * c0[u].y + -2.0 * c1[u].y);
      else
        c = make_double2(1.5 * c0[u].x + -2.0 * c1[u].x + 0.5 * c2[u].x,
                         1.5 * c0[u].y + -2.0 * c1[u].y + 0.5 * c2[u].y);
      if (j0 < ns) yk[j0] = c.x + t.x;
      if (j0 + 1 < ns) yk[j0 + 1] = c.y + t.y;
    }
  }
  FPC_PHM(6);
  cluster_sync_exit(cluster);  // keep both buffers alive until the partner has read them
}

template <int LOGM>
static cudaError_t launch_split(const double* v, double* y, int n_space, int n_time, int koff,
                                const double* eig_scaled, const double2* tw_base, cudaStream_t st) {
  constexpr int H = 1 << (LOGM - 1);
  constexpr size_t smem = size_t(padded(H)) * sizeof(double2);
  cudaError_t err = cudaFuncSetAttribute(k_matvec_split<LOGM>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         carveout_pct(smem, H / 16));
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_matvec_split<LOGM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return err;
  k_matvec_split<LOGM><<<2 * n_time, H / 16, smem, st>>>(v, y, n_space, koff, eig_scaled, tw_base); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_matvec_split(const double* v, double* y, int n_space, int n_time, int log_m, int koff,
                                const double* eig_scaled, const double2* tw_base, cudaStream_t st) {
  if (log_m == 13) return launch_split<13>(v, y, n_space, n_time, koff, eig_scaled, tw_base, st);
  if (log_m == 14) return launch_split<14>(v, y, n_space, n_time, koff, eig_scaled, tw_base, st);
  return cudaErrorInvalidValue;
}

}  // namespace fpc
