// kernels_1d.cu -- sm_100a kernels of the 1D hot path: all-at-once matvec (K1), the
// alpha-circulant preconditioner's time FFTs (K2/K4) and the tau shifted solves (K3).
//
// Data layout in HBM (matches the reference's time-major vectors, all_at_once.hpp:18-22):
//   v[k*Ns + p]            real fp64, k = time level, p = spatial index
//   Z[n*Ns + p]            complex128 half spectrum, n = 0..Nt/2 (frequency-major rows, so the
//                          tau solves of K3 read contiguous rows; alpha_circulant.hpp:153-156)
// Every transform is a power-of-two complex FFT run in shared memory by fft_block.cuh; the
// real-input transforms use the standard half-length packing (two reals per complex).
// Global-memory phases are unrolled (U independent loads in flight per thread) so the
// latency of HBM is overlapped; buffers of multi-buffer CTAs are skewed by one bank group.
#include <cooperative_groups.h>

#include <cstdlib>

// build.py compiles this file as three translation units (-DFPC_1D_PART=0: matvec, 1: time FFTs,
// 2: tau solves), so a cold build is not bound by one nvcc process working through every size
// instantiation; without the macro it is one unit (scripts/build_timing.sh, build_variant.sh).
#ifdef FPC_1D_PART
#define FPC_1D_HAS(p) (FPC_1D_PART == (p))
#ifdef FPC_PHASE_TIMING
#error "FPC_PHASE_TIMING builds compile kernels_1d.cu as one unit (no FPC_1D_PART)"
#endif
#else
#define FPC_1D_HAS(p) 1
#endif

#ifdef FPC_PHASE_TIMING
namespace fpc {
__device__ long long g_phase[1 << 16][16];
}
// stamps 8.. inside block_dst (first call per CTA wins the slot: later calls overwrite)
#define FPC_DST_PH(i) \
  do { if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) fpc::g_phase[blockIdx.x][8 + (i)] = clock64(); } while (0)
#endif
#include "dst_block.cuh"
#include "fft_block.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fpc {

#ifdef FPC_PHASE_TIMING
// development instrumentation: per-CTA clock64 stamps at phase boundaries (one thread per CTA)
#define FPC_PH(i) \
  do { if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) g_phase[blockIdx.x][i] = clock64(); } while (0)
extern "C" int fpc_debug_phases(long long* out, int nblocks) {
  return int(cudaMemcpyFromSymbol(out, g_phase, size_t(nblocks) * 16 * sizeof(long long)));
}
// time kernels: kid 0 = k_time_fwd, 1 = k_time_inv
__device__ long long g_phase_t[2][1 << 14][4];
#define FPC_PT(kid, i) \
  do { if (threadIdx.x == 0 && blockIdx.x < (1 << 14)) g_phase_t[kid][blockIdx.x][i] = clock64(); } while (0)
extern "C" int fpc_debug_phases_t(long long* out, int kid, int nblocks) {
  return int(cudaMemcpyFromSymbol(out, g_phase_t, size_t(nblocks) * 4 * sizeof(long long),
                                  size_t(kid) * (1 << 14) * 4 * sizeof(long long)));
}
#else
#define FPC_PH(i) \
  do {            \
  } while (0)
#define FPC_PT(kid, i) \
  do {                 \
  } while (0)
#endif

// buffer stride with stride % 8 == 1 (in 16-byte units): consecutive buffers start in
// consecutive bank groups, so "same slot, next buffer" accesses are conflict free
__host__ __device__ constexpr int skewed(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}

// Elements per CTA for a kernel family; B = buffers per CTA, NT = threads, BS = buffer stride.
template <int LOGM, int TOT, int E_ = 16>
struct Geo {
  static constexpr int E = E_;  // complex values per thread per FFT pass
  static constexpr int M = 1 << LOGM;
  static constexpr int B = (TOT / M) > 0 ? (TOT / M) : 1;
  static constexpr int NT = (B * M) / E;
  static constexpr int BS = B > 1 ? skewed(M) : padded(M);
  static constexpr size_t SMEM = size_t(B) * BS * sizeof(double2);
};

// CTAs per SM the register budget is sized for: radix-16 passes need ~128 registers per thread,
// so 256-thread CTAs run two per SM (16 warps) and 512-thread CTAs one.
__host__ __device__ constexpr int minb(int nt) { return nt <= 128 ? 4 : nt <= 256 ? 2 : 1; }

// L2 prefetch of a column tile: rows r < nrows, each covering bytes [base + r*stride, +width).
// Issues every row's lines at once without holding registers (the strided 32..128-byte row
// segments are latency bound when requested only as fast as register-staged loads retire).
__device__ __forceinline__ void l2_prefetch_column_tile(const void* base, size_t stride, int nrows, int width,
                                                        int nthr) {
  const char* b = static_cast<const char*>(base);
  for (int r = threadIdx.x; r < nrows; r += nthr) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(b + size_t(r) * stride);
    const uintptr_t l0 = a0 & ~uintptr_t(127), l1 = (a0 + uintptr_t(width) - 1) & ~uintptr_t(127);
    for (uintptr_t l = l0; l <= l1; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
  }
}

__device__ __forceinline__ double& comp(double2* s, int slot_padded, int c) {
  return reinterpret_cast<double*>(s + slot_padded)[c];
}

#if FPC_1D_HAS(0)
// =====================================================================================
// K1: 1D all-at-once matvec.  One buffer per time block k; real packing of the length-L
// circulant embedding (L = 2M = next_pow2(2 Ns), toeplitz.hpp:26) into an M-point FFT.
// eig'[k] = -dt * eig[k] / (2L), k = 0..M  (eig real & even: the circulant column is
// symmetric, toeplitz.hpp:27-33).  The BDF2 stencil part (time_stencil.hpp:16-26) is formed
// during the load phase (its three loads issued with the FFT input) and parked in smem.
// =====================================================================================
constexpr int kTotMv = 4096;

#ifndef FPC_MV_PARKED_DEEP
#define FPC_MV_PARKED_DEEP 1
#endif
#ifndef FPC_MV_CST_SMEM
#define FPC_MV_CST_SMEM 2
#endif
// Stencil part of the rows matvec.  Parked: formed in the load phase and kept in shared memory
// (fewest dependent memory round trips: best for the small grids of M >= 1024, config 0).  Not
// parked: the rows are loaded 16 deep, and the epilogue re-reads the three L2-resident rows
// (B200 config 2, M = 256: 2D matvec 1182 -> 932 us).  FPC_MV_CST_SMEM = 0 / 1 forces either.
template <int LOGM>
constexpr bool mv_cst_parked() { return FPC_MV_CST_SMEM == 1 || (FPC_MV_CST_SMEM == 2 && LOGM >= 10); }
template <int LOGM, int TOT = kTotMv>
struct MvGeo {
  using G = Geo<LOGM, TOT, 16>;
  static constexpr size_t SMEM = G::SMEM + (mv_cst_parked<LOGM>() ? size_t(G::B) * G::M * sizeof(double) : 0);
};

// e / d for 0 <= e < 2^24 by a float reciprocal and one correction step (a runtime integer
// division is a ~20-instruction dependent chain; these index splits sit in the latency-bound
// load and epilogue loops of the rows matvec, where ns and rows-per-level are runtime values)
__device__ __forceinline__ int div_small(int e, int d, float inv_d) {
  int q = __float2int_rz(__int2float_rn(e) * inv_d);
  q -= (q * d > e) ? 1 : 0;
  q += ((q + 1) * d <= e) ? 1 : 0;
  return q;
}

template <int LOGM, int TOT = kTotMv>
__global__ void __launch_bounds__(Geo<LOGM, TOT, 16>::NT, minb(Geo<LOGM, TOT, 16>::NT))
    k_matvec_1d(const double* __restrict__ v, double* __restrict__ y, int ns, int nrows, int rpt,
                int sstride, int koff, const double* __restrict__ eig,
                const double2* __restrict__ twb) {
  // Generic "Toeplitz along contiguous rows + BDF2 stencil" pass: row r (length ns) sits at
  // v + r*ns and belongs to time level k = r / rpt; the stencil reads the same position
  // sstride and 2*sstride earlier.  1D: rows = time blocks (rpt = 1, sstride = ns);
  // 2D: rows = lattice rows ix of every time block (rpt = n, sstride = n^2), the y-direction
  // half of jacobian.hpp:84-87.
  using G = Geo<LOGM, TOT, 16>;
  constexpr int M = G::M, B = G::B, L = 2 * M, BS = G::BS, NT = G::NT;
  constexpr int U = 4;
  extern __shared__ double2 smem[];
  double* cst = reinterpret_cast<double*>(smem + B * BS);  // stencil part, B x M
  const int k0 = blockIdx.x * B;
  const int nb = min(B, nrows - k0);
  const float inv_ns = 1.0f / float(ns), inv_rpt = 1.0f / float(rpt);

  constexpr bool kParked = mv_cst_parked<LOGM>();
  if (!kParked) {
    // rows k0 .. k0+nb-1 are one contiguous stretch of nb*ns doubles: 16 loads in flight per
    // thread (the load phase is latency bound), then the packed-slot stores
    constexpr int UL = 16;
    const int nreal = nb * ns;
    const double* src = v + size_t(k0) * ns;
    for (int e0 = threadIdx.x; e0 < nreal; e0 += UL * NT) {
      double x[UL];
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * NT;
        x[u] = e < nreal ? src[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * NT;
        if (e < nreal) {
          const int b = div_small(e, ns, inv_ns), idx = e - b * ns;
          comp(smem, b * BS + pad16(idx >> 1), idx & 1) = x[u];
        }
      }
    }
    // zero padding: slots whose both entries lie at idx >= ns, the odd half-slot, unused rows
    const int s0 = (ns + 1) >> 1;
    for (int t = threadIdx.x; t < B * M; t += NT) {
      const int b = t / M, m = t - b * M;
      if (b >= nb || m >= s0) smem[b * BS + pad16(m)] = make_double2(0.0, 0.0);
      else if ((ns & 1) && m == s0 - 1) comp(smem, b * BS + pad16(m), 1) = 0.0;
    }
  }
#if FPC_MV_PARKED_DEEP
  if (kParked) {
    // the nb rows are one contiguous stretch of nb*ns doubles: only the real elements are visited
    // (not the zero-padded half of the embedding), 3 x UP loads in flight per thread -- the phase is
    // one DRAM round trip per batch (B200 config 3: four batches of 12 loads -> two of 24)
    constexpr int UP = 8;
    const int nreal = nb * ns;
    const double* src = v + size_t(k0) * ns;
    for (int e0 = threadIdx.x; e0 < nreal; e0 += UP * NT) {
      double x0[UP], x1[UP], x2[UP];
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const int e = e0 + u * NT;
        const bool ok = e < nreal;
        const int b = div_small(ok ? e : 0, ns, inv_ns);
        const int k = div_small(k0 + b, rpt, inv_rpt) + koff;
        x0[u] = ok ? src[e] : 0.0;
        x1[u] = (ok && k >= 1) ? src[ptrdiff_t(e) - sstride] : 0.0;
        x2[u] = (ok && k >= 2) ? src[ptrdiff_t(e) - 2 * ptrdiff_t(sstride)] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const int e = e0 + u * NT;
        if (e < nreal) {
          const int b = div_small(e, ns, inv_ns), idx = e - b * ns;
          const int k = div_small(k0 + b, rpt, inv_rpt) + koff;
          comp(smem, b * BS + pad16(idx >> 1), idx & 1) = x0[u];
          double c;
          if (k == 0)
            c = x0[u];
          else if (k == 1)
            c = 1.5 * x0[u] + -2.0 * x1[u];
          else
            c = 1.5 * x0[u] + -2.0 * x1[u] + 0.5 * x2[u];
          cst[b * M + idx] = c;
        }
      }
    }
    const int s0 = (ns + 1) >> 1;
    for (int t = threadIdx.x; t < B * M; t += NT) {
      const int b = t / M, m = t - b * M;
      if (b >= nb || m >= s0) smem[b * BS + pad16(m)] = make_double2(0.0, 0.0);
      else if ((ns & 1) && m == s0 - 1) comp(smem, b * BS + pad16(m), 1) = 0.0;
    }
  }
#endif
  for (int e0 = threadIdx.x; e0 < ((kParked && !FPC_MV_PARKED_DEEP) ? B * L : 0); e0 += U * NT) {
    double x0[U], x1[U], x2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int b = e / L, idx = e - b * L;
      const int k = div_small(k0 + b, rpt, inv_rpt) + koff;
      const bool ok = e < B * L && b < nb && idx < ns;
      const size_t o = size_t(k0 + b) * ns + idx;
      x0[u] = ok ? v[o] : 0.0;
      if (kParked) {
        x1[u] = (ok && k >= 1) ? v[o - sstride] : 0.0;
        x2[u] = (ok && k >= 2) ? v[o - 2 * size_t(sstride)] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      if (e < B * L) {
        const int b = e / L, idx = e - b * L;
        const int k = div_small(k0 + b, rpt, inv_rpt) + koff;
        comp(smem, b * BS + pad16(idx >> 1), idx & 1) = x0[u];
        if (kParked && idx < ns) {
          double c;
          if (k == 0)
            c = x0[u];
          else if (k == 1)
            c = 1.5 * x0[u] + -2.0 * x1[u];
          else
            c = 1.5 * x0[u] + -2.0 * x1[u] + 0.5 * x2[u];
          cst[b * M + idx] = c;
        }
      }
    }
  }
  __syncthreads();
  block_fft<LOGM, -1, BS, G::E>(smem, twb + M, B);

  // pointwise product with the circulant eigenvalues, done on (k, M-k) pairs of the packed
  // spectrum: unpack -> X_k, X_{M-k}; Y = eig' X; repack for the inverse.
  const double2* twL = twb + L;
  for (int t = threadIdx.x; t < B * (M / 2 + 1); t += NT) {
    const int b = t / (M / 2 + 1), kk = t - b * (M / 2 + 1);
    double2* s = smem + b * BS;
    if (kk == 0) {
      const double2 z = s[0];
      const double y0 = eig[0] * (2.0 * (z.x + z.y));
      const double ym = eig[M] * (2.0 * (z.x - z.y));
      s[0] = make_double2(y0 + ym, y0 - ym);
    } else {
      const int i1 = pad16(kk), i2 = pad16(M - kk);
      const double2 w = __ldg(twL + kk);  // e^{-2 pi i k/L}
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
  block_fft<LOGM, 1, BS, G::E>(smem, twb + M, B);

  // epilogue: stencil part + spatial term
  if (kParked) {
    for (int b = 0; b < nb; ++b) {
      double* yb = y + size_t(k0 + b) * ns;
      for (int idx = threadIdx.x; idx < ns; idx += NT) {
        const double tv = comp(smem, b * BS + pad16(idx >> 1), idx & 1);
        yb[idx] = cst[b * M + idx] + tv;
      }
    }
  } else {
    constexpr int UE = 8;
    for (int e0 = threadIdx.x; e0 < nb * ns; e0 += UE * NT) {
      double x0[UE], x1[UE], x2[UE];
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        const int e = e0 + u * NT;
        const int b = div_small(e, ns, inv_ns), idx = e - b * ns;
        const int k = div_small(k0 + b, rpt, inv_rpt) + koff;
        const bool ok = e < nb * ns;
        const size_t o = size_t(k0 + b) * ns + idx;
        x0[u] = ok ? v[o] : 0.0;
        x1[u] = (ok && k >= 1) ? v[o - sstride] : 0.0;
        x2[u] = (ok && k >= 2) ? v[o - 2 * size_t(sstride)] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        const int e = e0 + u * NT;
        if (e >= nb * ns) continue;
        const int b = div_small(e, ns, inv_ns), idx = e - b * ns;
        const int k = div_small(k0 + b, rpt, inv_rpt) + koff;
        double c;  // time_stencil.hpp:16-26 (same association as all_at_once.hpp:44-53)
        if (k == 0)
          c = x0[u];
        else if (k == 1)
          c = 1.5 * x0[u] + -2.0 * x1[u];
        else
          c = 1.5 * x0[u] + -2.0 * x1[u] + 0.5 * x2[u];
        y[size_t(k0 + b) * ns + idx] = c + comp(smem, b * BS + pad16(idx >> 1), idx & 1);
      }
    }
  }
}

#endif  // part 0 kernels

#if FPC_1D_HAS(1)
// =====================================================================================
// K2: time FFT forward over spatial columns (alpha_circulant.hpp:146-156), Hermitian half.
// CTA = B columns; M = Nt/2.
// =====================================================================================
// Complex slots per CTA.  A CTA reads B = TOT/M columns of every time row, i.e. B*8-byte segments
// at a stride of Ns*8 bytes; for long series (M >= 1024) 8 columns per CTA (64-byte segments, one
// 512-thread CTA per SM) beat 4 columns at two CTAs per SM (B200, config 1: 155 -> 145 us),
// because the load/store phases are bound by DRAM efficiency on these strided segments.
template <int LOGM>
constexpr int tot_t() { return LOGM >= 10 ? 8192 : 4096; }

template <int LOGM, int TOT = tot_t<LOGM>()>
__global__ void __launch_bounds__(Geo<LOGM, TOT>::NT, minb(Geo<LOGM, TOT>::NT))
    k_time_fwd(const double* __restrict__ v, double2* __restrict__ Z, int ns,
               const double* __restrict__ sf, double s_in, const double2* __restrict__ twb) {
  using G = Geo<LOGM, TOT>;
  constexpr int M = G::M, B = G::B, NTIME = 2 * M, BS = G::BS, NT = G::NT;
#ifndef FPC_TF_U
#define FPC_TF_U 16
#endif
  constexpr int U = FPC_TF_U;
  extern __shared__ double2 smem[];
  const int p0 = blockIdx.x * B;
  FPC_PT(0, 0);
  // request every row segment of the tile at once (L2 prefetch: no registers held, full lines),
  // then the register-staged loads below mostly hit L2 (B200 config 1: 145 -> 131 us)
  l2_prefetch_column_tile(v + p0, size_t(ns) * 8, NTIME, B * 8, NT);

#ifndef FPC_TF_FUSED
#define FPC_TF_FUSED 1
#endif
  if (FPC_TF_FUSED) {
    FPC_PT(0, 1);
    block_fft_columns_from<LOGM, 1, B, BS, G::E>(smem, twb + M, [&](int c, int kk) {
      const int p = p0 + c;
      return p < ns ? __ldg(sf + kk) * (s_in * v[size_t(kk) * ns + p]) : 0.0;
    });
  } else {
  for (int e0 = threadIdx.x; e0 < B * NTIME; e0 += U * NT) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int c = e % B, kk = e / B;
      const int p = p0 + c;
      x[u] = (e < B * NTIME && p < ns) ? v[size_t(kk) * ns + p] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      if (e < B * NTIME) {
        const int c = e % B, kk = e / B;
        comp(smem, c * BS + pad16(kk >> 1), kk & 1) = __ldg(sf + kk) * (s_in * x[u]);
      }
    }
  }
  __syncthreads();
  FPC_PT(0, 1);
  block_fft<LOGM, 1, BS, G::E>(smem, twb + M, B);
  }
  FPC_PT(0, 2);

  const double2* twT = twb + NTIME;  // e^{-2 pi i n/Nt}; the forward kernel here is e^{+...}
  for (int t = threadIdx.x; t < B * (M / 2 + 1); t += NT) {
    const int c = t % B, n = t / B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const double2* s = smem + c * BS;
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
  FPC_PT(0, 3);
}

// =====================================================================================
// K4: inverse time FFT (alpha_circulant.hpp:167-198) from the half spectrum; the mirror
// Z_{Nt-n} = conj(Z_n) (alpha_circulant.hpp:167-175) is folded into the real-output packing.
// =====================================================================================
template <int LOGM, int TOT = tot_t<LOGM>()>
__global__ void __launch_bounds__(Geo<LOGM, TOT>::NT, minb(Geo<LOGM, TOT>::NT))
    k_time_inv(const double2* __restrict__ Z, double* __restrict__ z, int ns,
               const double* __restrict__ sb, const double2* __restrict__ twb) {
  using G = Geo<LOGM, TOT>;
  constexpr int M = G::M, B = G::B, NTIME = 2 * M, BS = G::BS, NT = G::NT;
  constexpr int U = 8;
  constexpr int TASKS = B * (M / 2 + 1);
  extern __shared__ double2 smem[];
  const int p0 = blockIdx.x * B;
  const double2* twT = twb + NTIME;
  FPC_PT(1, 0);
  l2_prefetch_column_tile(Z + p0, size_t(ns) * 16, M + 1, B * 16, NT);  // 149 -> 141 us

  for (int t0 = threadIdx.x; t0 < TASKS; t0 += U * NT) {
    double2 ya[U], yb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * NT;
      const int c = t % B, n = t / B;
      const int p = p0 + c;
      const bool ok = t < TASKS && p < ns;
      ya[u] = ok ? Z[size_t(n) * ns + p] : make_double2(0.0, 0.0);
      yb[u] = ok ? Z[size_t(M - n) * ns + p] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * NT;
      if (t >= TASKS) continue;
      const int c = t % B, n = t / B;
      double2* s = smem + c * BS;
      if (n == 0) {  // Y_0 and Y_M are both solved rows (alpha_circulant.hpp:158-166)
        const double2 A = cadd(ya[u], yb[u]), Bv = csub(ya[u], yb[u]);
        s[0] = cadd(A, mul_si<1>(Bv));
      } else {
        const double2 w = __ldg(twT + n);  // e^{-2 pi i n/Nt}
        const double2 A = cadd(ya[u], cconj(yb[u]));
        const double2 Bn = cmul(csub(ya[u], cconj(yb[u])), w);
        s[pad16(n)] = cadd(A, mul_si<1>(Bn));
        if (n != M - n) s[pad16(M - n)] = cadd(cconj(A), mul_si<1>(cconj(Bn)));
      }
    }
  }
  __syncthreads();
  FPC_PT(1, 1);
  block_fft<LOGM, -1, BS, G::E>(smem, twb + M, B);
  FPC_PT(1, 2);

  const double inv_nt = 1.0 / double(NTIME);
  for (int e = threadIdx.x; e < B * NTIME; e += NT) {
    const int c = e % B, kk = e / B;
    const int p = p0 + c;
    if (p >= ns) continue;
    const double val = comp(smem, c * BS + pad16(kk >> 1), kk & 1);
    z[size_t(kk) * ns + p] = (__ldg(sb + kk) * inv_nt) * val;
  }
  FPC_PT(1, 3);
}

#endif  // part 1 kernels

#if FPC_1D_HAS(2)
// =====================================================================================
// K3 (1D): tau shifted solves (tau.hpp:98-119): for each retained frequency row n,
//   Z_n <- DST( DST(Z_n) ./ (lambda_n - dt sigma) ),
// both DSTs by block_dst (dst_block.cuh: one N-point complex FFT per complex row, N = Ns + 1).
// B rows per CTA (one for N = 8192).  The singular-shift test of tau.hpp:109-112 is the plan's
// (alpha_circulant.hpp:110-123 checks every retained (n, i) with the same floor).
// =====================================================================================
constexpr int kTotTau = 4096;

template <int LOGM, int TOT = (LOGM >= 13 ? (1 << LOGM) : kTotTau)>
struct TauGeo {
  static constexpr int EE = (1 << LOGM) < 16 ? (1 << LOGM) : 16;
  using G = Geo<LOGM, TOT, EE>;
  static constexpr int BH = G::B > 1 ? skewed(G::M / 2) : padded(G::M / 2);
  static constexpr size_t SMEM = G::SMEM + size_t(G::B) * BH * sizeof(double2);
};

template <int LOGM, int MODE, int TOT = (LOGM >= 13 ? (1 << LOGM) : kTotTau)>  // MODE 0: DST rows only; 1: DST-divide-DST (solve); 2: DST-multiply-DST
__global__ void __launch_bounds__(TauGeo<LOGM, TOT>::G::NT, minb(TauGeo<LOGM, TOT>::G::NT))
    k_tau_solve_1d(double2* __restrict__ Z, int n_rows, const double2* __restrict__ lam,
                   const double* __restrict__ sigma, double dt, const double2* __restrict__ twb) {
  using G = typename TauGeo<LOGM, TOT>::G;
  constexpr int M = G::M, B = G::B, BS = G::BS, NT = G::NT, E = G::E;
  constexpr int NSR = M - 1;  // row length (n_space)
  constexpr int U = 4;
  extern __shared__ double2 smem[];
  double2* hbuf = smem + B * BS;  // DCT-III scratch rows (dst_block.cuh)
  constexpr int BH = TauGeo<LOGM, TOT>::BH;
  const int r0 = blockIdx.x * B;
  const int nb = min(B, n_rows - r0);
  const double scale = sqrt(2.0 / double(M));
  FPC_PH(0);

  // whole rows into L2 up front (contiguous; the staged loads below then hit L2)
  for (int b = 0; b < nb; ++b) {
    const char* zr = reinterpret_cast<const char*>(Z + size_t(r0 + b) * NSR);
    const uintptr_t l0 = reinterpret_cast<uintptr_t>(zr) & ~uintptr_t(127);
    const uintptr_t l1 = (reinterpret_cast<uintptr_t>(zr) + size_t(NSR) * 16 - 1) & ~uintptr_t(127);
    for (uintptr_t l = l0 + uintptr_t(threadIdx.x) * 128; l <= l1; l += uintptr_t(NT) * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
  }
  // one row, folded DST: the first DST reads the row from global memory directly
  constexpr bool kDirect = (LOGM == 13 && B == 1 && MODE != 0);
  // load rows: element i of row b -> slot i + 1.  The nb rows are one contiguous stretch, read 16
  // deep per thread (one memory round trip instead of one per row); rows b >= nb are zeroed
  if constexpr (!kDirect) {
    constexpr int UL = 16;
    const double2* zr = Z + size_t(r0) * NSR;
    for (int e0 = threadIdx.x; e0 < B * NSR; e0 += UL * NT) {
      double2 x[UL];
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * NT;
        x[u] = e < nb * NSR ? zr[e] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * NT;
        if (e < B * NSR) {
          const int b = e / NSR, i = e - b * NSR;
          smem[b * BS + pad16(i + 1)] = x[u];
        }
      }
    }
  }
  __syncthreads();
  FPC_PH(1);
  if constexpr (MODE != 0) {
    block_dst<LOGM, BS, BH, 1, LOGM == 13>(smem, hbuf, twb, scale, kDirect ? Z + size_t(r0) * NSR : nullptr);
    FPC_PH(2);
    // divide by the shifted tau eigenvalues (slot i + 1 <-> index i)
    if constexpr (B > 1) {  // several short rows: one flattened, 16-deep pass over all of them
      constexpr int UD = 16;
      for (int e0 = threadIdx.x; e0 < B * NSR; e0 += UD * NT) {
        double sg[UD];
#pragma unroll
        for (int u = 0; u < UD; ++u) {
          const int e = e0 + u * NT;
          sg[u] = e < B * NSR ? __ldg(sigma + (e % NSR)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UD; ++u) {
          const int e = e0 + u * NT;
          if (e >= B * NSR) continue;
          const int b = e / NSR, i = e - b * NSR;
          const double2 l = (b < nb) ? __ldg(lam + r0 + b) : make_double2(1.0, 0.0);
          double2* sl = smem + b * BS + pad16(i + 1);
          *sl = shift_apply<MODE>(*sl, l.x - dt * sg[u], l.y);
        }
      }
    }
    for (int b = 0; b < (B > 1 ? 0 : B); ++b) {
      double2* s = smem + b * BS;
      const double2 l = (b < nb) ? __ldg(lam + r0 + b) : make_double2(1.0, 0.0);
      for (int i0 = threadIdx.x; i0 < NSR; i0 += 4 * U * NT) {  // sigma loads batched ahead of use
        double sg[4 * U];
#pragma unroll
        for (int u = 0; u < 4 * U; ++u) sg[u] = i0 + u * NT < NSR ? __ldg(sigma + i0 + u * NT) : 0.0;
#pragma unroll
        for (int u = 0; u < 4 * U; ++u) {
          const int i = i0 + u * NT;
          if (i < NSR) s[pad16(i + 1)] = shift_apply<MODE>(s[pad16(i + 1)], l.x - dt * sg[u], l.y);
        }
      }
    }
    __syncthreads();
  }
  FPC_PH(3);
  block_dst<LOGM, BS, BH, 0, LOGM == 13>(smem, hbuf, twb, scale);
  FPC_PH(4);

  // store rows (slot i <-> index i), coalesced
  for (int b = 0; b < nb; ++b) {
    double2* zr = Z + size_t(r0 + b) * NSR;
    const double2* s = smem + b * BS;
    for (int i = threadIdx.x; i < NSR; i += NT) zr[i] = s[pad16(i)];
  }
  FPC_PH(5);
}

#endif  // part 2 kernels

// =====================================================================================
// launchers
// =====================================================================================
template <class K>
static cudaError_t prep(K kernel, size_t smem, int threads = 1024) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct(smem, threads));
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaSuccess;
}

#define FPC_DISPATCH_LOGM(logm, CALL)      \
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

// Small grids (config 0, the small config-4 points): the tuned tiles hold several rows / columns per
// CTA, which leaves most of the 148 SMs idle when there are only a few hundred rows (config 0: 64
// matvec CTAs, 33 tau CTAs, 32 time-FFT CTAs).  When the default tiling gives fewer than two waves,
// the same kernels run with 512-slot tiles (B = max(1, 512 / M): 1-4 rows or columns per CTA).
constexpr int kSmallGrid = 2 * 148;
// rows matvec: the 64-thread tiling wins at 128 default CTAs (1023 x 512: 27K -> 30K matvecs/s) and
// loses at 256 (1023 x 1024: 20K -> 17K)
constexpr int kSmallGridMv = 200;
template <int LM>
constexpr int small_tot() { return (1 << LM) >= 512 ? (1 << LM) : 512; }
template <int LM, int TOT>
constexpr bool is_smaller() { return small_tot<LM>() < TOT; }

#if FPC_1D_HAS(0)
cudaError_t launch_matvec_rows(const double* v, double* y, int len, int nrows, int rpt,
                               int sstride, int log_m, const double* eig_scaled,
                               const double2* tw_base, cudaStream_t st, int koff) {
  cudaError_t err = cudaSuccess;
  if (log_m == 8 && warp_kernels_enabled())
    return launch_matvec_rows_warp(v, y, len, nrows, rpt, sstride, log_m, eig_scaled, tw_base, st, koff);
  // one warp per row needs a full wave of warps (8 per SM) to pay; smaller grids keep the CTA kernel
  if (log_m == 10 && nrows >= warp32_min_rows() && warp32_kernels_enabled())
    return launch_matvec_rows_w32(v, y, len, nrows, rpt, sstride, eig_scaled, tw_base, st, koff);
#define CALL(LM)                                                                          \
  {                                                                                       \
    using G = Geo<LM, kTotMv, 16>;                                                        \
    if constexpr (is_smaller<LM, kTotMv>()) {                                             \
      if ((nrows + G::B - 1) / G::B < kSmallGridMv) {                                     \
        constexpr int T = small_tot<LM>();                                                \
        using GS = Geo<LM, T, 16>;                                                        \
        if ((err = prep(k_matvec_1d<LM, T>, MvGeo<LM, T>::SMEM, GS::NT)) != cudaSuccess) return err; \
        k_matvec_1d<LM, T><<<(nrows + GS::B - 1) / GS::B, GS::NT, MvGeo<LM, T>::SMEM, st>>>( \
            v, y, len, nrows, rpt, sstride, koff, eig_scaled, tw_base);                   \
        note_launch();                                                                    \
        return cudaGetLastError();                                                        \
      }                                                                                   \
    }                                                                                     \
    if ((err = prep(k_matvec_1d<LM>, MvGeo<LM>::SMEM, Geo<LM, kTotMv, 16>::NT)) != cudaSuccess) return err;        \
    k_matvec_1d<LM><<<(nrows + G::B - 1) / G::B, G::NT, MvGeo<LM>::SMEM, st>>>(           \
        v, y, len, nrows, rpt, sstride, koff, eig_scaled, tw_base); note_launch();                       \
  }
  FPC_DISPATCH_LOGM(log_m, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_matvec_1d(const double* v, double* y, int n_space, int n_time, int log_m,
                             const double* eig_scaled, const double2* tw_base, cudaStream_t st,
                             int koff) {
  cudaError_t err = cudaSuccess;
  if (log_m == 13 || log_m == 14)  // kernels_mv.cu: 2-CTA cluster, half-length FFTs
    return launch_matvec_split(v, y, n_space, n_time, log_m, koff, eig_scaled, tw_base, st);
  if (log_m >= 15)  // kernels_large.cu: 8..16-CTA clusters
    return launch_matvec_large(v, y, n_space, n_time, log_m, koff, eig_scaled, tw_base, st);
  (void)err;
  return launch_matvec_rows(v, y, n_space, n_time, 1, n_space, log_m, eig_scaled, tw_base, st, koff);
}

#endif  // part 0 launchers

static inline int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

#if FPC_1D_HAS(1)
cudaError_t launch_time_fwd(const double* v, double2* Z, int n_space, int n_time,
                            const double* scale_fwd, double s_in, const double2* tw_base,
                            cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  if (time_warp_supported(n_space, n_time))
    return launch_time_fwd_warp(v, Z, n_space, n_time, scale_fwd, s_in, tw_base, st);
  if (time_tma_supported(n_space, n_time, v, false))
    return launch_time_fwd_tma(v, Z, n_space, n_time, scale_fwd, s_in, tw_base, st);
  if (time_split_supported(n_time))
    return launch_time_fwd_split(v, Z, n_space, n_time, scale_fwd, s_in, tw_base, st);
  const int lm = ilog2(n_time) - 1;
#define CALL(LM)                                                                          \
  {                                                                                       \
    using G = Geo<LM, tot_t<LM>()>;                                                             \
    if constexpr (is_smaller<LM, tot_t<LM>()>() && LM <= 10) {  /* n_time >= 4096: one-column tiles (8-byte row segments) lose */                                        \
      if ((n_space + G::B - 1) / G::B < kSmallGrid) {                                     \
        constexpr int T = small_tot<LM>();                                                \
        using GS = Geo<LM, T>;                                                            \
        if ((err = prep(k_time_fwd<LM, T>, GS::SMEM, GS::NT)) != cudaSuccess) return err; \
        k_time_fwd<LM, T><<<(n_space + GS::B - 1) / GS::B, GS::NT, GS::SMEM, st>>>(       \
            v, Z, n_space, scale_fwd, s_in, tw_base);                                     \
        note_launch();                                                                    \
        return cudaGetLastError();                                                        \
      }                                                                                   \
    }                                                                                     \
    if ((err = prep(k_time_fwd<LM>, G::SMEM, G::NT)) != cudaSuccess) return err;                 \
    k_time_fwd<LM><<<(n_space + G::B - 1) / G::B, G::NT, G::SMEM, st>>>(                  \
        v, Z, n_space, scale_fwd, s_in, tw_base); note_launch();                                         \
  }
  FPC_DISPATCH_LOGM(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_time_inv(const double2* Z, double* z, int n_space, int n_time,
                            const double* scale_bwd, const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  if (time_warp_supported(n_space, n_time))
    return launch_time_inv_warp(Z, z, n_space, n_time, scale_bwd, tw_base, st);
  if (time_tma_supported(n_space, n_time, Z, true)) return launch_time_inv_tma(Z, z, n_space, n_time, scale_bwd, tw_base, st);
  if (time_split_supported(n_time)) return launch_time_inv_split(Z, z, n_space, n_time, scale_bwd, tw_base, st);
  const int lm = ilog2(n_time) - 1;
#define CALL(LM)                                                                            \
  {                                                                                         \
    using G = Geo<LM, tot_t<LM>()>;                                                               \
    if constexpr (is_smaller<LM, tot_t<LM>()>() && LM <= 10) {  /* n_time >= 4096: one-column tiles (8-byte row segments) lose */                                          \
      if ((n_space + G::B - 1) / G::B < kSmallGrid) {                                       \
        constexpr int T = small_tot<LM>();                                                  \
        using GS = Geo<LM, T>;                                                              \
        if ((err = prep(k_time_inv<LM, T>, GS::SMEM, GS::NT)) != cudaSuccess) return err;   \
        k_time_inv<LM, T><<<(n_space + GS::B - 1) / GS::B, GS::NT, GS::SMEM, st>>>(Z, z, n_space, \
                                                                                 scale_bwd, tw_base); \
        note_launch();                                                                      \
        return cudaGetLastError();                                                          \
      }                                                                                     \
    }                                                                                       \
    if ((err = prep(k_time_inv<LM>, G::SMEM, G::NT)) != cudaSuccess) return err;                   \
    k_time_inv<LM><<<(n_space + G::B - 1) / G::B, G::NT, G::SMEM, st>>>(Z, z, n_space,       \
                                                                        scale_bwd, tw_base); note_launch(); \
  }
  FPC_DISPATCH_LOGM(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

#endif  // part 1 launchers

#if FPC_1D_HAS(2)
// in-place orthonormal DST-I of n_rows contiguous complex rows of length n (n + 1 = 2^k)
cudaError_t launch_dst_rows(double2* Z, int n, int n_rows, const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  if (n == 255 && warp_kernels_enabled())
    return launch_dst_rows_warp(Z, n, n_rows, nullptr, nullptr, 0.0, tw_base, st, 0);
  if (n == 1023 && n_rows >= warp32_min_rows() && warp32_kernels_enabled())
    return launch_dst_rows_w32(Z, n, n_rows, nullptr, nullptr, 0.0, tw_base, st, 0);
  const int lm = ilog2(n + 1);
#define CALL(LM)                                                                          \
  {                                                                                       \
    using TG = TauGeo<LM>;                                                                \
    if ((err = prep(k_tau_solve_1d<LM, 0>, TG::SMEM, TG::G::NT)) != cudaSuccess) return err;     \
    const int grid = (n_rows + TG::G::B - 1) / TG::G::B;                                  \
    k_tau_solve_1d<LM, 0><<<grid, TG::G::NT, TG::SMEM, st>>>(Z, n_rows, nullptr, nullptr, \
                                                                 0.0, tw_base); note_launch();           \
  }
  FPC_DISPATCH_LOGM(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

template <int LM, int MODE>
static cudaError_t tau1d(double2* Z, int n_rows, const double2* lambda, const double* sigma,
                         double dt, const double2* tw_base, cudaStream_t st) {
  using TG = TauGeo<LM>;
  constexpr int TD = (LM >= 13 ? (1 << LM) : kTotTau);
  if constexpr (is_smaller<LM, TD>()) {
    if ((n_rows + TG::G::B - 1) / TG::G::B < kSmallGrid) {
      constexpr int T = small_tot<LM>();
      using TS = TauGeo<LM, T>;
      cudaError_t err = prep(k_tau_solve_1d<LM, MODE, T>, TS::SMEM, TS::G::NT);
      if (err != cudaSuccess) return err;
      k_tau_solve_1d<LM, MODE, T><<<(n_rows + TS::G::B - 1) / TS::G::B, TS::G::NT, TS::SMEM, st>>>(
          Z, n_rows, lambda, sigma, dt, tw_base);
      note_launch();
      return cudaGetLastError();
    }
  }
  cudaError_t err = prep(k_tau_solve_1d<LM, MODE>, TG::SMEM, TG::G::NT);
  if (err != cudaSuccess) return err;
  const int grid = (n_rows + TG::G::B - 1) / TG::G::B;
  k_tau_solve_1d<LM, MODE><<<grid, TG::G::NT, TG::SMEM, st>>>(Z, n_rows, lambda, sigma, dt, tw_base); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tau_solve_1d(double2* Z, int n_space, int n_rows, const double2* lambda,
                                const double* sigma, double dt, const double2* tw_base,
                                cudaStream_t st, bool forward) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2(n_space + 1);
  if (lm >= 14) return launch_tau_large(Z, n_space, n_rows, lambda, sigma, dt, tw_base, st, forward);
  if (n_space == 255 && warp_kernels_enabled())
    return launch_dst_rows_warp(Z, n_space, n_rows, lambda, sigma, dt, tw_base, st, forward ? 2 : 1);
  if (n_space == 1023 && n_rows >= warp32_min_rows() && warp32_kernels_enabled())
    return launch_dst_rows_w32(Z, n_space, n_rows, lambda, sigma, dt, tw_base, st, forward ? 2 : 1);
#define CALL(LM)                                                                  \
  err = forward ? tau1d<LM, 2>(Z, n_rows, lambda, sigma, dt, tw_base, st)         \
                : tau1d<LM, 1>(Z, n_rows, lambda, sigma, dt, tw_base, st);
  FPC_DISPATCH_LOGM(lm, CALL)
#undef CALL
  return err;
}

#endif  // part 2 launchers

}  // namespace fpc
