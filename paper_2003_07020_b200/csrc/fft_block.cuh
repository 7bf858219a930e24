// fft_block.cuh -- CTA-level fp64 complex FFT engine in shared memory (sm_100a).
//
// Replaces the reference's scalar radix-2 `fft_pow2` (fft.hpp:49-67) on the hot path.  Design:
//   * Stockham autosort, radix 16/8/4/2 passes; each thread owns E = 16 complex values per pass
//     (one radix-16 butterfly, two radix-8, ...), reads them from smem, __syncthreads, applies
//     twiddles + the in-register DFT, writes them to their autosorted slots, __syncthreads.
//     In-place in one buffer: every read of a pass completes before any write.
//   * Buffers are padded one complex per 16 (pad(i) = i + i/16) so the radix-R strided writes of
//     the first pass and the unit-stride reads of every pass are bank-conflict free for 16-byte
//     (double2) accesses.
//   * Twiddles: two loads per butterfly from a per-size table tw_N[t] = e^{-2 pi i t/N}
//     (built on the host with the reference's polar() formula, fft.hpp:36-37), the remaining
//     powers by <=3 complex products.
//   * Batched: a CTA runs B independent transforms of size N = 2^LOGN (buffers at stride
//     padded(N)), NT = B*N/16 threads.
// Kernel sign convention: SIGN = +1 computes x[k] = sum_j x[j] e^{+2 pi i jk/N} (fft.hpp:93-95).
#pragma once
#include <cuda_runtime.h>

namespace fpc {

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 4); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by S*i (S = +-1)
template <int S>
__device__ __forceinline__ double2 mul_si(double2 a) {
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// a / (cr + i ci) as a conj(c) / |c|^2: one fp64 division per mode instead of Smith's three
// (std::complex division, tau.hpp:114, agrees to a few ulp; the shifted eigenvalues are O(1)..
// O(1e8) in magnitude, far from the range where |c|^2 could overflow or underflow)
__device__ __forceinline__ double2 cdiv_recip(double2 a, double cr, double ci) {
  const double inv = 1.0 / fma(cr, cr, ci * ci);
  return make_double2(fma(a.x, cr, a.y * ci) * inv, fma(a.y, cr, -a.x * ci) * inv);
}

// the per-mode step of the shifted tau action (tau.hpp:109-118): MODE 1 = solve (divide by the
// shifted eigenvalue), MODE 2 = forward action (multiply)
template <int MODE>
__device__ __forceinline__ double2 shift_apply(double2 a, double cr, double ci) {
  if constexpr (MODE == 2) return cmul(a, make_double2(cr, ci));
  return cdiv_recip(a, cr, ci);
}

// cos/sin(2 pi k / 16), k = 0..15
__device__ __constant__ double kC16[16] = {
    1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
    0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
    -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977,
    0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674};

// In-register DFT of size R with kernel e^{S 2 pi i jk/R}: natural order in and out.
// Recursive radix-2 DIT; all indices compile-time after unrolling.
template <int R, int S>
struct Dft {
  __device__ __forceinline__ static void run(double2* v) {
    double2 e[R / 2], o[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    Dft<R / 2, S>::run(e);
    Dft<R / 2, S>::run(o);
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      // w^k = e^{S 2 pi i k / R}; index into the 16-point table
      constexpr int step = 16 / R;
      double2 t;
      const int idx = k * step;
      if (idx == 0) {
        t = o[k];
      } else if (idx == 4) {
        t = mul_si<S>(o[k]);
      } else if (idx == 8) {
        t = make_double2(-o[k].x, -o[k].y);
      } else if (idx == 12) {
        t = mul_si<-S>(o[k]);
      } else {
        const double c = kC16[idx];
        const double s = S * kC16[(idx + 12) & 15];  // sin(2 pi idx/16) = cos(2 pi (idx-4)/16)
        t = make_double2(fma(o[k].x, c, -o[k].y * s), fma(o[k].x, s, o[k].y * c));
      }
      v[k] = cadd(e[k], t);
      v[k + R / 2] = csub(e[k], t);
    }
  }
};
template <int S>
struct Dft<2, S> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};
template <int S>
struct Dft<4, S> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    const double2 s13 = cadd(v[1], v[3]), d13 = mul_si<S>(csub(v[1], v[3]));
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13);
    v[3] = csub(d02, d13);
  }
};

// Twiddle table access: tw points at a size-N table, tw[t] = e^{-2 pi i t / N}, 0 <= t < N (every
// table lives at tw_base + N, so the tables of all sizes are reachable from any one of them).
template <int S>
__device__ __forceinline__ double2 twid(const double2* __restrict__ tw, int t) {
  const double2 w = __ldg(tw + t);
  return S > 0 ? cconj(w) : w;
}

// Multiply v[r] (r = 1..R-1) by w^r, w = tw[t1] (w4 = tw4[t1] = w^4 when R > 4: tw4 is the table a
// quarter the size of tw's, so w4 is the same double as tw[4 t1]).  t1 = 0 gives the identity
// through the table (tw[0] = 1), so there is no divergent early exit.
template <int R, int S>
__device__ __forceinline__ void apply_twiddles(double2* v, const double2* __restrict__ tw,
                                               const double2* __restrict__ tw4, int t1) {
  const double2 w1 = twid<S>(tw, t1);
  if constexpr (R == 2) {
    v[1] = cmul(v[1], w1);
  } else if constexpr (R == 4) {
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
  } else {
    // powers built and applied on the fly (few live twiddles -> fewer registers):
    // w^{4a+b} = (w^4)^a w^b, at most three products deep
    const double2 w4 = twid<S>(tw4, t1);
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], cmul(w4, w1));
    v[6] = cmul(v[6], cmul(w4, w2));
    v[7] = cmul(v[7], cmul(w4, w3));
    if constexpr (R == 16) {
      const double2 w8 = cmul(w4, w4);
      const double2 w12 = cmul(w8, w4);
      v[8] = cmul(v[8], w8);
      v[9] = cmul(v[9], cmul(w8, w1));
      v[10] = cmul(v[10], cmul(w8, w2));
      v[11] = cmul(v[11], cmul(w8, w3));
      v[12] = cmul(v[12], w12);
      v[13] = cmul(v[13], cmul(w12, w1));
      v[14] = cmul(v[14], cmul(w12, w2));
      v[15] = cmul(v[15], cmul(w12, w3));
    }
  }
}

// Cluster barrier without memory ordering (barrier.cluster.arrive.relaxed): for barriers that only
// order execution -- "every CTA of the cluster has started" or "the partner has finished reading my
// shared memory" (its DSMEM loads have returned: their values were consumed before it arrived).
// cg::cluster_group::sync() is arrive.release, i.e. MEMBAR.ALL.GPU, which waits for every
// outstanding global store of the thread (the epilogue's) before the CTA can retire.
// FPC_CLUSTER_RELAXED=0 restores cluster.sync() everywhere (A/B).
#ifndef FPC_CLUSTER_RELAXED
#define FPC_CLUSTER_RELAXED 1
#endif
template <class Cluster>
__device__ __forceinline__ void cluster_sync_relaxed(Cluster& cluster) {
  if constexpr (FPC_CLUSTER_RELAXED)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;\n" ::: "memory");
  else
    cluster.sync();
}

// Exit barrier of a cluster kernel whose CTAs read each other's shared memory: "every DSMEM read
// of my partners' buffers has been performed before any partner may retire".  A relaxed arrive
// does not order a load whose value is never consumed (e.g. a predicated-off store's operand), so
// these use arrive.release (the memory model's guarantee; it also waits for the CTA's outstanding
// global stores, ~2% on the split matvec).  FPC_CLUSTER_EXIT_RELAXED=1 restores the relaxed form (A/B).
#ifndef FPC_CLUSTER_EXIT_RELAXED
#define FPC_CLUSTER_EXIT_RELAXED 0
#endif
template <class Cluster>
__device__ __forceinline__ void cluster_sync_exit(Cluster& cluster) {
  if constexpr (FPC_CLUSTER_EXIT_RELAXED)
    cluster_sync_relaxed(cluster);
  else
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.aligned;\n" ::: "memory");
}

// Barrier policies: the whole CTA, or a named barrier over a thread group (warp-specialised
// kernels running independent transforms in different groups).
struct CtaSync {
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
template <int ID, int NTHR>
struct GroupSync {
  __device__ __forceinline__ static void sync() { asm volatile("bar.sync %0, %1;\n" ::"n"(ID), "n"(NTHR) : "memory"); }
};

// One Stockham pass of radix R over B buffers of size N = 2^LOGN held in smem (buffer stride BS,
// pad16 inside a buffer).  NS = current sub-transform length (compile time, so all index
// arithmetic folds to shifts/masks).  Each thread processes E/R butterflies (E complex values).
// The pass in two halves (operands read + butterflies into registers; autosorted writes), so a
// caller can interleave the halves of independent transforms between its own barriers.
template <int LOGN, int R, int S, int BS, int E, int NS>
__device__ __forceinline__ void stockham_load(const double2* s, const double2* __restrict__ tw, int tid, int nthr,
                                              double2 (&v)[E / R][R], int (&dst)[E / R]) {
  constexpr int N = 1 << LOGN;
  constexpr int NB = N / R;
  constexpr int PER = E / R;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int g = tid + q * nthr;
    const int b = g / NB;
    const int j = g & (NB - 1);
    const double2* base = s + b * BS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q][r] = base[pad16(j + r * NB)];
    const int jm = j & (NS - 1);
    if constexpr (NS > 1) apply_twiddles<R, S>(v[q], tw - N + NS * R, tw - N + (NS * R) / 4, jm);
    Dft<R, S>::run(v[q]);
    dst[q] = b * BS + (j - jm) * R + jm;
  }
}

template <int R, int BS, int E, int NS>
__device__ __forceinline__ void stockham_store(double2* s, const double2 (&v)[E / R][R], const int (&dst)[E / R]) {
#pragma unroll
  for (int q = 0; q < E / R; ++q) {
    const int b = dst[q] / BS;
    const int off = dst[q] - b * BS;
    double2* base = s + b * BS;
#pragma unroll
    for (int r = 0; r < R; ++r) base[pad16(off + r * NS)] = v[q][r];
  }
}

template <int LOGN, int R, int S, int BS, int E, int NS, class Sync>
__device__ __forceinline__ void stockham_pass(double2* s, const double2* __restrict__ tw, int tid, int nthr) {
  constexpr int N = 1 << LOGN;
  constexpr int NB = N / R;   // butterflies per buffer
  constexpr int PER = E / R;  // butterflies per thread
  double2 v[PER][R];
  int dst[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int g = tid + q * nthr;  // butterfly index across buffers
    const int b = g / NB;
    const int j = g & (NB - 1);
    const double2* base = s + b * BS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q][r] = base[pad16(j + r * NB)];
    const int jm = j & (NS - 1);
    // w = e^{-2 pi i jm/(NS R)}: read from the dense size-(NS R) table (tw_base + NS R), not the
    // size-N table at stride N/(NS R) -- the same doubles (power-of-two index scaling), a much
    // smaller L1 footprint
    if constexpr (NS > 1) apply_twiddles<R, S>(v[q], tw - N + NS * R, tw - N + (NS * R) / 4, jm);
    Dft<R, S>::run(v[q]);
    dst[q] = b * BS + (j - jm) * R + jm;  // buffer base + logical offset (pad applied below)
  }
  Sync::sync();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = dst[q] / BS;
    const int off = dst[q] - b * BS;
    double2* base = s + b * BS;
#pragma unroll
    for (int r = 0; r < R; ++r) base[pad16(off + r * NS)] = v[q][r];
  }
  Sync::sync();
}

// Passes from sub-transform length NS up to (not including) NEND (default: the whole transform).
template <int LOGN, int S, int BS, int E, int NS, class Sync, int NEND = (1 << LOGN)>
__device__ __forceinline__ void fft_passes(double2* s, const double2* __restrict__ tw, int tid, int nthr) {
  if constexpr (NS < NEND) {
    constexpr int LE = E == 16 ? 4 : E == 8 ? 3 : E == 4 ? 2 : 1;
    // the remainder radix goes first (NS = 1 needs no twiddles), full radix-E passes after it,
    // so the twiddle sets the later passes touch stay small and L1 resident
    constexpr int rem = (NS == 1) ? (LOGN % LE) : 0;
    constexpr int R = rem == 3 ? 8 : rem == 2 ? 4 : rem == 1 ? 2 : E;
    stockham_pass<LOGN, R, S, BS, E, NS, Sync>(s, tw, tid, nthr);
    fft_passes<LOGN, S, BS, E, NS * R, Sync, NEND>(s, tw, tid, nthr);
  }
}

// Full transform of B buffers: requires blockDim.x * E == B * N (every buffer is transformed;
// unused buffers must hold finite data).  E = complex values per thread per pass (16: radix-16
// passes; 8: radix-8 passes at twice the threads).  The caller must __syncthreads() before the
// call and may read the result after it returns.
template <int LOGN, int S, int BS = padded(1 << LOGN), int E = 16>
__device__ __forceinline__ void block_fft(double2* s, const double2* __restrict__ tw, int /*nbuf*/) {
  fft_passes<LOGN, S, BS, E, 1, CtaSync>(s, tw, int(threadIdx.x), int(blockDim.x));
}

// Full transform of one buffer whose input is produced by load(i) (i = logical index, e.g. straight
// from global memory): the first Stockham pass (NS = 1, no twiddles) takes its operands from the
// loader instead of shared memory, which saves the staging write, one read pass and a barrier.
// Requires blockDim.x * E == N.  Ends with the result in s (natural order).
template <int LOGN, int S, int BS, int E, class Load, int NEND = (1 << LOGN)>
__device__ __forceinline__ void block_fft_from(double2* s, const double2* __restrict__ tw, Load load) {
  constexpr int N = 1 << LOGN;
  constexpr int LE = E == 16 ? 4 : E == 8 ? 3 : E == 4 ? 2 : 1;
  constexpr int rem = LOGN % LE;
  constexpr int R = rem == 3 ? 8 : rem == 2 ? 4 : rem == 1 ? 2 : E;
  constexpr int NB = N / R, PER = E / R;
  const int tid = int(threadIdx.x), nthr = int(blockDim.x);
  double2 v[PER][R];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = tid + q * nthr;
#pragma unroll
    for (int r = 0; r < R; ++r) v[q][r] = load(j + r * NB);
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = tid + q * nthr;
    Dft<R, S>::run(v[q]);
#pragma unroll
    for (int r = 0; r < R; ++r) s[pad16(j * R + r)] = v[q][r];
  }
  __syncthreads();
  fft_passes<LOGN, S, BS, E, R, CtaSync, NEND>(s, tw, tid, nthr);
}

// B real columns of length 2N packed into B complex N-point buffers (slot m = x[2m] + i x[2m+1]),
// transformed with the first Stockham pass taken straight from the loader: load(b, k) returns
// element k of column b (already scaled).  Threads map to butterflies column-fastest, so the
// loads of consecutive threads hit consecutive columns of one row (the caller's coalescing unit),
// and every thread issues all 2E of its loads before the first use.  Saves the staging write, one
// shared-memory read pass and a barrier against packing into shared memory first.
// Requires blockDim.x * E == B * N.  Ends with the spectra in s (natural order).
template <int LOGN, int S, int B, int BS, int E, class Load>
__device__ __forceinline__ void block_fft_columns_from(double2* s, const double2* __restrict__ tw, Load load) {
  constexpr int N = 1 << LOGN;
  constexpr int LE = E == 16 ? 4 : E == 8 ? 3 : E == 4 ? 2 : 1;
  constexpr int rem = LOGN % LE;
  constexpr int R = rem == 3 ? 8 : rem == 2 ? 4 : rem == 1 ? 2 : E;
  constexpr int NB = N / R, PER = E / R;
  const int tid = int(threadIdx.x), nthr = int(blockDim.x);
  double2 v[PER][R];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int g = tid + q * nthr;
    const int b = g % B, j = g / B;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = j + r * NB;
      v[q][r] = make_double2(load(b, 2 * m), load(b, 2 * m + 1));
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int g = tid + q * nthr;
    const int b = g % B, j = g / B;
    Dft<R, S>::run(v[q]);
#pragma unroll
    for (int r = 0; r < R; ++r) s[b * BS + pad16(j * R + r)] = v[q][r];
  }
  __syncthreads();
  fft_passes<LOGN, S, BS, E, R, CtaSync>(s, tw, tid, nthr);
}

// Two independent single-buffer transforms in radix-16 passes, software pipelined between CTA
// barriers: the N = 2^LOGA point transform of `a` on all nthr threads (passes from NSA) and the
// 2^LOGB point transform of `b` on threads tid < nb (passes from NSB), the same number of passes
// each.  Interval order: load a_p | store a_p, load b_p | store b_p, load a_{p+1} | ... | store
// b_last: every in-place pass still reads all its operands before any write (a barrier between),
// a thread holds one pass's 16 values at a time, and 2k+1 barriers replace the 4k of the two
// transforms run one after the other (the second on half the CTA, the other half idle).
// Requires nthr * 16 == 2^LOGA and nb * 16 == 2^LOGB.  Ends with a barrier.
template <int LOGA, int BSA, int NSA, int LOGB, int BSB, int NSB, int S>
__device__ __forceinline__ void dual_fft_passes(double2* a, const double2* __restrict__ twa, double2* b,
                                                const double2* __restrict__ twb, int tid, int nthr, int nb) {
  if constexpr (NSA < (1 << LOGA)) {
    static_assert(NSB < (1 << LOGB) && NSA * 16 <= (1 << LOGA) && NSB * 16 <= (1 << LOGB), "pass counts differ");
    double2 va[1][16];
    int da[1];
    stockham_load<LOGA, 16, S, BSA, 16, NSA>(a, twa, tid, nthr, va, da);
    __syncthreads();
    stockham_store<16, BSA, 16, NSA>(a, va, da);
    double2 vb[1][16];
    int db[1];
    if (tid < nb) stockham_load<LOGB, 16, S, BSB, 16, NSB>(b, twb, tid, nb, vb, db);
    __syncthreads();
    if (tid < nb) stockham_store<16, BSB, 16, NSB>(b, vb, db);
    dual_fft_passes<LOGA, BSA, NSA * 16, LOGB, BSB, NSB * 16, S>(a, twa, b, twb, tid, nthr, nb);
  } else {
    __syncthreads();
  }
}

// The same over a thread group of NTHR threads (local index tid) synchronised by named barrier ID;
// NTHR * E == B * N.
template <int LOGN, int S, int BS, int E, int NTHR, int ID>
__device__ __forceinline__ void group_fft(double2* s, const double2* __restrict__ tw, int tid) {
  fft_passes<LOGN, S, BS, E, 1, GroupSync<ID, NTHR>>(s, tw, tid, NTHR);
}

}  // namespace fpc
