// kernels_time_tma.cu -- the preconditioner's time FFTs (alpha_circulant.hpp:146-156 forward,
// 167-198 inverse) for n_time = 128..512 as persistent CTAs fed by the tensor-memory accelerator.
//
// The column-tile kernels of kernels_1d.cu (k_time_fwd / k_time_inv) read a [n_time][B] column tile
// with register-staged strided loads: every CTA sits out a full DRAM round trip before its first
// butterfly, and 60% of its stall samples are that wait (profiles/r2_summary.md).  Here each CTA
// loops over column tiles; the tile after the current one is fetched by one elected thread with
// cp.async.bulk.tensor (2D boxes, mbarrier completion) into a staging buffer while the CTA
// transforms the current tile, so the memory round trip overlaps the butterflies and the epilogue
// stores of the same CTA.
//
// Tensor views (the reference's time-major layout, all_at_once.hpp:18-22, rows of odd length are
// only 8-byte aligned, TMA needs 16-byte strides):
//   forward input  v[k][p] real     -> [n_time/2][2 ns] doubles, row stride 16 ns bytes: a row holds
//                                      time levels 2m (columns 0..ns) and 2m+1 (columns ns..2ns);
//                                      a tile is two boxes of n_time/2 rows: [B] columns of the even
//                                      levels and, because a box must start on a 16-byte boundary
//                                      (an odd ns puts column ns + p0 8 bytes off: the copy engine
//                                      raises an illegal-instruction fault), [B + 2] columns from
//                                      ns - 1 + p0 of the odd levels (second tensor map)
//   inverse input  Z[n][p] complex  -> [n_time/2+1][2 ns] doubles, row stride 16 ns bytes; a tile is
//                                      two boxes of [n_time/4+1][2B]
// Arithmetic, packing and output layout are those of k_time_fwd / k_time_inv (bit-identical
// results: same operand order in every product and sum).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "bulk_copy.cuh"
#include "fft_block.cuh"
#include "kernels.cuh"

namespace fpc {

namespace {

__host__ __device__ constexpr int skewed_t(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}

// 2048 packed complex slots per CTA: B = 8 columns at n_time = 512, 16 at 256, 32 at 128;
// 128 threads, ~67 KB of shared memory: three CTAs per SM, each with its own tile in flight.
template <int LOGM>
struct TmaGeo {
  static constexpr int M = 1 << LOGM, NTIME = 2 * M;
  static constexpr int B = 2048 / M;
  static constexpr int NT = B * M / 16;
  static constexpr int BS = skewed_t(M);
  // a TMA box has at most 256 rows: the forward tile is NBF boxes of RF time-level pairs per parity,
  // the inverse's spectrum tile (M + 1 rows) NBI boxes of RB rows (RB B a multiple of 8, so every
  // box lands 128-byte aligned; rows past M are zero filled)
  static constexpr int RF = M < 256 ? M : 256, NBF = M / RF;
  static constexpr int NBI = (M + 1 + 255) / 256;
  static constexpr int RBQ = B >= 8 ? 1 : 8 / B;
  static constexpr int RB = ((M + 1 + NBI - 1) / NBI + RBQ - 1) / RBQ * RBQ;
  static constexpr bool TABLE = LOGM <= 8;  // scale_bwd / Nt in shared memory (no room at M = 512)
  static constexpr size_t FFT = size_t(B) * BS * sizeof(double2);
  static constexpr size_t STAGE_EVEN = size_t(M) * B * sizeof(double);
  static constexpr size_t STAGE_FWD = STAGE_EVEN + size_t(M) * (B + 2) * sizeof(double);
  static constexpr size_t STAGE_INV = size_t(NBI * RB) * B * sizeof(double2);
  static constexpr size_t TAB = TABLE ? size_t(NTIME) * sizeof(double) : 0;
  static constexpr size_t SMEM_FWD = STAGE_FWD + FFT + 16;
  static constexpr size_t SMEM_INV = STAGE_INV + FFT + TAB + 16;
};
constexpr int kCtasPerSm = 3;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

// K2 on TMA: Z[n][p] = sum_k s_in scale_fwd[k] v[k][p] e^{+2 pi i kn/Nt}, n = 0..Nt/2.
template <int LOGM>
__global__ void __launch_bounds__(TmaGeo<LOGM>::NT, kCtasPerSm)
    k_time_fwd_tma(const __grid_constant__ CUtensorMap map_even, const __grid_constant__ CUtensorMap map_odd,
                   double2* __restrict__ Z, int ns, int n_tiles, const double* __restrict__ sf, double s_in,
                   const double2* __restrict__ twb) {
  using G = TmaGeo<LOGM>;
  constexpr int M = G::M, NTIME = G::NTIME, B = G::B, NT = G::NT, BS = G::BS, E = 16;
  constexpr int LE = 4, rem = LOGM % LE;
  constexpr int R = rem == 3 ? 8 : rem == 2 ? 4 : rem == 1 ? 2 : E;
  constexpr int NB = M / R, PER = E / R;
  extern __shared__ __align__(128) unsigned char smem_raw[];  // TMA destinations: 128-byte aligned
  unsigned char* base = smem_raw;  // (no integer round trip: the compiler must keep the shared state space)
  const int off = ns & 1;       // odd levels start 8 bytes off a 16-byte boundary when ns is odd
  const int po = B + 2 * off;   // row pitch of the odd-level box
  double* stage = reinterpret_cast<double*>(base);                            // even levels [M][B]
  double* stage_o = reinterpret_cast<double*>(base + G::STAGE_EVEN) + off;    // odd levels [M][po], column c at +off
  double2* fb = reinterpret_cast<double2*>(base + G::STAGE_FWD);              // B packed M-point buffers
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + G::STAGE_FWD + G::FFT);
  const int tid = int(threadIdx.x);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto fetch = [&](int tile) {  // one thread: both boxes of the tile, one barrier phase
    mbar_arrive_expect_tx(bar, uint32_t(M * (B + po) * sizeof(double)));
#pragma unroll
    for (int bi = 0; bi < G::NBF; ++bi) {
      tma_load_2d(stage + bi * G::RF * B, &map_even, tile * B, bi * G::RF, bar);
      tma_load_2d(base + G::STAGE_EVEN + size_t(bi) * G::RF * po * sizeof(double), &map_odd, ns - off + tile * B,
                  bi * G::RF, bar);
    }
  };
  int tile = int(blockIdx.x);
  uint32_t phase = 0;
  if (tid == 0 && tile < n_tiles) fetch(tile);
  const int c = tid % B;  // NT is a multiple of B: a thread keeps its column in every loop below
  const double2* twT = twb + NTIME;  // e^{-2 pi i n/Nt}; the forward kernel here is e^{+...}
  for (; tile < n_tiles; tile += int(gridDim.x)) {
    const int p0 = tile * B;
    mbar_wait(bar, phase);
    phase ^= 1u;
    // first Stockham pass straight from the staged tile (block_fft_columns_from's loader)
    double2 v[PER][R];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = (tid + q * NT) / B;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int m = j + r * NB;
        v[q][r] = make_double2(__ldg(sf + 2 * m) * (s_in * stage[m * B + c]),
                               __ldg(sf + 2 * m + 1) * (s_in * stage_o[m * po + c]));
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = (tid + q * NT) / B;
      Dft<R, 1>::run(v[q]);
#pragma unroll
      for (int r = 0; r < R; ++r) fb[c * BS + pad16(j * R + r)] = v[q][r];
    }
    __syncthreads();  // the staging buffer has been read by every thread: refill it
    {
      const int next = tile + int(gridDim.x);
      if (tid == 0 && next < n_tiles) fetch(next);
    }
    fft_passes<LOGM, 1, BS, E, R, CtaSync>(fb, twb + M, tid, NT);

    // Hermitian half of the real transform from the packed one; a thread's bins are
    // n = tid / B + i (NT / B); loads of a batch are issued before its first product
    const int p = p0 + c;
    constexpr int STEP = NT / B, ITER = (M / 2) / STEP + 1, UB = 3;
    const double2* s = fb + c * BS;
    if (p < ns) {
#pragma unroll
      for (int i0 = 0; i0 < ITER; i0 += UB) {
        double2 a[UB], bq[UB], w[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int n = tid / B + (i0 + u) * STEP;
          if (i0 + u < ITER && n <= M / 2) {
            a[u] = s[pad16(n)];
            bq[u] = s[pad16((M - n) & (M - 1))];
            w[u] = cconj(__ldg(twT + n));  // e^{+2 pi i n/Nt}
          }
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int n = tid / B + (i0 + u) * STEP;
          if (i0 + u < ITER && n <= M / 2) {
            if (n == 0) {
              Z[p] = make_double2(a[u].x + a[u].y, 0.0);
              Z[size_t(M) * ns + p] = make_double2(a[u].x - a[u].y, 0.0);
            } else {
              const double2 P = cadd(a[u], cconj(bq[u])), Q = csub(a[u], cconj(bq[u]));
              const double2 iwQ = mul_si<1>(cmul(w[u], Q));
              Z[size_t(n) * ns + p] = cscale(csub(P, iwQ), 0.5);
              if (n != M - n) Z[size_t(M - n) * ns + p] = cscale(cconj(cadd(P, iwQ)), 0.5);
            }
          }
        }
      }
    }
    __syncthreads();  // the buffers are rewritten by the next tile's first pass
  }
}

// K4 on TMA: z[k][p] = Re(scale_bwd[k]/Nt sum_n Z_n e^{-2 pi i kn/Nt}), Z_{Nt-n} = conj(Z_n).
template <int LOGM>
__global__ void __launch_bounds__(TmaGeo<LOGM>::NT, kCtasPerSm)
    k_time_inv_tma(const __grid_constant__ CUtensorMap tmap, double* __restrict__ z, int ns, int n_tiles,
                   const double* __restrict__ sb, const double2* __restrict__ twb) {
  using G = TmaGeo<LOGM>;
  constexpr int M = G::M, NTIME = G::NTIME, B = G::B, NT = G::NT, BS = G::BS, RB = G::RB;
  extern __shared__ __align__(128) unsigned char smem_raw[];  // TMA destinations: 128-byte aligned
  unsigned char* base = smem_raw;  // (no integer round trip: the compiler must keep the shared state space)
  double2* stage = reinterpret_cast<double2*>(base);                      // spectrum rows [2 RB][B]
  double2* fb = reinterpret_cast<double2*>(base + G::STAGE_INV);
  double* sbs = reinterpret_cast<double*>(base + G::STAGE_INV + G::FFT);  // scale_bwd / Nt
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + G::STAGE_INV + G::FFT + G::TAB);
  const int tid = int(threadIdx.x);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  const double inv_nt = 1.0 / double(NTIME);
  if constexpr (G::TABLE)
    for (int i = tid; i < NTIME; i += NT) sbs[i] = __ldg(sb + i) * inv_nt;
  __syncthreads();
  auto fetch = [&](int tile) {
    mbar_arrive_expect_tx(bar, uint32_t(G::STAGE_INV));
#pragma unroll
    for (int bi = 0; bi < G::NBI; ++bi)  // rows past n_time/2 are zero filled
      tma_load_2d(stage + bi * RB * B, &tmap, 2 * tile * B, bi * RB, bar);
  };
  int tile = int(blockIdx.x);
  uint32_t phase = 0;
  if (tid == 0 && tile < n_tiles) fetch(tile);
  const int c = tid % B;
  const double2* twT = twb + NTIME;
  constexpr int STEP = NT / B;
  for (; tile < n_tiles; tile += int(gridDim.x)) {
    const int p0 = tile * B;
    mbar_wait(bar, phase);
    phase ^= 1u;
    // packed inverse input from the bin pairs (n, M - n) of the staged half spectrum
    {
      constexpr int ITER = (M / 2) / STEP + 1, UB = 3;
      double2* s = fb + c * BS;
#pragma unroll
      for (int i0 = 0; i0 < ITER; i0 += UB) {
        double2 ya[UB], yb[UB], w[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int n = tid / B + (i0 + u) * STEP;
          if (i0 + u < ITER && n <= M / 2) {
            ya[u] = stage[n * B + c];
            yb[u] = stage[(M - n) * B + c];
            w[u] = __ldg(twT + n);  // e^{-2 pi i n/Nt}
          }
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int n = tid / B + (i0 + u) * STEP;
          if (i0 + u < ITER && n <= M / 2) {
            if (n == 0) {  // Y_0 and Y_M are both solved rows (alpha_circulant.hpp:158-166)
              const double2 A = cadd(ya[u], yb[u]), Bv = csub(ya[u], yb[u]);
              s[0] = cadd(A, mul_si<1>(Bv));
            } else {
              const double2 A = cadd(ya[u], cconj(yb[u]));
              const double2 Bn = cmul(csub(ya[u], cconj(yb[u])), w[u]);
              s[pad16(n)] = cadd(A, mul_si<1>(Bn));
              if (n != M - n) s[pad16(M - n)] = cadd(cconj(A), mul_si<1>(cconj(Bn)));
            }
          }
        }
      }
    }
    __syncthreads();  // staging consumed, packed input complete
    {
      const int next = tile + int(gridDim.x);
      if (tid == 0 && next < n_tiles) fetch(next);
    }
    block_fft<LOGM, -1, BS, 16>(fb, twb + M, B);
    const int p = p0 + c;
    if (p < ns) {
      const double2* s = fb + c * BS;
      constexpr int ITER = NTIME / STEP;  // a thread's levels kk = tid / B + i STEP
#pragma unroll 8
      for (int i = 0; i < ITER; ++i) {
        const int kk = tid / B + i * STEP;
        const double val = reinterpret_cast<const double*>(s + pad16(kk >> 1))[kk & 1];
        z[size_t(kk) * ns + p] = (G::TABLE ? sbs[kk] : __ldg(sb + kk) * inv_nt) * val;
      }
    }
    __syncthreads();
  }
}

namespace {

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// [rows][2 ns] doubles, row stride 16 ns bytes, boxes of [box_rows][box_cols]
bool make_map(CUtensorMap* map, const void* base, int ns, int rows, int box_cols, int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cuuint64_t(2) * cuuint64_t(ns), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(16) * cuuint64_t(ns)};
  const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// FPC_TIME_TMA: 0 = off, f = forward only, i = inverse only (A/B, debugging); default both
bool tma_enabled(bool inverse) {
  static const int mode = [] {
    const char* e = std::getenv("FPC_TIME_TMA");
    if (!e || !e[0]) return 3;
    return e[0] == '0' ? 0 : e[0] == 'f' ? 1 : e[0] == 'i' ? 2 : 3;
  }();
  return (mode & (inverse ? 2 : 1)) != 0;
}

template <class K>
cudaError_t prep_tma(K kernel, size_t smem) {
  // all of the L1/shared array as shared memory: three CTAs of ~67 KB, and nothing here is
  // re-read through L1 but the 4 KB of twiddles
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

}  // namespace

bool time_tma_supported(int n_space, int n_time, const void* in, bool inverse) {
  static const bool t1024 = [] {  // n_time = 1024: the 2-CTA split kernels unless FPC_TIME_TMA_1024=1 (A/B)
    const char* e = std::getenv("FPC_TIME_TMA_1024");
    return e && e[0] == '1';
  }();
  if (!tma_enabled(inverse) || (n_time != 128 && n_time != 256 && n_time != 512 && !(n_time == 1024 && t1024)))
    return false;
  if (reinterpret_cast<uintptr_t>(in) & 15) return false;
  const int b = 2048 / (n_time / 2);
  return (n_space + b - 1) / b >= 2 * sm_count() && encode_fn() != nullptr;
}

cudaError_t launch_time_fwd_tma(const double* v, double2* Z, int n_space, int n_time, const double* scale_fwd,
                                double s_in, const double2* tw_base, cudaStream_t st) {
  alignas(64) CUtensorMap map, map_odd;
#define CALL(LM)                                                                                         \
  {                                                                                                      \
    using G = TmaGeo<LM>;                                                                                \
    if (!make_map(&map, v, n_space, G::M, G::B, G::RF) ||                                                \
        !make_map(&map_odd, v, n_space, G::M, G::B + 2 * (n_space & 1), G::RF))                          \
      return cudaErrorInvalidValue;                                                                      \
    const int tiles = (n_space + G::B - 1) / G::B;                                                       \
    const int grid = tiles < kCtasPerSm * sm_count() ? tiles : kCtasPerSm * sm_count();                  \
    cudaError_t e = prep_tma(k_time_fwd_tma<LM>, G::SMEM_FWD);                                           \
    if (e != cudaSuccess) return e;                                                                      \
    k_time_fwd_tma<LM><<<grid, G::NT, G::SMEM_FWD, st>>>(map, map_odd, Z, n_space, tiles, scale_fwd, s_in, \
                                                         tw_base);                                       \
    note_launch();                                                                                       \
  }
  if (n_time == 1024) CALL(9) else if (n_time == 512) CALL(8) else if (n_time == 256) CALL(7) else if (n_time == 128) CALL(6) else return cudaErrorNotSupported;
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_time_inv_tma(const double2* Z, double* z, int n_space, int n_time, const double* scale_bwd,
                                const double2* tw_base, cudaStream_t st) {
  alignas(64) CUtensorMap map;
#define CALL(LM)                                                                                     \
  {                                                                                                  \
    using G = TmaGeo<LM>;                                                                            \
    if (!make_map(&map, Z, n_space, G::M + 1, 2 * G::B, G::RB)) return cudaErrorInvalidValue;        \
    const int tiles = (n_space + G::B - 1) / G::B;                                                   \
    const int grid = tiles < kCtasPerSm * sm_count() ? tiles : kCtasPerSm * sm_count();              \
    cudaError_t e = prep_tma(k_time_inv_tma<LM>, G::SMEM_INV);                                       \
    if (e != cudaSuccess) return e;                                                                  \
    k_time_inv_tma<LM><<<grid, G::NT, G::SMEM_INV, st>>>(map, z, n_space, tiles, scale_bwd, tw_base); \
    note_launch();                                                                                   \
  }
  if (n_time == 1024) CALL(9) else if (n_time == 512) CALL(8) else if (n_time == 256) CALL(7) else if (n_time == 128) CALL(6) else return cudaErrorNotSupported;
#undef CALL
  return cudaGetLastError();
}

}  // namespace fpc
