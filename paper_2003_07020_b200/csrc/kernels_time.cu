// kernels_time.cu -- the alpha-circulant preconditioner's time-direction FFTs (K2/K4,
// alpha_circulant.hpp:146-156 and 167-198) as persistent, double-buffered kernels.
//
// Each CTA walks column tiles (B spatial columns x all Nt time levels).  While tile i is being
// transformed in one shared-memory buffer set, the cp.async (LDGSTS) copies of tile i+1 land in the
// other, so HBM traffic overlaps the FFT work (the time FFTs need as many bytes as FLOPs/6, close
// to the B200 ridge).  Copies land directly in the FFT buffer layout (8-byte granules for the real
// input, 16-byte for the half spectrum); ragged columns are zero-filled by the copy itself.
// (TMA is not usable here: an odd Ns gives row strides that are not 16-byte multiples.)
#include <algorithm>

#include "fft_block.cuh"
#include "kernels.cuh"

namespace fpc {

namespace {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ constexpr int skew_t(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}

template <int LOGM, int B>
struct TGeo {
  static constexpr int M = 1 << LOGM;
  static constexpr int E = M < 16 ? M : 16;
  static constexpr int NT = B * M / E;
  static constexpr int BS = skew_t(M + 1);  // M + 1 slots: the inverse lands Z_0..Z_M raw
  static constexpr int SET = B * BS;         // one buffer set
  static constexpr size_t SMEM = size_t(2) * SET * sizeof(double2);
};

template <class K>
cudaError_t prep_t(K kernel, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaSuccess;
}

int sm_count() {
  static int n = [] {
    int dev = 0, c = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c;
  }();
  return n;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// K2: Z[n][p] = sum_k (s_in * scale_fwd[k]) v[k][p] e^{+2 pi i kn/Nt}, n = 0..Nt/2
// ------------------------------------------------------------------------------------------
template <int LOGM, int B>
__global__ void __launch_bounds__(TGeo<LOGM, B>::NT, 1)
    k_time_fwd_pipe(const double* __restrict__ v, double2* __restrict__ Z, int ns,
                    const double* __restrict__ sf, double s_in, const double2* __restrict__ twb) {
  using G = TGeo<LOGM, B>;
  constexpr int M = G::M, NTIME = 2 * M, NT = G::NT, BS = G::BS, SET = G::SET, E = G::E;
  extern __shared__ double2 smem[];
  const int ntiles = (ns + B - 1) / B;
  const double2* twT = twb + NTIME;

  auto issue = [&](int tile, double2* set) {
    const int p0 = tile * B;
    for (int e = threadIdx.x; e < B * NTIME; e += NT) {
      const int c = e % B, kk = e / B;
      const int p = p0 + c;
      double* dst = reinterpret_cast<double*>(set + c * BS + pad16(kk >> 1)) + (kk & 1);
      const bool ok = p < ns;
      cp_async8(dst, ok ? v + size_t(kk) * ns + p : v, ok);
    }
  };

  int tile = blockIdx.x;
  int cur = 0;
  if (tile < ntiles) issue(tile, smem);
  cp_commit();
  while (tile < ntiles) {
    const int next = tile + gridDim.x;
    double2* set = smem + cur * SET;
    if (next < ntiles) issue(next, smem + (cur ^ 1) * SET);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    // scale (alpha_circulant.hpp:149): x_k *= s_in * scale_fwd[k]
    for (int e = threadIdx.x; e < B * M; e += NT) {
      const int c = e / M, m = e - c * M;
      double2* q = set + c * BS + pad16(m);
      const double2 x = *q;
      *q = make_double2(__ldg(sf + 2 * m) * (s_in * x.x), __ldg(sf + 2 * m + 1) * (s_in * x.y));
    }
    __syncthreads();
    block_fft<LOGM, 1, BS, E>(set, twb + M, B);
    const int p0 = tile * B;
    for (int t = threadIdx.x; t < B * (M / 2 + 1); t += NT) {
      const int c = t % B, n = t / B;
      const int p = p0 + c;
      if (p >= ns) continue;
      const double2* s = set + c * BS;
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
    __syncthreads();  // the set is free for the copies issued next iteration
    cur ^= 1;
    tile = next;
  }
  cp_wait<0>();
}

// ------------------------------------------------------------------------------------------
// K4: z[k][p] = Re( scale_bwd[k]/Nt * sum_n Z_n e^{-2 pi i kn/Nt} ), Z_{Nt-n} = conj(Z_n)
// ------------------------------------------------------------------------------------------
template <int LOGM, int B>
__global__ void __launch_bounds__(TGeo<LOGM, B>::NT, 1)
    k_time_inv_pipe(const double2* __restrict__ Z, double* __restrict__ z, int ns,
                    const double* __restrict__ sb, const double2* __restrict__ twb) {
  using G = TGeo<LOGM, B>;
  constexpr int M = G::M, NTIME = 2 * M, NT = G::NT, BS = G::BS, SET = G::SET, E = G::E;
  extern __shared__ double2 smem[];
  const int ntiles = (ns + B - 1) / B;
  const double2* twT = twb + NTIME;

  auto issue = [&](int tile, double2* set) {
    const int p0 = tile * B;
    for (int e = threadIdx.x; e < B * (M + 1); e += NT) {
      const int c = e % B, n = e / B;
      const int p = p0 + c;
      const bool ok = p < ns;
      cp_async16(set + c * BS + pad16(n), ok ? Z + size_t(n) * ns + p : Z, ok);
    }
  };

  int tile = blockIdx.x;
  int cur = 0;
  if (tile < ntiles) issue(tile, smem);
  cp_commit();
  const double inv_nt = 1.0 / double(NTIME);
  while (tile < ntiles) {
    const int next = tile + gridDim.x;
    double2* set = smem + cur * SET;
    if (next < ntiles) issue(next, smem + (cur ^ 1) * SET);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    // repack the Hermitian half into the packed real-output transform, in place on (n, M-n)
    for (int t = threadIdx.x; t < B * (M / 2 + 1); t += NT) {
      const int c = t % B, n = t / B;
      double2* s = set + c * BS;
      if (n == 0) {  // Y_0 and Y_M are both solved rows (alpha_circulant.hpp:158-166)
        const double2 y0 = s[0], ym = s[pad16(M)];
        s[0] = cadd(cadd(y0, ym), mul_si<1>(csub(y0, ym)));
      } else {
        const double2 a = s[pad16(n)], bq = s[pad16(M - n)];
        const double2 w = __ldg(twT + n);  // e^{-2 pi i n/Nt}
        const double2 A = cadd(a, cconj(bq));
        const double2 Bn = cmul(csub(a, cconj(bq)), w);
        s[pad16(n)] = cadd(A, mul_si<1>(Bn));
        if (n != M - n) s[pad16(M - n)] = cadd(cconj(A), mul_si<1>(cconj(Bn)));
      }
    }
    __syncthreads();
    block_fft<LOGM, -1, BS, E>(set, twb + M, B);
    const int p0 = tile * B;
    for (int e = threadIdx.x; e < B * NTIME; e += NT) {
      const int c = e % B, kk = e / B;
      const int p = p0 + c;
      if (p >= ns) continue;
      const double val = reinterpret_cast<const double*>(set + c * BS + pad16(kk >> 1))[kk & 1];
      z[size_t(kk) * ns + p] = (__ldg(sb + kk) * inv_nt) * val;
    }
    __syncthreads();
    cur ^= 1;
    tile = next;
  }
  cp_wait<0>();
}

// ------------------------------------------------------------------------------------------
constexpr int kTB = 4;  // columns per tile (4 x 8 B = one 32-byte sector per time row)

#define FPC_DISPATCH_T(logm, CALL)         \
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
    default: return cudaErrorInvalidValue; \
  }

static int ilog2t(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// tiles of B columns: up to kTB (one 32-byte sector per time row), fewer when two buffer sets
// would not fit in shared memory, more for short transforms so a CTA keeps >= 64 threads
template <int LOGM>
constexpr int tile_b() {
  constexpr int M = 1 << LOGM, E = M < 16 ? M : 16;
  constexpr int a = (4096 / M) < kTB ? (4096 / M) : kTB;
  constexpr int a1 = a < 1 ? 1 : a;
  constexpr int b = 64 * E / M;
  return a1 > b ? a1 : b;
}

cudaError_t launch_time_fwd_pipe(const double* v, double2* Z, int n_space, int n_time,
                                 const double* scale_fwd, double s_in, const double2* tw_base,
                                 cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2t(n_time) - 1;
#define CALL(LM)                                                                           \
  {                                                                                        \
    constexpr int BB = tile_b<LM>();                                                       \
    using G = TGeo<LM, BB>;                                                                \
    if ((err = prep_t(k_time_fwd_pipe<LM, BB>, G::SMEM)) != cudaSuccess) return err;       \
    int occ = 1;                                                                           \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_time_fwd_pipe<LM, BB>, G::NT, G::SMEM); \
    const int tiles = (n_space + BB - 1) / BB;                                             \
    const int grid = std::min(tiles, std::max(1, occ) * sm_count());                       \
    k_time_fwd_pipe<LM, BB><<<grid, G::NT, G::SMEM, st>>>(v, Z, n_space, scale_fwd, s_in, tw_base); \
  }
  FPC_DISPATCH_T(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_time_inv_pipe(const double2* Z, double* z, int n_space, int n_time,
                                 const double* scale_bwd, const double2* tw_base, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const int lm = ilog2t(n_time) - 1;
#define CALL(LM)                                                                           \
  {                                                                                        \
    constexpr int BB = tile_b<LM>();                                                       \
    using G = TGeo<LM, BB>;                                                                \
    if ((err = prep_t(k_time_inv_pipe<LM, BB>, G::SMEM)) != cudaSuccess) return err;       \
    int occ = 1;                                                                           \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_time_inv_pipe<LM, BB>, G::NT, G::SMEM); \
    const int tiles = (n_space + BB - 1) / BB;                                             \
    const int grid = std::min(tiles, std::max(1, occ) * sm_count());                       \
    k_time_inv_pipe<LM, BB><<<grid, G::NT, G::SMEM, st>>>(Z, z, n_space, scale_bwd, tw_base); \
  }
  FPC_DISPATCH_T(lm, CALL)
#undef CALL
  return cudaGetLastError();
}

}  // namespace fpc
