// kernels_full.cu -- InnerSweep::full (alpha_circulant.hpp:158-159, 177-198): every one of the Nt
// frequencies is solved (no conjugate mirror), and the inverse time transform is a full complex
// FFT whose imaginary residue is measured (the reference throws when it exceeds 1e-10 of the
// output norm, alpha_circulant.hpp:196-198).  A diagnostic path: the half sweep is the default.
#include "fft_block.cuh"
#include "kernels.cuh"

namespace fpc {

namespace {
// grid = dots_grid(): the per-CTA partials are summed by launch_reduce over dots_grid() rows

__host__ __device__ constexpr int skew_f(int m) {
  return m < 16 ? padded(m) : padded(m) + ((9 - padded(m) % 8) % 8);
}

template <int LOGN>
struct FGeo {
  static constexpr int N = 1 << LOGN;
  static constexpr int E = N < 16 ? N : 16;
  static constexpr int B = (4096 / N) > 1 ? 4096 / N : 1;
  static constexpr int NT = B * N / E;
  static constexpr int BS = B > 1 ? skew_f(N) : padded(N);
  static constexpr size_t SMEM = size_t(B) * BS * sizeof(double2);
};

template <class K>
cudaError_t prep_f(K kernel, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  return cudaSuccess;
}
}  // namespace

// rows n = Nt/2+1 .. Nt-1 of the forward spectrum: Z_n = conj(Z_{Nt-n}) -- what the reference's
// complex forward FFT of a real (scaled) input produces for them
__global__ void k_mirror_fill(double2* __restrict__ Z, int ns, int nt) {
  const int M = nt / 2;
  const size_t total = size_t(nt - M - 1) * ns;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t n = M + 1 + e / ns, p = e % ns;
    Z[n * ns + p] = cconj(Z[(nt - n) * ns + p]);
  }
}

// z[k][p] = Re( scale_bwd[k]/Nt * sum_n Z[n][p] e^{-2 pi i kn/Nt} ), plus per-CTA partial sums of
// Im^2 and |.|^2 of the scaled complex result (alpha_circulant.hpp:187-195)
template <int LOGN>
__global__ void __launch_bounds__(FGeo<LOGN>::NT)
    k_time_inv_full(const double2* __restrict__ Z, double* __restrict__ z, int ns,
                    const double* __restrict__ sb, const double2* __restrict__ twb,
                    double* __restrict__ partial) {
  using G = FGeo<LOGN>;
  constexpr int N = G::N, B = G::B, NT = G::NT, BS = G::BS, E = G::E;
  extern __shared__ double2 smem[];
  __shared__ double red[2][NT / 32 + 1];
  double im2 = 0.0, tot2 = 0.0;
  const int ntiles = (ns + B - 1) / B;
  const double inv_nt = 1.0 / double(N);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int p0 = tile * B;
    for (int e = threadIdx.x; e < B * N; e += NT) {
      const int c = e % B, n = e / B;
      const int p = p0 + c;
      smem[c * BS + pad16(n)] = p < ns ? Z[size_t(n) * ns + p] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    block_fft<LOGN, -1, BS, E>(smem, twb + N, B);
    for (int e = threadIdx.x; e < B * N; e += NT) {
      const int c = e % B, kk = e / B;
      const int p = p0 + c;
      if (p >= ns) continue;
      const double s = __ldg(sb + kk) * inv_nt;
      const double2 v = cscale(smem[c * BS + pad16(kk)], s);
      z[size_t(kk) * ns + p] = v.x;
      im2 = fma(v.y, v.y, im2);
      tot2 = fma(v.x, v.x, fma(v.y, v.y, tot2));
    }
    __syncthreads();
  }
  // deterministic block reduction of the two partials
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    im2 += __shfl_xor_sync(0xffffffffu, im2, off);
    tot2 += __shfl_xor_sync(0xffffffffu, tot2, off);
  }
  if (lane == 0) {
    red[0][warp] = im2;
    red[1][warp] = tot2;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += red[threadIdx.x][w];
    partial[size_t(blockIdx.x) * 2 + threadIdx.x] = s;
  }
}

cudaError_t launch_mirror_fill(double2* Z, int n_space, int n_time, cudaStream_t st) {
  k_mirror_fill<<<148 * 4, 256, 0, st>>>(Z, n_space, n_time); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_time_inv_full(const double2* Z, double* z, int n_space, int n_time,
                                 const double* scale_bwd, const double2* tw_base, double* partial,
                                 cudaStream_t st) {
  int l = 0;
  while ((1 << l) < n_time) ++l;
  cudaError_t err = cudaSuccess;
#define CALL(LN)                                                                           \
  {                                                                                        \
    using G = FGeo<LN>;                                                                    \
    if ((err = prep_f(k_time_inv_full<LN>, G::SMEM)) != cudaSuccess) return err;           \
    k_time_inv_full<LN><<<dots_grid(), G::NT, G::SMEM, st>>>(Z, z, n_space, scale_bwd, tw_base, partial); note_launch(); \
  }
  switch (l) {
    case 2: CALL(2); break;
    case 3: CALL(3); break;
    case 4: CALL(4); break;
    case 5: CALL(5); break;
    case 6: CALL(6); break;
    case 7: CALL(7); break;
    case 8: CALL(8); break;
    case 9: CALL(9); break;
    case 10: CALL(10); break;
    case 11: CALL(11); break;
    case 12: CALL(12); break;
    case 13: CALL(13); break;
    default: return cudaErrorInvalidValue;
  }
#undef CALL
  return cudaGetLastError();
}

}  // namespace fpc
