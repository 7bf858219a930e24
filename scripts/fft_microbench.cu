// Microbenchmark of the smem FFT engine: each CTA loads B buffers of N complex, runs a forward +
// inverse transform, stores.  Reports ns per transform pair and effective fp64 throughput.
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2003_07020_b200/csrc/fft_block.cuh"
using namespace fpc;

template <int LOGN, int B, int E, int MINB>
__global__ void __launch_bounds__(B * (1 << LOGN) / E, MINB) kbench(const double2* __restrict__ in, double2* __restrict__ out,
                                                             const double2* __restrict__ twb) {
  constexpr int N = 1 << LOGN;
  constexpr int BS = B > 1 ? padded(N) + 1 : padded(N);
  extern __shared__ double2 sm[];
  const int NT = blockDim.x;
  const double2* src = in + size_t(blockIdx.x) * B * N;
  for (int e = threadIdx.x; e < B * N; e += NT) sm[(e / N) * BS + pad16(e % N)] = src[e];
  __syncthreads();
  block_fft<LOGN, -1, BS, E>(sm, twb + N, B);
  block_fft<LOGN, 1, BS, E>(sm, twb + N, B);
  double2* dst = out + size_t(blockIdx.x) * B * N;
  for (int e = threadIdx.x; e < B * N; e += NT) dst[e] = sm[(e / N) * BS + pad16(e % N)];
}

template <int LOGN, int B, int E, int MINB = 1>
void run(const double2* in, double2* out, const double2* tw, int total_ffts) {
  constexpr int N = 1 << LOGN;
  constexpr int BS = B > 1 ? padded(N) + 1 : padded(N);
  size_t smem = size_t(B) * BS * 16;
  cudaFuncSetAttribute(kbench<LOGN, B, E, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(kbench<LOGN, B, E, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int grid = total_ffts / B;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) kbench<LOGN, B, E, MINB><<<grid, B * N / E, smem>>>(in, out, tw);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) kbench<LOGN, B, E, MINB><<<grid, B * N / E, smem>>>(in, out, tw);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double t = ms / 10 * 1e-3;
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kbench<LOGN, B, E, MINB>, B * N / E, smem);
  double flops = 2.0 * 5.0 * N * LOGN * total_ffts;
  printf("MINB=%d N=%5d B=%2d E=%2d thr=%4d smem=%6zu occ=%d : %8.1f us  %.2f us/Mpt-pair  %.1f TF(5NlogN)  %.0f GB/s\n", MINB, N, B, E,
         B * N / E, smem, occ, t * 1e6, t * 1e6 / (double(N) * total_ffts / 1e6), flops / t / 1e12,
         32.0 * N * total_ffts / t / 1e9);
  cudaError_t err = cudaGetLastError(); if (err) printf("err %s\n", cudaGetErrorString(err));
}

int main() {
  const size_t total = size_t(1) << 24;  // complex values per launch (256 MB in)
  double2 *in, *out, *tw;
  cudaMalloc(&in, total * 16); cudaMalloc(&out, total * 16);
  cudaMemset(in, 0, total * 16);
  std::vector<double2> h(size_t(2) << 17);
  for (int l = 0; l <= 17; ++l) { size_t N = size_t(1) << l; for (size_t t = 0; t < N; ++t) { double th = -2 * M_PI * t / N; h[N + t] = make_double2(cos(th), sin(th)); } }
  cudaMalloc(&tw, h.size() * 16); cudaMemcpy(tw, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  run<13, 1, 16, 1>(in, out, tw, total >> 13);
  run<12, 1, 16, 3>(in, out, tw, total >> 12);
  run<12, 1, 16, 2>(in, out, tw, total >> 12);
  run<12, 1, 16, 3>(in, out, tw, total >> 12);
  run<12, 2, 16, 1>(in, out, tw, total >> 12);
  run<11, 2, 16, 2>(in, out, tw, total >> 11);
  run<11, 2, 16, 3>(in, out, tw, total >> 11);
  run<10, 4, 16, 2>(in, out, tw, total >> 10);
  run<10, 4, 16, 3>(in, out, tw, total >> 10);
  run<10, 2, 16, 4>(in, out, tw, total >> 10);
  run<10, 2, 16, 6>(in, out, tw, total >> 10);
  run<10, 1, 16, 8>(in, out, tw, total >> 10);
  run<8, 16, 16, 3>(in, out, tw, total >> 8);
  return 0;
}
