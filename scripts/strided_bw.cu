// Effective HBM bandwidth of column-tile reads of a row-major [rows][ns] fp64 matrix, W columns
// (8W-byte row segments) per CTA, all rows of the tile per CTA (the time-FFT access pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_timing/strided_bw scripts/strided_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W>
__global__ void __launch_bounds__(512) k_tile(const double* __restrict__ v, int ns, int rows, double* out) {
  const int p0 = blockIdx.x * W;
  double acc = 0;
  constexpr int U = 16;
  for (int e0 = threadIdx.x; e0 < W * rows; e0 += U * 512) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * 512;
      const int c = e % W, kk = e / W;
      x[u] = (e < W * rows && p0 + c < ns) ? v[size_t(kk) * ns + p0 + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += x[u];
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int W>
void run(const double* v, int ns, int rows, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = (ns + W - 1) / W;
  k_tile<W><<<grid, 512>>>(v, ns, rows, out);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) k_tile<W><<<grid, 512>>>(v, ns, rows, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  printf("W=%3d (%4d B segments): %8.1f us  %7.0f GB/s\n", W, 8 * W, ms * 1e3, double(ns) * rows * 8 / ms / 1e6);
}

int main() {
  const int ns = 8191, rows = 2048;
  double *v, *out;
  cudaMalloc(&v, size_t(ns) * rows * 8 + 64);
  cudaMalloc(&out, 8);
  cudaMemset(v, 0, size_t(ns) * rows * 8);
  run<1>(v, ns, rows, out);
  run<4>(v, ns, rows, out);
  run<8>(v, ns, rows, out);
  run<16>(v, ns, rows, out);
  run<32>(v, ns, rows, out);
  run<64>(v, ns, rows, out);
  return 0;
}
