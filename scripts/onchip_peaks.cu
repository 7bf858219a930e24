// On-chip roofs for the FFT kernels (development aid): fp64 FMA throughput and shared-memory
// bandwidth (16-byte accesses), measured on the whole GPU with CUDA events.
// fp64_add_gops: DADD instructions per second (the FFT butterflies are add-heavy: one flop each).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/onchip_peaks scripts/onchip_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dadd(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] + c;
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_smem(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 v = buf[(idx + u * 256) & 2047];
      acc.x += v.x;
      acc.y += v.y;
    }
    idx = (idx + 32) & 2047;
  }
  if (acc.x == 12345.678) out[0] = acc.y;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 1 << 14;
  k_dfma<<<sms * 4, 512>>>(d, iters);
  cudaEventRecord(e0);
  k_dfma<<<sms * 4, 512>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * iters * double(sms) * 4 * 512;
  printf("{\"fp64_fma_tflops\": %.2f, ", flops / ms / 1e9);
  k_dadd<<<sms * 4, 512>>>(d, iters);
  cudaEventRecord(e0);
  k_dadd<<<sms * 4, 512>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"fp64_add_gops\": %.1f, ", 8.0 * iters * double(sms) * 4 * 512 / ms / 1e6);
  k_smem<<<sms * 4, 256>>>(d, iters);
  cudaEventRecord(e0);
  k_smem<<<sms * 4, 256>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 16.0 * 8 * iters * double(sms) * 4 * 256;
  printf("\"smem_tbs\": %.2f, \"sms\": %d}\n", bytes / ms / 1e9, sms);
  return 0;
}
