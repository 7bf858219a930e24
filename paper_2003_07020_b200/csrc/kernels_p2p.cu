// kernels_p2p.cu -- the sharded PC apply's transpositions (time <-> space <-> frequency
// layouts around alpha_circulant.hpp:146-198) as ONE peer-store kernel per exchange over NVLink.
//
// The NCCL path packs every destination's block into a send buffer, runs all_to_all_single, and
// concatenates the received blocks into the consumer's layout (three passes over the data plus the
// transfer).  Here each rank's kernel reads its source matrix once and stores every element straight
// into its final slot of the owning rank's receive buffer (an IPC-mapped peer pointer; the own rank's
// buffer is local), so packing, transfer and unpacking are one pass.  Ordering: the kernel ends with
// a system-scope fence, and the caller follows it with a stream-ordered NCCL barrier (one-element
// all-reduce on the same stream): a consumer reads its buffer only after every producer's kernel has
// completed, and a producer writes a buffer again only after the consumer of its previous contents
// has passed a later barrier (every exchange uses its own buffer).
//
// Source: a [rows][cols] matrix of elements of ES doubles (1: real, 2: complex), row stride cols.
// The split dimension (columns if split_cols, else rows) is partitioned by off[0..G]; element (i, j)
// owned by d goes to
//   split_cols: dst[d][(row_base + i) * stride[d] + col_base + (j - off[d])]
//   split rows: dst[d][(row_base + i - off[d]) * stride[d] + col_base + j]
// (all four exchanges of the reference ordering and both of the commuted one are instances).
#include <algorithm>

#include "kernels.cuh"

namespace fpc {

template <int ES>
struct Elem;
template <>
struct Elem<1> {
  using T = double;
};
template <>
struct Elem<2> {
  using T = double2;
};

// Tiles of one source row x kChunk columns, one tile per CTA iteration (one division per tile, none
// per element); every thread issues its kPer loads before its stores.
constexpr int kP2PThreads = 256, kP2PPer = 8, kP2PChunk = kP2PThreads * kP2PPer;

template <int ES, bool SPLIT_COLS>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_scatter(const double* __restrict__ src, int rows, int cols,
                                                             P2PScatter a, int nranks, int row_base, int col_base) {
  using T = typename Elem<ES>::T;
  const T* s = reinterpret_cast<const T*>(src);
  const int nchunk = (cols + kP2PChunk - 1) / kP2PChunk;
  const long ntile = long(rows) * nchunk;
  for (long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int i = int(tile / nchunk), j0 = int(tile - long(i) * nchunk) * kP2PChunk;
    const T* srow = s + size_t(i) * size_t(cols);
    T v[kP2PPer];
#pragma unroll
    for (int u = 0; u < kP2PPer; ++u) {
      const int j = j0 + int(threadIdx.x) + u * kP2PThreads;
      if (j < cols) v[u] = srow[j];
    }
    if constexpr (SPLIT_COLS) {
#pragma unroll
      for (int u = 0; u < kP2PPer; ++u) {
        const int j = j0 + int(threadIdx.x) + u * kP2PThreads;
        if (j >= cols) continue;
        int d = 0;
#pragma unroll
        for (int r = 1; r < kP2PMaxRanks; ++r)
          if (r < nranks && j >= a.off[r]) d = r;
        reinterpret_cast<T*>(a.dst[d])[size_t(row_base + i) * size_t(a.stride[d]) + size_t(col_base + j - a.off[d])] =
            v[u];
      }
    } else {
      int d = 0;
#pragma unroll
      for (int r = 1; r < kP2PMaxRanks; ++r)
        if (r < nranks && i >= a.off[r]) d = r;
      T* drow = reinterpret_cast<T*>(a.dst[d]) + size_t(row_base + i - a.off[d]) * size_t(a.stride[d]) + col_base;
#pragma unroll
      for (int u = 0; u < kP2PPer; ++u) {
        const int j = j0 + int(threadIdx.x) + u * kP2PThreads;
        if (j < cols) drow[j] = v[u];
      }
    }
  }
  // one system-scope fence per CTA, after the CTA barrier (cumulative over the CTA's stores), instead
  // of one per thread
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

cudaError_t launch_p2p_scatter(const double* src, int rows, int cols, int es, bool split_cols, const P2PScatter& a,
                               int nranks, int row_base, int col_base, cudaStream_t st) {
  const size_t total = size_t(rows) * size_t(cols);
  if (total == 0) return cudaSuccess;
  const size_t ntile = size_t(rows) * size_t((cols + kP2PChunk - 1) / kP2PChunk);
  const int grid = int(std::min<size_t>(ntile, size_t(148) * 8));
  if (es == 1 && split_cols)
    { k_p2p_scatter<1, true><<<grid, kP2PThreads, 0, st>>>(src, rows, cols, a, nranks, row_base, col_base); note_launch(); }
  else if (es == 1)
    { k_p2p_scatter<1, false><<<grid, kP2PThreads, 0, st>>>(src, rows, cols, a, nranks, row_base, col_base); note_launch(); }
  else if (split_cols)
    { k_p2p_scatter<2, true><<<grid, kP2PThreads, 0, st>>>(src, rows, cols, a, nranks, row_base, col_base); note_launch(); }
  else
    { k_p2p_scatter<2, false><<<grid, kP2PThreads, 0, st>>>(src, rows, cols, a, nranks, row_base, col_base); note_launch(); }
  return cudaGetLastError();
}

}  // namespace fpc
