// Ordered stream compaction / exclusive scan with the element count read on
// the device, so whole stages chain without host synchronisation.
//
// reduce-then-scan over fixed chunks of kThreads*kItems elements:
//   1. chunk_reduce: per chunk sum of f.value(i)            -> sums[c]
//   2. chunk_scan  : one block turns sums[] into exclusive bases, *total
//   3. chunk_emit  : recompute values, block-scan, f.emit(i, base+prefix, v)
// A functor F provides `T value(int64_t i)` and
// `void emit(int64_t i, T prefix, T value)`; n comes from *n_dev when
// non-null (else n_host). The persistent grids loop over chunks, so launch
// sizes never depend on device-side counts.
#pragma once
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "fvv_common.cuh"

namespace fvv {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanChunk = kScanThreads * kScanItems;  // 1024 elements per chunk
constexpr int kScanGrid = 148 * 4;

__device__ __forceinline__ int64_t scan_len(const int64_t *n_dev, int64_t n_host) {
  return device_count(n_dev, n_host);
}

template <class F, typename T>
__global__ void __launch_bounds__(kScanThreads)
    chunk_reduce_kernel(const __grid_constant__ F f, const int64_t *n_dev, int64_t n_host, T *sums) {
  using Reduce = cub::BlockReduce<T, kScanThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  const int64_t n = scan_len(n_dev, n_host);
  const int64_t nchunks = (n + kScanChunk - 1) / kScanChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    T s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int64_t i = c * kScanChunk + (int64_t)threadIdx.x * kScanItems + it;
      if (i < n) s += f.value(i);
    }
    s = Reduce(tmp).Sum(s);
    if (threadIdx.x == 0) sums[c] = s;
    __syncthreads();
  }
}

// Single block: sums[c] <- exclusive prefix; *total <- grand total.
template <typename T>
__global__ void __launch_bounds__(1024)
    chunk_scan_kernel(T *sums, const int64_t *n_dev, int64_t n_host, T *total) {
  using Scan = cub::BlockScan<T, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ T carry;
  const int64_t n = scan_len(n_dev, n_host);
  const int64_t nchunks = (n + kScanChunk - 1) / kScanChunk;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nchunks; base += 1024) {
    const int64_t c = base + threadIdx.x;
    T v = c < nchunks ? sums[c] : T(0);
    T ex, agg;
    Scan(tmp).ExclusiveSum(v, ex, agg);
    if (c < nchunks) sums[c] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

template <class F, typename T>
__global__ void __launch_bounds__(kScanThreads)
    chunk_emit_kernel(const __grid_constant__ F f, const int64_t *n_dev, int64_t n_host, const T *bases) {
  using Scan = cub::BlockScan<T, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t n = scan_len(n_dev, n_host);
  const int64_t nchunks = (n + kScanChunk - 1) / kScanChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    T v[kScanItems], ex[kScanItems];
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int64_t i = c * kScanChunk + (int64_t)threadIdx.x * kScanItems + it;
      v[it] = i < n ? f.value(i) : T(0);
    }
    Scan(tmp).ExclusiveSum(v, ex);
    const T base = bases[c];
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int64_t i = c * kScanChunk + (int64_t)threadIdx.x * kScanItems + it;
      if (i < n) f.emit(i, base + ex[it], v[it]);
    }
    __syncthreads();
  }
}

// Runs the three phases on `st`. `sums` needs ceil(n_max / kScanChunk)
// elements, where n_max bounds the device-side count.
template <class F, typename T>
inline void ordered_scan(const F &f, const int64_t *n_dev, int64_t n_host, T *sums, T *total,
                         cudaStream_t st) {
  chunk_reduce_kernel<F, T><<<kScanGrid, kScanThreads, 0, st>>>(f, n_dev, n_host, sums);
  chunk_scan_kernel<T><<<1, 1024, 0, st>>>(sums, n_dev, n_host, total);
  chunk_emit_kernel<F, T><<<kScanGrid, kScanThreads, 0, st>>>(f, n_dev, n_host, sums);
  note_launches(3);
}

inline int64_t scan_chunks(int64_t n_max) { return (n_max + kScanChunk - 1) / kScanChunk + 1; }

}  // namespace fvv
