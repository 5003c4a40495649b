// Ordered stream compaction / exclusive scan with the element count read on
// the device, so whole stages chain without host synchronisation: a
// single-pass decoupled look-back scan (one launch per scan). The grid is
// persistent and takes chunks from a ticket counter, so launch sizes never
// depend on device-side counts; n comes from *n_dev when non-null (else
// n_host).
#pragma once
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

inline int64_t scan_chunks(int64_t n_max, int items = kScanItems) {
  const int64_t chunk = (int64_t)kScanThreads * items;
  return (n_max + chunk - 1) / chunk + 1;
}

// Elements per thread of a functor's scan: F::kItems when it declares one
// (heavy loads: fewer per thread, more chunks in flight), else kScanItems.
template <class F, class = void>
struct scan_items {
  static constexpr int value = kScanItems;
};
template <class F>
struct scan_items<F, decltype((void)F::kItems)> {
  static constexpr int value = F::kItems;
};

// ---- single pass: decoupled look-back ----------------------------------------
// Chunks are taken in order from a ticket counter; each publishes its
// aggregate, then (after looking back over its predecessors) its inclusive
// prefix. The functor is split so each element is decoded once:
// `Item load(int64_t i)`, `T value(const Item &)` and
// `void emit(int64_t i, T prefix, const Item &)`.
template <typename T>
struct ScanStatus {
  T agg, incl;
  int flag;  // 0 none, 1 aggregate, 2 inclusive prefix
};

// L2 read of a status value written by another SM (never a stale L1 line)
template <typename T>
__device__ __forceinline__ T ldcg_value(const T *p) {
  static_assert(sizeof(T) % 4 == 0, "scan values are whole 32-bit words");
  T v;
  const int *src = reinterpret_cast<const int *>(p);
  int *dst = reinterpret_cast<int *>(&v);
#pragma unroll
  for (int k = 0; k < (int)(sizeof(T) / 4); ++k) dst[k] = __ldcg(src + k);
  return v;
}

template <typename T>
__device__ __forceinline__ T shfl_xor_value(const T &v, int o) {
  T r;
  const int *src = reinterpret_cast<const int *>(&v);
  int *dst = reinterpret_cast<int *>(&r);
#pragma unroll
  for (int k = 0; k < (int)(sizeof(T) / 4); ++k) dst[k] = __shfl_xor_sync(0xffffffffu, src[k], o);
  return r;
}

template <typename T>
__device__ __forceinline__ void scan_publish(ScanStatus<T> *st, const T &agg, const T &incl,
                                             int flag) {
  volatile ScanStatus<T> *v = st;
  if (flag == 1) {
    st->agg = agg;
  } else {
    st->incl = incl;
  }
  __threadfence();
  v->flag = flag;
}

template <class F, typename T>
__global__ void __launch_bounds__(kScanThreads)
    onepass_scan_kernel(const __grid_constant__ F f, const int64_t *n_dev, int64_t n_host,
                        ScanStatus<T> *status, unsigned long long *ticket, T *total) {
  pdl_wait();
  using Scan = cub::BlockScan<T, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long tile_s;
  __shared__ T prefix_s;
  const int64_t n = scan_len(n_dev, n_host);
  constexpr int kItems = scan_items<F>::value;
  constexpr int64_t kChunk = (int64_t)kScanThreads * kItems;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  while (true) {
    if (threadIdx.x == 0) tile_s = (long long)atomicAdd(ticket, 1ull);
    __syncthreads();
    const int64_t c = tile_s;
    if (c >= nchunks) break;
    typename F::Item item[kItems];
    T v[kItems], ex[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t i = c * kChunk + (int64_t)threadIdx.x * kItems + it;
      item[it] = i < n ? f.load(i) : typename F::Item();
      v[it] = i < n ? f.value(item[it]) : T(0);
    }
    T agg;
    Scan(tmp).ExclusiveSum(v, ex, agg);
    if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 tiles at a time
      const int lane = threadIdx.x;
      T prefix = T(0);
      if (c == 0) {
        if (lane == 0) scan_publish(status + c, agg, agg, 2);
      } else {
        if (lane == 0) scan_publish(status + c, agg, agg, 1);
        for (int64_t q0 = c - 1;; q0 -= 32) {
          const int64_t q = q0 - lane;
          int fl = 2;  // before tile 0: an inclusive prefix of zero
          T val = T(0);
          if (q >= 0) {
            volatile ScanStatus<T> *sq = status + q;
            while ((fl = sq->flag) == 0) {
            }
            __threadfence();
            val = fl == 2 ? ldcg_value(&status[q].incl) : ldcg_value(&status[q].agg);
          }
          const unsigned inc = __ballot_sync(0xffffffffu, fl == 2);
          const int first = inc ? __ffs(inc) - 1 : 32;  // nearest inclusive tile
          T part = lane <= first ? val : T(0);
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) part = part + shfl_xor_value(part, o);
          prefix = prefix + part;
          if (inc) break;
        }
        if (lane == 0) scan_publish(status + c, agg, prefix + agg, 2);
      }
      if (lane == 0) {
        if (c == nchunks - 1 && total) *total = prefix + agg;
        prefix_s = prefix;
      }
    }
    __syncthreads();
    const T base = prefix_s;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t i = c * kChunk + (int64_t)threadIdx.x * kItems + it;
      if (i < n) f.emit(i, base + ex[it], item[it]);
    }
    __syncthreads();
  }
  if (nchunks == 0 && blockIdx.x == 0 && threadIdx.x == 0 && total) *total = T(0);
}

// Workspace of onepass_scan for n_max elements: status words + ticket.
template <typename T>
inline size_t onepass_status_bytes(int64_t n_max) {  // 8-byte aligned ticket after it
  return (sizeof(ScanStatus<T>) * (size_t)scan_chunks(n_max, 1) + 15) & ~(size_t)15;
}

template <typename T>
inline size_t onepass_bytes(int64_t n_max) {
  return onepass_status_bytes<T>(n_max) + 64;
}

template <class F, typename T>
inline void onepass_scan(const F &f, const int64_t *n_dev, int64_t n_host, int64_t n_max,
                         void *ws, T *total, cudaStream_t st) {
  const size_t sbytes = onepass_status_bytes<T>(n_max);
  cudaMemsetAsync(ws, 0, sbytes + 64, st);
  launch_k(onepass_scan_kernel<F, T>, kScanGrid, kScanThreads, 0, st, f, n_dev, n_host, (ScanStatus<T> *)ws, (unsigned long long *)((char *)ws + sbytes),
      total);
  note_launches(1);
}

}  // namespace fvv
