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
#ifndef FVV_SCAN_ITEMS
#define FVV_SCAN_ITEMS 4
#endif
constexpr int kScanItems = FVV_SCAN_ITEMS;
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
//
// The grid's first wave takes ~600 chunks at once, so a late chunk's
// predecessors are still looking back themselves and it sums aggregates a
// long way. So a status is read in one L2 round trip, no fence between flag
// and value: 8-byte values share one 16-byte word with their flag; values of
// up to 24 bytes (the mesh's 5-slot counts) are split over two 16-byte
// halves that each carry the flag, and a reader takes a status only when
// both halves show the same nonzero flag (each half is written by one vector
// store, and a flag value is published once per status). Each lane reads
// FVV_SCAN_LB statuses of 8-byte values per round (EdgeFlags 42 -> 31 us at
// C3; 4 or 8 per lane were slower).
#ifndef FVV_SCAN_LB
#define FVV_SCAN_LB 2
#endif
#ifndef FVV_SCAN_LB2
#define FVV_SCAN_LB2 1
#endif

// 1: (value, flag) in 16 bytes; 2: two 16-byte halves (flag + 12 value bytes each)
template <typename T>
struct status_kind {
  static constexpr int value =
      sizeof(T) == 8 ? 1 : ((sizeof(T) % 4 == 0 && sizeof(T) <= 24) ? 2 : 0);
};

template <typename T, int kKind = status_kind<T>::value>
struct ScanStatus {
  T agg, incl;
  int flag;  // 0 none, 1 aggregate, 2 inclusive prefix
};
template <typename T>
struct __align__(16) ScanStatus<T, 1> {
  unsigned long long value;  // the aggregate (flag 1) or the inclusive prefix (flag 2)
  unsigned long long flag;
};
template <typename T>
struct __align__(16) ScanStatus<T, 2> {
  unsigned half[2][4];  // [h][0] flag, [h][1..3] value words 3h .. 3h+2
};

template <typename T>
__device__ __forceinline__ T from_bits(unsigned long long b) {
  static_assert(sizeof(T) == 8, "packed scan values are 8 bytes");
  T v;
  memcpy(&v, &b, 8);
  return v;
}
template <typename T>
__device__ __forceinline__ unsigned long long to_bits(const T &v) {
  unsigned long long b;
  memcpy(&b, &v, 8);
  return b;
}

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
__device__ __forceinline__ void scan_publish(ScanStatus<T, 0> *st, const T &agg, const T &incl,
                                             int flag) {
  volatile ScanStatus<T, 0> *v = st;
  if (flag == 1) {
    st->agg = agg;
  } else {
    st->incl = incl;
  }
  __threadfence();
  v->flag = flag;
}
template <typename T>
__device__ __forceinline__ void scan_publish(ScanStatus<T, 1> *st, const T &agg, const T &incl,
                                             int flag) {
  const unsigned long long v = to_bits(flag == 1 ? agg : incl), f = (unsigned long long)flag;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(st), "l"(v), "l"(f) : "memory");
}
template <typename T>
__device__ __forceinline__ void scan_publish(ScanStatus<T, 2> *st, const T &agg, const T &incl,
                                             int flag) {
  unsigned w[6] = {0u, 0u, 0u, 0u, 0u, 0u};
  memcpy(w, flag == 1 ? &agg : &incl, sizeof(T));
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(&st->half[h][0]),
                 "r"((unsigned)flag), "r"(w[3 * h]), "r"(w[3 * h + 1]), "r"(w[3 * h + 2])
                 : "memory");
}

// K statuses once published: flags (1 or 2) and the matching values (q < 0:
// before tile 0, an inclusive prefix of zero). Unpacked: all flags first,
// one fence, then the values.
template <typename T, int K>
__device__ __forceinline__ void scan_wait(const ScanStatus<T, 0> *status, const int64_t *q,
                                          int *fl, T *val) {
#pragma unroll
  for (int r = 0; r < K; ++r) {
    fl[r] = 2;
    if (q[r] >= 0) {
      volatile const ScanStatus<T, 0> *sq = status + q[r];
      while ((fl[r] = sq->flag) == 0) {
      }
    }
  }
  __threadfence();
#pragma unroll
  for (int r = 0; r < K; ++r)
    val[r] = q[r] < 0 ? T(0)
                      : (fl[r] == 2 ? ldcg_value(&status[q[r]].incl) : ldcg_value(&status[q[r]].agg));
}
template <typename T, int K>
__device__ __forceinline__ void scan_wait(const ScanStatus<T, 1> *status, const int64_t *q,
                                          int *fl, T *val) {
#pragma unroll
  for (int r = 0; r < K; ++r) {
    unsigned long long v = 0, f = 2;
    if (q[r] >= 0) {
      do {
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                     : "=l"(v), "=l"(f) : "l"(status + q[r]) : "memory");
      } while (f == 0);
    }
    fl[r] = (int)f;
    val[r] = from_bits<T>(v);
  }
}
template <typename T, int K>
__device__ __forceinline__ void scan_wait(const ScanStatus<T, 2> *status, const int64_t *q,
                                          int *fl, T *val) {
#pragma unroll
  for (int r = 0; r < K; ++r) {
    unsigned a[4] = {2u, 0u, 0u, 0u}, b[4] = {2u, 0u, 0u, 0u};
    if (q[r] >= 0) {
      do {
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                     : "l"(&status[q[r]].half[0][0]) : "memory");
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                     : "l"(&status[q[r]].half[1][0]) : "memory");
      } while (a[0] == 0u || a[0] != b[0]);
    }
    fl[r] = (int)a[0];
    const unsigned w[6] = {a[1], a[2], a[3], b[1], b[2], b[3]};
    memcpy(&val[r], w, sizeof(T));
  }
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
    constexpr int kLookBack = status_kind<T>::value == 1 ? FVV_SCAN_LB
                              : (status_kind<T>::value == 2 ? FVV_SCAN_LB2 : 1);
    if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 x kLookBack tiles at a time
      const int lane = threadIdx.x;
      T prefix = T(0);
      if (c == 0) {
        if (lane == 0) scan_publish(status + c, agg, agg, 2);
      } else {
        if (lane == 0) scan_publish(status + c, agg, agg, 1);
        for (int64_t q0 = c - 1;; q0 -= 32 * kLookBack) {
          // lane's tiles q0 - kLookBack lane - r (r = 0 .. kLookBack-1: farther back);
          // its part stops at its nearest inclusive tile
          T val[kLookBack];
          int fl[kLookBack];
          int64_t q[kLookBack];
#pragma unroll
          for (int r = 0; r < kLookBack; ++r) q[r] = q0 - (int64_t)kLookBack * lane - r;
          scan_wait<T, kLookBack>(status, q, fl, val);
          T part = T(0);
          bool has = false;
#pragma unroll
          for (int r = 0; r < kLookBack; ++r) {
            if (!has) part = part + val[r];
            has = has || fl[r] == 2;
          }
          const unsigned inc = __ballot_sync(0xffffffffu, has);
          const int first = inc ? __ffs(inc) - 1 : 32;  // lane holding the nearest inclusive tile
          if (lane > first) part = T(0);
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
                         void *ws, T *total, cudaStream_t st, bool zeroed = false) {
  const size_t sbytes = onepass_status_bytes<T>(n_max);
  if (!zeroed) fill_async(ws, 0, sbytes + 64, st);  // (zeroed: the caller cleared ws)
  launch_k(onepass_scan_kernel<F, T>, kScanGrid, kScanThreads, 0, st, f, n_dev, n_host, (ScanStatus<T> *)ws, (unsigned long long *)((char *)ws + sbytes),
      total);
  note_launches(1);
}

}  // namespace fvv
