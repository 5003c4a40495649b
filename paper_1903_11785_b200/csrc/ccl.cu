// B-2: 26-connected component labelling, noise filter support
// (hull.py:122-269).
//
// Works on the compacted set of ON voxels instead of the whole grid (the
// coarse stage grid is ~0.6% ON): an ordered popcount scan over the
// occupancy words gives every ON voxel its rank r (ranks ascend with the
// linear index), so a union-find forest over ranks keeps the reference's
// canonical numbering:
//   1. rank scan      : word_prefix[w], on_list[r] = l, parent[r] = r
//   2. union          : runs of ON voxels along i are linked to their first
//                       voxel; each run unites with the runs among its 13
//                       lexicographically negative 26-neighbours
//                       (hull.py:124-133); roots are linked by atomicMin, so
//                       every root ends as its component's minimum rank =
//                       minimum linear index
//   3. root scan      : label(root) = 1 + #roots before it — ascending
//                       minimum linear index, as hull.py:195-197 numbers them
//                       (and the component's stats record initialised)
//   4. stats          : each voxel's root by find, per-label count and
//                       inclusive bbox with warp-aggregated integer atomics
//                       (hull.py:201-214); the last block out writes the
//                       component table
// Integer-only and order independent; results are bit-identical to the
// reference for every launch configuration (its block_dims independence,
// tests/test_hull.py:159-168, holds trivially).
#include <cooperative_groups.h>
#include <cstring>

#include "scan.cuh"

namespace fvv {

struct CclWs {
  int64_t *counts;     // [0] n_on, [1] ncomp
  int64_t *sums;       // scan chunk sums
  int32_t *word_prefix;
  int32_t *on_list;
  int32_t *parent;
  int32_t *rank_label;
  int32_t *stats;      // [ncomp][8]: count, min ijk, max ijk, pad
  int64_t words, nvox, comp_cap;
};

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

constexpr int kMaxFusedGrid = 4096;
#ifndef FVV_CCL_BPS
#define FVV_CCL_BPS 2  // blocks per SM of the cooperative CCL grid
#endif  // blocks of ccl_fused_kernel (sums capacity)

// Most components a 26-connected grid can hold: one per 2x2x2 block.
static int64_t max_components(const int64_t *dims) {
  return ((dims[0] + 1) / 2) * ((dims[1] + 1) / 2) * ((dims[2] + 1) / 2);
}

static CclWs ccl_layout(void *base, const int64_t *dims) {
  CclWs w;
  char *p = (char *)base;
  const int64_t nvox = dims[0] * dims[1] * dims[2];
  w.nvox = nvox;
  w.words = (nvox + 31) / 32;
  w.comp_cap = max_components(dims);
  w.counts = (int64_t *)p;  // (first: the frame executor reads n_on / ncomp here in place)
  p += align256(4 * sizeof(int64_t));
  w.sums = (int64_t *)p;  // scan statuses, or the fused kernel's 2 x grid block sums
  const size_t scan_ws = onepass_bytes<int64_t>(nvox > w.words ? nvox : w.words);
  const size_t fused_ws = 2 * sizeof(int64_t) * kMaxFusedGrid;
  p += align256(scan_ws > fused_ws ? scan_ws : fused_ws);
  w.word_prefix = (int32_t *)p;
  p += align256(sizeof(int32_t) * w.words);
  w.on_list = (int32_t *)p;
  p += align256(sizeof(int32_t) * nvox);
  w.parent = (int32_t *)p;
  p += align256(sizeof(int32_t) * nvox);
  w.rank_label = (int32_t *)p;
  p += align256(sizeof(int32_t) * nvox);
  w.stats = (int32_t *)p;
  p += align256(sizeof(int32_t) * 8 * w.comp_cap);
  return w;
}

static size_t ccl_bytes(const int64_t *dims) {
  CclWs w = ccl_layout(nullptr, dims);
  return (size_t)((char *)w.stats - (char *)nullptr) + align256(sizeof(int32_t) * 8 * w.comp_cap);
}

// -- 1. rank scan over occupancy words --------------------------------------
struct WordRank {
  const uint32_t *occ;
  int32_t *word_prefix, *on_list, *parent;
  int64_t words, nvox;
  __device__ uint32_t word(int64_t w) const {
    uint32_t v = occ[w];
    if (w == words - 1 && (nvox & 31)) v &= (1u << (nvox & 31)) - 1u;
    return v;
  }
  typedef uint32_t Item;
  __device__ uint32_t load(int64_t w) const { return word(w); }
  __device__ int64_t value(uint32_t v) const { return __popc(v); }
  __device__ void emit(int64_t w, int64_t prefix, uint32_t v) const {
    word_prefix[w] = (int32_t)prefix;
    int32_t r = (int32_t)prefix;
    while (v) {
      int b = __ffs(v) - 1;
      v &= v - 1;
      on_list[r] = (int32_t)(w * 32 + b);
      parent[r] = r;
      ++r;
    }
  }
};

__device__ __forceinline__ int32_t uf_find(const int32_t *parent, int32_t x) {
  int32_t p = __ldcg(parent + x);
  while (p != x) {
    x = p;
    p = __ldcg(parent + x);
  }
  return x;
}

// find with path halving: every visited node is re-pointed at its
// grandparent. Plain stores are safe: they only ever replace a parent by one
// of its ancestors (smaller index), never touch a root, and the atomicMin
// linking in uf_unite re-checks roots, so connectivity and the min-root
// invariant are preserved (the forest only gets shallower).
__device__ __forceinline__ int32_t uf_find_halving(int32_t *parent, int32_t x) {
  int32_t p = __ldcg(parent + x);
  while (p != x) {
    const int32_t g = __ldcg(parent + p);
    if (g != p) __stcg(parent + x, g);
    x = p;
    p = g;
  }
  return x;
}

// Link the two trees; the smaller root wins (hull.py:146-153 links likewise).
__device__ __forceinline__ void uf_unite(int32_t *parent, int32_t a, int32_t b) {
  bool done;
  do {
    a = uf_find_halving(parent, a);
    b = uf_find_halving(parent, b);
    if (a < b) {
      int32_t old = atomicMin(parent + b, a);
      done = (old == b);
      b = old;
    } else if (b < a) {
      int32_t old = atomicMin(parent + a, b);
      done = (old == a);
      a = old;
    } else {
      done = true;
    }
  } while (!done);
}

__device__ __forceinline__ bool occ_bit(const uint32_t *occ, int64_t l) {
  return (__ldg(occ + (l >> 5)) >> (l & 31)) & 1u;
}

__device__ __forceinline__ int32_t rank_of(const uint32_t *occ, const int32_t *word_prefix,
                                           int64_t l) {
  uint32_t w = __ldg(occ + (l >> 5));
  return word_prefix[l >> 5] + __popc(w & ((1u << (l & 31)) - 1u));
}

// -- 2. union over runs ---------------------------------------------------------
// ON voxels come in runs along i (consecutive linear indices, so consecutive
// ranks). A run needs no union inside: every voxel points at the run's first
// rank. The 13 lexicographically negative 26-neighbours (hull.py:124-133) of
// a run's voxels are its own row's i - 1 (inside the run) and, in the four
// rows (dj, dk) = (-1, 0), (-1, -1), (0, -1), (1, -1), the voxels with
// i in [i0 - 1, i1 + 1]; the run is united with every run meeting that range,
// once per run instead of once per (voxel, offset).

// first voxel of the run holding ON position p (row positions [row0, p])
__device__ __forceinline__ int64_t run_first(const uint32_t *occ, int64_t row0, int64_t p) {
  int64_t q = p;
  while (q > row0) {
    const int64_t b = q - 1, wbase = b & ~31ll;
    const int sh = (int)(b & 31);
    uint32_t off = ~__ldg(occ + (b >> 5)) & (sh == 31 ? 0xffffffffu : ((2u << sh) - 1u));
    if (row0 > wbase) off &= 0xffffffffu << (row0 - wbase);
    if (off) return wbase + (31 - __clz(off)) + 1;  // one past the nearest OFF bit
    if (wbase <= row0) return row0;
    q = wbase;
  }
  return row0;
}

// last voxel of the run holding ON position p (row positions [p, row1))
__device__ __forceinline__ int64_t run_last(const uint32_t *occ, int64_t row1, int64_t p) {
  int64_t b = p + 1;
  while (b < row1) {
    const int64_t wbase = b & ~31ll;
    const uint32_t off = ~__ldg(occ + (b >> 5)) & (0xffffffffu << (b & 31));
    if (off) {
      const int64_t z = wbase + __ffs(off) - 1;
      return (z < row1 ? z : row1) - 1;
    }
    b = wbase + 32;
  }
  return row1 - 1;
}

// first ON position in [p, pe], or -1
__device__ __forceinline__ int64_t next_on(const uint32_t *occ, int64_t p, int64_t pe) {
  while (p <= pe) {
    const int64_t wbase = p & ~31ll;
    const uint32_t on = __ldg(occ + (p >> 5)) & (0xffffffffu << (p & 31));
    if (on) {
      const int64_t z = wbase + __ffs(on) - 1;
      return z <= pe ? z : -1;
    }
    p = wbase + 32;
  }
  return -1;
}

__global__ void ccl_union_kernel(const uint32_t *__restrict__ occ, CclWs w, int64_t nx, int64_t ny,
                                 int64_t nz) {
  pdl_wait();
  // four threads per ON voxel: the run's first voxel unites with the runs of
  // one neighbour row each; the others link to their run's first voxel.
  // 32-bit index arithmetic (nvox < 2^31, fvv_ccl26)
  const int64_t n_on = __ldcg(w.counts);
  const uint32_t ux = (uint32_t)nx, uy = (uint32_t)ny;
  const int djs[4] = {-1, -1, 0, 1}, dks[4] = {0, -1, -1, -1};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 4 * n_on;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e >> 2;
    const int n = (int)(e & 3);
    const uint32_t l = (uint32_t)w.on_list[r];
    const uint32_t q = l / ux, k = q / uy;
    const uint32_t i = l - q * ux, j = q - k * uy;
    const int64_t row0 = (int64_t)l - i;
    const int64_t first = run_first(occ, row0, l);
    if (first != (int64_t)l) {  // inside a run: link to its first voxel (consecutive ranks)
      if (n == 0) w.parent[r] = (int32_t)(r - ((int64_t)l - first));
      continue;
    }
    const int64_t jj = (int64_t)j + djs[n], kk = (int64_t)k + dks[n];
    if (jj < 0 || jj >= ny || kk < 0) continue;
    const int64_t last = run_last(occ, row0 + nx, l);
    const int64_t a = i > 0 ? i - 1 : 0, i1 = last - row0, b = i1 + 1 < nx ? i1 + 1 : nx - 1;
    const int64_t nrow = nx * (jj + ny * kk);
    int64_t p = nrow + a;
    const int64_t pe = nrow + b;
    while (p <= pe) {
      const int64_t s = next_on(occ, p, pe);
      if (s < 0) break;
      const int64_t sf = run_first(occ, nrow, s);
      uf_unite(w.parent, (int32_t)r, rank_of(occ, w.word_prefix, sf));
      p = run_last(occ, nrow + nx, s) + 2;  // (the bit after a run is OFF)
    }
  }
}

// -- 4. label roots in rank order --------------------------------------------
// (a root's emit also initialises its component's stats record)
struct RootLabel {
  const int32_t *parent;
  int32_t *rank_label;
  int32_t *stats;
  typedef int Item;
  __device__ int load(int64_t r) const { return parent[r] == (int32_t)r; }
  __device__ int64_t value(int v) const { return v; }
  __device__ void emit(int64_t r, int64_t prefix, int v) const {
    if (!v) return;
    rank_label[r] = (int32_t)(prefix + 1);
    int32_t *s = stats + 8 * prefix;
    s[0] = 0;
    s[1] = s[2] = s[3] = 0x7fffffff;
    s[4] = s[5] = s[6] = -1;
    s[7] = 0;
  }
};

// -- 5. per-rank label + component count/bbox ----------------------------------
__device__ __forceinline__ void export_components(const CclWs &w, fvv_component *out, int64_t cap,
                                                  int64_t tid, int64_t stride) {
  const int64_t ncomp = __ldcg(w.counts + 1);
  const int64_t n = ncomp < cap ? ncomp : cap;
  for (int64_t c = tid; c < n; c += stride) {
    const int32_t *s = w.stats + 8 * c;
    fvv_component rec;
    rec.id = c + 1;
    rec.voxel_count = __ldcg(s);
    for (int d = 0; d < 3; ++d) {
      rec.bbox_min[d] = __ldcg(s + 1 + d);
      rec.bbox_max[d] = __ldcg(s + 4 + d);
    }
    out[c] = rec;
  }
}

// Labels and component stats of every ON voxel; the root comes from the
// union-find forest directly (no separate flatten pass). With `out`, the
// last block to finish writes the component table (counts[2] counts the
// finished blocks).
__global__ void ccl_stats_kernel(CclWs w, int64_t nx, int64_t ny, fvv_component *out,
                                 int64_t cap) {
  pdl_wait();
  const int64_t n_on = __ldcg(w.counts);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; r0 < n_on;
       r0 += stride) {
    const int64_t r = r0 + lane;
    const bool act = r < n_on;
    int32_t lab = 0;
    unsigned i = 0, j = 0, k = 0;
    if (act) {
      const int32_t root = uf_find(w.parent, (int32_t)r);
      lab = __ldcg(w.rank_label + root);
      if (root != (int32_t)r) w.rank_label[r] = lab;
      const uint32_t l = (uint32_t)w.on_list[r];
      const uint32_t q = l / (uint32_t)nx;
      k = q / (uint32_t)ny;
      i = l - q * (uint32_t)nx;
      j = q - k * (uint32_t)ny;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, act ? lab : -1);
    const unsigned mn_i = __reduce_min_sync(grp, i), mx_i = __reduce_max_sync(grp, i);
    const unsigned mn_j = __reduce_min_sync(grp, j), mx_j = __reduce_max_sync(grp, j);
    const unsigned mn_k = __reduce_min_sync(grp, k), mx_k = __reduce_max_sync(grp, k);
    if (act && lane == __ffs(grp) - 1) {
      int32_t *s = w.stats + 8 * (int64_t)(lab - 1);
      atomicAdd(s + 0, __popc(grp));
      atomicMin(s + 1, (int32_t)mn_i);
      atomicMin(s + 2, (int32_t)mn_j);
      atomicMin(s + 3, (int32_t)mn_k);
      atomicMax(s + 4, (int32_t)mx_i);
      atomicMax(s + 5, (int32_t)mx_j);
      atomicMax(s + 6, (int32_t)mx_k);
    }
  }
  if (out == nullptr) return;
  __shared__ bool last;
  __threadfence();  // this block's stats atomics before its completion count
  __syncthreads();
  if (threadIdx.x == 0)
    last = atomicAdd((unsigned long long *)(w.counts + 2), 1ull) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    export_components(w, out, cap, threadIdx.x, blockDim.x);
  }
}

__global__ void ccl_export_kernel(CclWs w, fvv_component *out, int64_t cap) {
  pdl_wait();
  export_components(w, out, cap, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
}

__global__ void ccl_expand_kernel(CclWs w, int32_t *labels) {
  pdl_wait();
  const int64_t n_on = __ldcg(w.counts);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_on;
       r += (int64_t)gridDim.x * blockDim.x)
    labels[w.on_list[r]] = w.rank_label[r];
}

// hull.py:257-269: keep[label] selects survivors; ids are not renumbered.
__global__ void ccl_filter_kernel(CclWs w, const uint8_t *__restrict__ keep, int32_t *labels,
                                  uint32_t *occ_out, int64_t *kept) {
  pdl_wait();
  const int64_t n_on = __ldcg(w.counts);
  int64_t mine = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_on;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t lab = w.rank_label[r];
    if (!keep[lab]) continue;
    const int64_t l = w.on_list[r];
    if (labels) labels[l] = lab;
    if (occ_out) atomicOr(occ_out + (l >> 5), 1u << (l & 31));
    ++mine;
  }
  if (kept && mine) atomicAdd((unsigned long long *)kept, (unsigned long long)mine);
}

// Same filter for a caller-supplied dense label array (no CCL workspace).
__global__ void dense_filter_kernel(const int32_t *__restrict__ in, int64_t nvox, int64_t nkeep,
                                    const uint8_t *__restrict__ keep, int32_t *out,
                                    uint32_t *occ_out, int64_t *kept) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  int64_t mine = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t l0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; l0 < nvox;
       l0 += stride) {
    const int64_t l = l0 + lane;
    int32_t lab = l < nvox ? in[l] : 0;
    const bool on = lab > 0 && lab < nkeep && keep[lab];
    if (l < nvox && out) out[l] = on ? lab : 0;
    const uint32_t bits = __ballot_sync(0xffffffffu, on);
    if (lane == 0) {
      if (occ_out) occ_out[l0 >> 5] = bits;
      mine += __popc(bits);
    }
  }
  if (kept && mine) atomicAdd((unsigned long long *)kept, (unsigned long long)mine);
}

constexpr int kCclGrid = 148 * 8;

// ---- all of B-2 in one cooperative launch -----------------------------------
// The separate launches above are latency chains over a few thousand ON
// voxels (C3: ~12k in a 10M-voxel stage grid): seven launches whose ramps
// and drains dominate. Here one co-resident grid runs the same steps with
// grid-wide barriers in between, in the same order and with the same
// integer operations, so the numbering is unchanged: rank scan (block
// ranges of words, block sums, grid barrier, block prefixes), union over
// runs, root scan over ranks, per-component stats, component table. Values
// written in one step are read in later ones through L2 (ld.cg), never
// through a possibly stale L1 line.
constexpr int kFusedThreads = 256;

// exclusive prefix of this block's `mine` over blocks 0 .. blockIdx.x - 1,
// from the per-block sums written before the last grid barrier
__device__ __forceinline__ int64_t block_offset(const int64_t *sums, int64_t *total) {
  __shared__ int64_t part[kFusedThreads / 32];
  int64_t acc = 0, all = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const int64_t v = __ldcg(sums + b);
    if (b < (int)blockIdx.x) acc += v;
    all += v;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    all += __shfl_xor_sync(0xffffffffu, all, o);
  }
  __shared__ int64_t part_all[kFusedThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    part[threadIdx.x >> 5] = acc;
    part_all[threadIdx.x >> 5] = all;
  }
  __syncthreads();
  int64_t off = 0, tot = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
    off += part[k];
    tot += part_all[k];
  }
  __syncthreads();
  *total = tot;
  return off;
}

__global__ void __launch_bounds__(kFusedThreads)
    ccl_fused_kernel(const uint32_t *__restrict__ occ, CclWs w, int64_t nx, int64_t ny, int64_t nz,
                     fvv_component *out, int64_t cap) {
  namespace cg = cooperative_groups;
  pdl_wait();
  cg::grid_group grid = cg::this_grid();
  using Scan = cub::BlockScan<int, kFusedThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t s_run;
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int64_t gtid = b * (int64_t)blockDim.x + threadIdx.x, gstride = (int64_t)G * blockDim.x;
  const WordRank wr{occ, w.word_prefix, w.on_list, w.parent, w.words, w.nvox};

  // 1. ranks: block b owns words [w0, w1)
  const int64_t w0 = w.words * b / G, w1 = w.words * (b + 1) / G;
  {
    int64_t mine = 0;
    for (int64_t q = w0 + threadIdx.x; q < w1; q += blockDim.x) mine += __popc(wr.word(q));
    mine = __reduce_add_sync(0xffffffffu, (unsigned)mine);
    __shared__ int64_t bsum;
    if (threadIdx.x == 0) bsum = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)&bsum, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0) w.sums[b] = bsum;
  }
  grid.sync();
  {
    int64_t n_on;
    const int64_t off = block_offset(w.sums, &n_on);
    if (b == 0 && threadIdx.x == 0) w.counts[0] = n_on;
    if (threadIdx.x == 0) s_run = off;
    __syncthreads();
    for (int64_t c0 = w0; c0 < w1; c0 += blockDim.x) {
      const int64_t q = c0 + threadIdx.x;
      const uint32_t v = q < w1 ? wr.word(q) : 0u;
      int ex, agg;
      Scan(tmp).ExclusiveSum((int)__popc(v), ex, agg);
      if (q < w1) wr.emit(q, s_run + ex, v);
      __syncthreads();
      if (threadIdx.x == 0) s_run += agg;
      __syncthreads();
    }
  }
  grid.sync();
  const int64_t n_on = __ldcg(w.counts);

  // 2. union over runs (ccl_union_kernel's step, values through L2)
  {
    const uint32_t ux = (uint32_t)nx, uy = (uint32_t)ny;
    const int djs[4] = {-1, -1, 0, 1}, dks[4] = {0, -1, -1, -1};
    for (int64_t e = gtid; e < 4 * n_on; e += gstride) {
      const int64_t r = e >> 2;
      const int n = (int)(e & 3);
      const uint32_t l = (uint32_t)__ldcg(w.on_list + r);
      const uint32_t q = l / ux, k = q / uy;
      const uint32_t i = l - q * ux, j = q - k * uy;
      const int64_t row0 = (int64_t)l - i;
      const int64_t first = run_first(occ, row0, l);
      if (first != (int64_t)l) {
        if (n == 0) __stcg(w.parent + r, (int32_t)(r - ((int64_t)l - first)));
        continue;
      }
      const int64_t jj = (int64_t)j + djs[n], kk = (int64_t)k + dks[n];
      if (jj < 0 || jj >= ny || kk < 0) continue;
      const int64_t last = run_last(occ, row0 + nx, l);
      const int64_t a = i > 0 ? i - 1 : 0, i1 = last - row0, bb = i1 + 1 < nx ? i1 + 1 : nx - 1;
      const int64_t nrow = nx * (jj + ny * kk);
      int64_t p = nrow + a;
      const int64_t pe = nrow + bb;
      while (p <= pe) {
        const int64_t s = next_on(occ, p, pe);
        if (s < 0) break;
        const int64_t sf = run_first(occ, nrow, s);
        const uint32_t wv = __ldg(occ + (sf >> 5));
        const int32_t rs = __ldcg(w.word_prefix + (sf >> 5)) + __popc(wv & ((1u << (sf & 31)) - 1u));
        uf_unite(w.parent, (int32_t)r, rs);
        p = run_last(occ, nrow + nx, s) + 2;
      }
    }
  }
  grid.sync();

  // 3. root labels: block b owns ranks [r0, r1)
  const int64_t r0 = n_on * b / G, r1 = n_on * (b + 1) / G;
  {
    int64_t mine = 0;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) mine += __ldcg(w.parent + r) == (int32_t)r;
    mine = __reduce_add_sync(0xffffffffu, (unsigned)mine);
    __shared__ int64_t bsum2;
    if (threadIdx.x == 0) bsum2 = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)&bsum2, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0) w.sums[G + b] = bsum2;
  }
  grid.sync();
  {
    int64_t ncomp;
    const int64_t off = block_offset(w.sums + G, &ncomp);
    if (b == 0 && threadIdx.x == 0) w.counts[1] = ncomp;
    if (threadIdx.x == 0) s_run = off;
    __syncthreads();
    for (int64_t c0 = r0; c0 < r1; c0 += blockDim.x) {
      const int64_t r = c0 + threadIdx.x;
      const int root = r < r1 && __ldcg(w.parent + r) == (int32_t)r;
      int ex, agg;
      Scan(tmp).ExclusiveSum(root, ex, agg);
      if (root) {
        const int64_t lab = s_run + ex;
        w.rank_label[r] = (int32_t)(lab + 1);
        int32_t *st = w.stats + 8 * lab;
        st[0] = 0;
        st[1] = st[2] = st[3] = 0x7fffffff;
        st[4] = st[5] = st[6] = -1;
        st[7] = 0;
      }
      __syncthreads();
      if (threadIdx.x == 0) s_run += agg;
      __syncthreads();
    }
  }
  grid.sync();

  // 4. labels and component stats (ccl_stats_kernel's step)
  {
    const int lane = threadIdx.x & 31;
    for (int64_t q0 = gtid & ~31ll; q0 < n_on; q0 += gstride) {
      const int64_t r = q0 + lane;
      const bool act = r < n_on;
      int32_t lab = 0;
      unsigned i = 0, j = 0, k = 0;
      if (act) {
        const int32_t root = uf_find(w.parent, (int32_t)r);
        lab = __ldcg(w.rank_label + root);
        if (root != (int32_t)r) w.rank_label[r] = lab;
        const uint32_t l = (uint32_t)__ldcg(w.on_list + r);
        const uint32_t q = l / (uint32_t)nx;
        k = q / (uint32_t)ny;
        i = l - q * (uint32_t)nx;
        j = q - k * (uint32_t)ny;
      }
      const unsigned grp = __match_any_sync(0xffffffffu, act ? lab : -1);
      const unsigned mn_i = __reduce_min_sync(grp, i), mx_i = __reduce_max_sync(grp, i);
      const unsigned mn_j = __reduce_min_sync(grp, j), mx_j = __reduce_max_sync(grp, j);
      const unsigned mn_k = __reduce_min_sync(grp, k), mx_k = __reduce_max_sync(grp, k);
      if (act && lane == __ffs(grp) - 1) {
        int32_t *st = w.stats + 8 * (int64_t)(lab - 1);
        atomicAdd(st + 0, __popc(grp));
        atomicMin(st + 1, (int32_t)mn_i);
        atomicMin(st + 2, (int32_t)mn_j);
        atomicMin(st + 3, (int32_t)mn_k);
        atomicMax(st + 4, (int32_t)mx_i);
        atomicMax(st + 5, (int32_t)mx_j);
        atomicMax(st + 6, (int32_t)mx_k);
      }
    }
  }
  if (out == nullptr) return;
  grid.sync();
  export_components(w, out, cap, gtid, gstride);
}

// blocks of ccl_fused_kernel that are co-resident on every SM (cooperative launch)
static int ccl_fused_grid() {
  static const int g = [] {
    int nb = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, ccl_fused_kernel, kFusedThreads, 0) !=
            cudaSuccess || nb < 1)
      return 0;
    const int g = sms * (nb < FVV_CCL_BPS ? nb : FVV_CCL_BPS);
    return g < kMaxFusedGrid ? g : kMaxFusedGrid;
  }();
  return g;
}

static bool ccl_fused_enabled() {
  static const bool on = [] {
    const char *e = getenv("FVV_CCL_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace fvv

using namespace fvv;

extern "C" {

size_t fvv_ccl_workspace_bytes(const fvv_grid *grid) { return ccl_bytes(grid->dims); }

int fvv_ccl26(const uint32_t *occ_dev, const fvv_grid *grid, void *ws_dev, size_t ws_bytes,
              fvv_component *comps_dev, int64_t comp_cap, int64_t *counts_dev, void *stream) {
  const int64_t nx = grid->dims[0], ny = grid->dims[1], nz = grid->dims[2];
  const int64_t nvox = nx * ny * nz;
  if (nvox <= 0 || nvox >= (1ll << 31)) {
    set_error("fvv_ccl26: grid of %lld voxels (need 1 .. 2^31-1)", (long long)nvox);
    return FVV_E_ARG;
  }
  if (ws_bytes < ccl_bytes(grid->dims)) {
    set_error("fvv_ccl26: workspace %zu < %zu bytes", ws_bytes, ccl_bytes(grid->dims));
    return FVV_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  CclWs w = ccl_layout(ws_dev, grid->dims);
  const int fg = ccl_fused_enabled() ? ccl_fused_grid() : 0;
  if (fg > 0) {  // one cooperative launch (w.sums holds its 2 x grid block sums)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = fg;
    cfg.blockDim = kFusedThreads;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, ccl_fused_kernel, occ_dev, w, nx, ny, nz, comps_dev, comp_cap);
    note_launches(1);
    if (counts_dev) cudaMemcpyAsync(counts_dev, w.counts, 2 * sizeof(int64_t),
                                    cudaMemcpyDeviceToDevice, st);
    return cuda_check("fvv_ccl26");
  }
  fill_async(w.counts, 0, 4 * sizeof(int64_t), st);
  WordRank wr{occ_dev, w.word_prefix, w.on_list, w.parent, w.words, nvox};
  onepass_scan(wr, nullptr, w.words, w.words, (void *)w.sums, w.counts + 0, st);
  launch_k(ccl_union_kernel, kCclGrid, 256, 0, st, occ_dev, w, nx, ny, nz);
  RootLabel rl{w.parent, w.rank_label, w.stats};
  onepass_scan(rl, w.counts + 0, 0, nvox, (void *)w.sums, w.counts + 1, st);
  launch_k(ccl_stats_kernel, kCclGrid, 256, 0, st, w, nx, ny, comps_dev, comp_cap);
  note_launches(2);
  if (counts_dev) cudaMemcpyAsync(counts_dev, w.counts, 2 * sizeof(int64_t),
                                  cudaMemcpyDeviceToDevice, st);
  return cuda_check("fvv_ccl26");
}

int fvv_ccl_components(const fvv_grid *grid, const void *ws_dev, fvv_component *comps_dev,
                       int64_t comp_cap, void *stream) {
  const int64_t nvox = grid->dims[0] * grid->dims[1] * grid->dims[2];
  CclWs w = ccl_layout((void *)ws_dev, grid->dims);
  launch_k(ccl_export_kernel, kCclGrid, 256, 0, (cudaStream_t)stream, w, comps_dev, comp_cap);
  note_launches(1);
  return cuda_check("fvv_ccl_components");
}

int fvv_ccl_labels(const fvv_grid *grid, const void *ws_dev, int32_t *labels_dev, void *stream) {
  const int64_t nvox = grid->dims[0] * grid->dims[1] * grid->dims[2];
  CclWs w = ccl_layout((void *)ws_dev, grid->dims);
  cudaStream_t st = (cudaStream_t)stream;
  fill_async(labels_dev, 0, sizeof(int32_t) * nvox, st);
  launch_k(ccl_expand_kernel, kCclGrid, 256, 0, st, w, labels_dev);
  note_launches(1);
  return cuda_check("fvv_ccl_labels");
}

int fvv_filter_labels(const fvv_grid *grid, const void *ws_dev, const uint8_t *keep_dev,
                      int32_t *labels_dev, uint32_t *occ_dev, int64_t *kept_dev, void *stream) {
  const int64_t nvox = grid->dims[0] * grid->dims[1] * grid->dims[2];
  CclWs w = ccl_layout((void *)ws_dev, grid->dims);
  cudaStream_t st = (cudaStream_t)stream;
  if (labels_dev) fill_async(labels_dev, 0, sizeof(int32_t) * nvox, st);
  if (occ_dev) fill_async(occ_dev, 0, sizeof(uint32_t) * ((nvox + 31) / 32), st);
  if (kept_dev) fill_async(kept_dev, 0, sizeof(int64_t), st);
  launch_k(ccl_filter_kernel, kCclGrid, 256, 0, st, w, keep_dev, labels_dev, occ_dev, kept_dev);
  note_launches(1);
  return cuda_check("fvv_filter_labels");
}

int fvv_filter_dense(const int32_t *labels_in_dev, int64_t nvox, const uint8_t *keep_dev,
                     int64_t nkeep, int32_t *labels_dev, uint32_t *occ_dev, int64_t *kept_dev,
                     void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (kept_dev) fill_async(kept_dev, 0, sizeof(int64_t), st);
  launch_k(dense_filter_kernel, kCclGrid, 256, 0, st, labels_in_dev, nvox, nkeep, keep_dev, labels_dev,
                                                occ_dev, kept_dev);
  note_launches(1);
  return cuda_check("fvv_filter_dense");
}

}  // extern "C"
