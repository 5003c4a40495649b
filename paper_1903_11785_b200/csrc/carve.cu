// B-1 sparse carve / B-3 dense carve (hull.py:78-119, hull.py:287-302).
//
// Work is tiled: 16^3 / 8^3 voxel tiles are first classified per camera
// from certified bounds at their corners (all-background culls the tile,
// all-foreground passes the camera for every voxel), then the surviving
// tiles' voxels are tested against the remaining "mixed" cameras, one thread
// per voxel. A warp covers 32 voxels of one tile: rows of kT consecutive i
// (kT = tile edge) in 32 / kT consecutive j; a warp ballot packs the ON flags
// and one lane per row ORs the row's bits into the occupancy words (one or
// two 32-bit atomics per row instead of one per ON voxel). Every grid of the
// batch (the coarse stage grid, or all ROI grids) is carved by one launch:
// blocks are assigned to grids by a prefix table in the parameter block.
//
// Exactness: each (voxel, camera) test is decided either by a certified
// FP32 evaluation (below) or by the reference's float64 chain
// (fvv_common.cuh project_exact); both give the reference's pixel. A voxel
// stops at the first camera that sees it on background: it is OFF whatever
// the remaining cameras say (hull.py:91 ANDs them), so the early exit
// cannot change the result.
#include <algorithm>
#include <cstring>

#include "affine.cuh"
#include "fvv_common.cuh"

namespace fvv {

constexpr int kCarveThreads = 256;
#ifndef FVV_CARVE_MINB
#define FVV_CARVE_MINB 6  // resident 256-thread blocks per SM the tile kernels are built for
#endif
constexpr int kCarveWordsPerBlock = 128;  // 4096 voxels per block
#ifndef FVV_AMB_CAP
#define FVV_AMB_CAP (1 << 22)  // 64 MB: large grids x many cameras (C5 1024^3) fill 1M
#endif
constexpr int64_t kAmbCap = FVV_AMB_CAP;  // deferred-voxel queue entries
constexpr int64_t kTileCap = 1 << 19;    // split mode: surviving-tile records
// split mode: the octant kernel's grid (resident blocks taking octants)
// octant kernel blocks of kThreads threads (resident threads per SM as for
// FVV_CARVE_MINB 256-thread blocks): 128 for ROI batches, where a block's
// barriers (octant classification, the slowest warp's voxels) idle fewer
// warps (B-3 146 -> 132 us at C3), 256 for the stage grid (B-1: 44 vs 48 us)
template <int kThreads>
constexpr int oct_min_blocks() { return FVV_CARVE_MINB * 256 / kThreads; }

struct CarveParams {
  int ncam, min_views;
  const uint32_t *sil;
  uint32_t *occ;
  int64_t *count;
  unsigned long long *amb;  // [0] = queued voxels, then {key, camera mask} entries
  int64_t amb_cap;
  const struct CamAffine *affine;  // [ngrid][ncam] (carve_affine_kernel)
  unsigned long long *tile_stats;  // culled tiles, sum of fg cameras, sum of mixed cameras;
                                   // culled octants, carved octants, their mixed cameras
  int tile_log2;                   // tile edge 1 << tile_log2 voxels
  struct TileWork *tiles;          // split mode: surviving tiles (carve_voxels_kernel)
  unsigned long long *ntiles;      //   and their count
  int64_t tile_cap;
  uint32_t tiles_x[FVV_MAX_GRIDS], tiles_y[FVV_MAX_GRIDS];
  // 8x8-pixel cell maps per camera (carve_cells_kernel): bit = some / every
  // pixel of the cell is foreground; rows of cell_words[c] words
  uint32_t *cell_any, *cell_all;
  int64_t cell_off[FVV_MAX_CAMS], cell_total;
  int32_t cell_words[FVV_MAX_CAMS];
  int k1;                    // cameras order[0 .. k1) are tested in phase 1
  int order[FVV_MAX_CAMS];   // camera test order (a permutation of 0 .. ncam-1)
  int64_t sil_off[FVV_MAX_CAMS];
  int32_t sil_stride[FVV_MAX_CAMS];
  fvv_camera cams[FVV_MAX_CAMS];
  const CarveGrids *gt;  // the batch's grids (device memory)
};

// (i, j, k) of linear voxel index l (F order), 32-bit when the grid allows.
__device__ __forceinline__ void voxel_ijk(int64_t l, int64_t nx, int64_t ny, bool small,
                                          int64_t &i, int64_t &j, int64_t &k) {
  if (small) {
    const uint32_t l32 = (uint32_t)l, nx32 = (uint32_t)nx, ny32 = (uint32_t)ny;
    const uint32_t q = l32 / nx32;
    i = l32 - q * nx32;
    j = q % ny32;
    k = q / ny32;
  } else {
    i = l % nx;
    j = (l / nx) % ny;
    k = l / (nx * ny);
  }
}

// The reference's float64 chain for one voxel (hull.py:83-91), over the
// cameras in cam_mask (bit c); seen / the result carry the decided rest.
// `cams` may be a shared-memory copy (lanes index different cameras).
__device__ __forceinline__ bool carve_exact(const CarveParams &p, const fvv_camera *cams,
                                            const fvv_grid &G, int64_t l,
                                            unsigned long long cam_mask, int seen) {
  const int64_t nx = G.dims[0], ny = G.dims[1];
  const int64_t nvox = nx * ny * G.dims[2];
  int64_t i, j, k;
  voxel_ijk(l, nx, ny, nvox <= 0xffffffffll, i, j, k);
  double x, y, z;
  voxel_center(G, i, j, k, x, y, z);
  const bool gemv = (nvox % kCarveChunk == 1) && l == nvox - 1;  // 1-row BLAS chunk
  while (cam_mask) {
    const int c = __ffsll((long long)cam_mask) - 1;
    cam_mask &= cam_mask - 1;
    double u, v, zc;
    if (!project_exact(cams[c], x, y, z, true, gemv, u, v, zc)) continue;
    ++seen;
    if (!sil_bit(p.sil + p.sil_off[c], sil_stride_words(cams[c].width), (int)rint(u),
                 (int)rint(v)))
      return false;
  }
  return seen >= p.min_views;
}

// A voxel no FP32 camera rejected: ON/OFF from the counts, or, when some
// tests were undecided (amb_mask, bit c), the float64 chain for those
// cameras (deferred to carve_exact_kernel; queue entries are
// {grid << 40 | seen << 47 | voxel, camera mask}).
__device__ __forceinline__ bool settle(const CarveParams &p, const fvv_grid &G, int g, int64_t l,
                                       int seen, unsigned long long amb_mask) {
  if (!amb_mask) return seen >= p.min_views;
  const unsigned long long slot = atomicAdd(p.amb, 1ull);
  if ((int64_t)slot < p.amb_cap) {
    p.amb[1 + 2 * slot] = ((unsigned long long)g << 40) | ((unsigned long long)seen << 47) |
                          (unsigned long long)l;
    p.amb[2 + 2 * slot] = amb_mask;
    return false;  // its bit is set by carve_exact_kernel
  }
  return carve_exact(p, p.cams, G, l, amb_mask, seen);
}

// ---- tile culling ---------------------------------------------------------
// A block carves one tile of T^3 voxels (T = 8, or 16 for large grids). For each camera it first bounds,
// in FP32 with the same certified error terms, the pixels the tile's voxel
// centres can round to: u = U/Z is linear-fractional, so over the tile (a
// box of voxel centres, Z > 0) its extrema are at the 8 corner centres. If
// that pixel rectangle lies inside the image, every voxel of the tile is in
// the camera's frustum, and then
//   - all rectangle pixels background -> every voxel is OFF (hull.py:91),
//   - all foreground -> the camera passes every voxel (one more view each),
//   - otherwise the camera is tested per voxel.
// Per-voxel work is thus confined to the cameras whose silhouette boundary
// crosses the tile; empty space and hull interiors cost a few word loads.
constexpr int kRectMaxPx = 4096;        // larger rectangles: test per voxel
enum : int { kTileBg = 0, kTileFg = 1, kTileMixed = 2 };

__device__ __forceinline__ void corner_bound(const CamAffine &a, float fi, float fj, float fk,
                                             bool &zok, float &u0, float &u1, float &v0,
                                             float &v1, float &rz_out) {
  const float Z = fmaf(fk, a.z[3], fmaf(fj, a.z[2], fmaf(fi, a.z[1], a.z[0])));
  const float U = fmaf(fk, a.u[3], fmaf(fj, a.u[2], fmaf(fi, a.u[1], a.u[0])));
  const float V = fmaf(fk, a.v[3], fmaf(fj, a.v[2], fmaf(fi, a.v[1], a.v[0])));
  zok = Z >= a.ez;  // Z > 0 for certain
  const float rz = recip(zok ? Z : 1.0f);
  rz_out = rz;
  const float u = U * rz, v = V * rz;
  const float k = fmaf(a.A, rz, 3.75f * kEps);
  // + 1e-3 covers the rounding of these few float operations
  const float eu = fmaf(fabsf(u) + 1.0f, k, fmaf(a.bu, rz, 9.5367432e-7f)) + 1e-3f;
  const float ev = fmaf(fabsf(v) + 1.0f, k, fmaf(a.bv, rz, 9.5367432e-7f)) + 1e-3f;
  u0 = u - eu;
  u1 = u + eu;
  v0 = v - ev;
  v1 = v + ev;
}

// Eight lanes (one group of a warp; g8 = lane & 7) classify camera c for
// the tile [i0, i1] x [j0, j1] x [k0, k1]; every lane of the warp calls this
// (c < 0: idle group) and gets its own group's result.
// Also returns (box, eu, ev) the per-voxel rounding bounds of classify32_box
// over the tile, box = false when they do not hold (some corner's Z not
// certainly positive): the voxels then take classify32.
__device__ int tile_camera(const CarveParams &p, const CamAffine *aff, int c, int i0, int i1,
                           int j0, int j1, int k0, int k1, int lane, bool &box, float &beu,
                           float &bev) {
  const int g8 = lane & 7, grp = lane >> 3;
  float u0 = INFINITY, u1 = -INFINITY, v0 = INFINITY, v1 = -INFINITY, rz = 0.0f;
  bool zok = false;
  if (c >= 0)
    corner_bound(aff[c], (float)((g8 & 1) ? i1 : i0), (float)((g8 & 2) ? j1 : j0),
                 (float)((g8 & 4) ? k1 : k0), zok, u0, u1, v0, v1, rz);
  for (int o = 4; o >= 1; o >>= 1) {  // min/max over the group's 8 corners
    u0 = fminf(u0, __shfl_xor_sync(0xffffffffu, u0, o));
    u1 = fmaxf(u1, __shfl_xor_sync(0xffffffffu, u1, o));
    v0 = fminf(v0, __shfl_xor_sync(0xffffffffu, v0, o));
    v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, o));
    rz = fmaxf(rz, __shfl_xor_sync(0xffffffffu, rz, o));
  }
  const unsigned gmask = 0xffu << (8 * grp);
  zok = (__ballot_sync(0xffffffffu, zok) & gmask) == gmask;
  box = zok && c >= 0;
  beu = bev = 0.0f;
  if (box)  // (u0..u1 / v0..v1 include each corner's own bound: |u| <= max(|u0|, |u1|))
    box_bounds(aff[c], fmaxf(fabsf(u0), fabsf(u1)), fmaxf(fabsf(v0), fabsf(v1)), rz, beu, bev);
  bool query = c >= 0 && zok;
  // rint(x) lies in [floor(x - 0.5), ceil(x + 0.5)] for x in [u0, u1]
  const float xl = floorf(u0 - 0.5f), xh = ceilf(u1 + 0.5f);
  const float yl = floorf(v0 - 0.5f), yh = ceilf(v1 + 0.5f);
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
  if (query) {
    const CamAffine &a = aff[c];
    query = xl >= 0.0f && yl >= 0.0f && xh <= (float)(a.w - 1) && yh <= (float)(a.h - 1);
    if (query) {  // (false for NaN, or partly outside the image: per voxel)
      x0 = (int)xl;
      x1 = (int)xh;
      y0 = (int)yl;
      y1 = (int)yh;
      query = (int64_t)(x1 - x0 + 1) * (y1 - y0 + 1) <= kRectMaxPx;
    }
  }
  bool any = false, all = true;
  if (query && y1 - y0 >= 16) {  // large rectangle: 8x8 cells covering it
    const int cx0 = x0 >> 3, cx1 = x1 >> 3, cy0 = y0 >> 3, cy1 = y1 >> 3;
    const uint32_t *ca = p.cell_any + p.cell_off[c], *cl = p.cell_all + p.cell_off[c];
    const int stride = p.cell_words[c];
    const int w0 = cx0 >> 5, w1 = cx1 >> 5;
    const uint32_t mlo = 0xffffffffu << (cx0 & 31), mhi = 0xffffffffu >> (31 - (cx1 & 31));
    for (int y = cy0 + g8; y <= cy1; y += 8) {
      for (int wq = w0; wq <= w1; ++wq) {
        const uint32_t m = (wq == w0 ? mlo : 0xffffffffu) & (wq == w1 ? mhi : 0xffffffffu);
        any |= (__ldg(ca + (int64_t)y * stride + wq) & m) != 0;
        all &= (__ldg(cl + (int64_t)y * stride + wq) & m) == m;
      }
    }
  } else if (query) {
    const uint32_t *plane = p.sil + aff[c].sil_off;
    const int stride = aff[c].sil_stride;
    const int w0 = x0 >> 5, w1 = x1 >> 5;
    const uint32_t mlo = 0xffffffffu << (x0 & 31), mhi = 0xffffffffu >> (31 - (x1 & 31));
    // rows g8, g8 + 8, ...; four rows' words in flight per step
    for (int y = y0 + g8; y <= y1; y += 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int yy = y + 8 * q;
        if (yy > y1) break;
        const uint32_t *row = plane + (int64_t)yy * stride;
        for (int wq = w0; wq <= w1; ++wq) {
          const uint32_t m = (wq == w0 ? mlo : 0xffffffffu) & (wq == w1 ? mhi : 0xffffffffu);
          const uint32_t bits = __ldg(row + wq) & m;
          any |= bits != 0;
          all &= bits == m;
        }
      }
    }
  }
  any = (__ballot_sync(0xffffffffu, any) & gmask) != 0;
  all = (__ballot_sync(0xffffffffu, all) & gmask) == gmask;
  if (!query) return kTileMixed;
  return !any ? kTileBg : (all ? kTileFg : kTileMixed);
}

// 8x8-pixel cell maps of every camera's silhouette bits: any / all
// foreground over the cell's in-image pixels. One thread per 32 cells.
__device__ __forceinline__ void carve_cells(const CarveParams &p, int bid, int nblocks) {
  for (int64_t e = bid * (int64_t)blockDim.x + threadIdx.x; e < p.cell_total;
       e += (int64_t)nblocks * blockDim.x) {
    int c = 0;
    while (c + 1 < p.ncam && e >= p.cell_off[c + 1]) ++c;
    const int64_t local = e - p.cell_off[c];
    const int W = p.cams[c].width, H = p.cams[c].height;
    const int cw = p.cell_words[c];
    const int cy = (int)(local / cw), wq = (int)(local - (int64_t)cy * cw);
    const uint32_t *plane = p.sil + p.sil_off[c];
    const int stride = p.sil_stride[c];
    uint32_t any = 0, all = 0;
    // cells 32 wq .. 32 wq + 31 span pixel words 8 wq .. 8 wq + 7 (4 cells each)
    for (int q = 0; q < 8; ++q) {
      const int pw = 8 * wq + q;
      if (pw >= stride) break;
      // pixels beyond the right edge count as foreground for "all"
      const int x_end = W - 32 * pw;  // valid bits in this word
      const uint32_t valid = x_end >= 32 ? 0xffffffffu : (x_end <= 0 ? 0u : (1u << x_end) - 1u);
      uint32_t o = 0, a = 0xffffffffu;
      for (int r = 0; r < 8; ++r) {
        const int y = 8 * cy + r;
        if (y >= H) break;
        const uint32_t w = __ldg(plane + (int64_t)y * stride + pw);
        o |= w;
        a &= w | ~valid;
      }
      for (int bb = 0; bb < 4; ++bb) {
        const uint32_t bo = (o >> (8 * bb)) & 0xffu, ba = (a >> (8 * bb)) & 0xffu;
        any |= (uint32_t)(bo != 0) << (4 * q + bb);
        all |= (uint32_t)(ba == 0xffu) << (4 * q + bb);
      }
    }
    p.cell_any[e] = any;
    p.cell_all[e] = all;
  }
}

// Per-(grid, camera) FP32 coefficients, once per launch.
__device__ __forceinline__ void carve_affine(const CarveParams &p, CamAffine *out, int bid,
                                             int nblocks) {
  const int n = p.gt->ngrid * p.ncam;
  for (int e = bid * blockDim.x + threadIdx.x; e < n; e += nblocks * blockDim.x) {
    cam_affine(p.cams[e % p.ncam], p.gt->grids[e / p.ncam], out[e]);
    out[e].sil_off = (int)p.sil_off[e % p.ncam];  // (< 2^31 words: checked in carve_batch)
    out[e].sil_stride = p.sil_stride[e % p.ncam];
  }
}

struct __align__(16) TileWork {
  int g, i0, j0, k0, n_fg, nm;
  uint8_t mixed[FVV_MAX_CAMS];  // cameras whose silhouette boundary crosses the tile, test order
  int pad[2];
};

// The voxels v0 .. v1 of a tile (v = di + kT (dj + kT dk)): the mixed
// cameras per voxel in FP32 (float64 deferral via settle), ON bits set.
// Returns this thread's ON count.
__device__ __forceinline__ int carve_voxels(const CarveParams &p, const CamAffine *aff,
                                            const fvv_grid &G, int g, int i0, int j0, int k0,
                                            int i1, int j1, int k1, const int *mixed,
                                            const float2 *mbound, int nm,
                                            int n_fg, int v0, int v1, int tl,
                                            int64_t word_off) {
  const int kT = 1 << tl;
  uint32_t *occ_g = p.occ + word_off;
  const int64_t nx = G.dims[0], ny = G.dims[1];
  int my_on = 0;
  const int lane = threadIdx.x & 31;
  // (v1 - v0 and blockDim.x are multiples of 32: whole warps take the loop)
  for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    const int i = i0 + (v & (kT - 1)), j = j0 + ((v >> tl) & (kT - 1)), k = k0 + (v >> (2 * tl));
    const bool inside = i <= i1 && j <= j1 && k <= k1;
    const float fi = (float)i, fj = (float)j, fk = (float)k;
    int seen = n_fg;
    bool off = !inside;
    unsigned long long amb = 0;
    for (int m = 0; m < (inside ? nm : 0); ++m) {
      const int c = mixed[m];
      const float2 eb = mbound[m];  // (negative: no box bounds for this camera)
      int px, py;
      const int st = eb.x >= 0.0f ? classify32_box(aff[c], eb.x, eb.y, fi, fj, fk, px, py)
                                  : classify32(aff[c], fi, fj, fk, px, py);
      if (st == kOut) continue;
      if (st == kAmb) {
        amb |= 1ull << c;
        continue;
      }
      ++seen;
      const CamAffine &a = aff[c];  // (32-bit word index: planes < 2^31 words)
      const uint32_t wi = (uint32_t)a.sil_off + (uint32_t)py * (uint32_t)a.sil_stride +
                          ((uint32_t)px >> 5);
      if (!((__ldg(p.sil + wi) >> (px & 31)) & 1u)) {
        off = true;
        break;
      }
    }
    const int64_t l = (int64_t)i + nx * ((int64_t)j + ny * (int64_t)k);
    const bool on = !off && settle(p, G, g, l, seen, amb);
    my_on += on;
    // warp-ballot packing: lane r * kT holds row r's ON bits (consecutive i,
    // so consecutive linear indices l .. l + kT - 1)
    const unsigned ballot = __ballot_sync(0xffffffffu, on);
    if ((lane & (kT - 1)) == 0) {
      const unsigned rowmask = kT >= 32 ? 0xffffffffu : ((1u << kT) - 1u);
      const unsigned row = (ballot >> lane) & rowmask;
      if (row) {
        uint32_t *w = occ_g + (l >> 5);
        const int sh = (int)(l & 31);
        atomicOr(w, row << sh);
        if (sh + kT > 32 && (row >> (32 - sh))) atomicOr(w + 1, row >> (32 - sh));
      }
    }
  }
  return my_on;
}

// One block per tile: classify the tile for every camera, then (fused mode)
// carve its voxels, or (kSplit, the 16^3 stage-grid tiles) append the
// surviving tile to p.tiles for carve_voxels_kernel.
template <bool kSplit>
__global__ void __launch_bounds__(kCarveThreads, FVV_CARVE_MINB)
    carve_kernel(const __grid_constant__ CarveParams p) {
  pdl_wait();
  __shared__ CamAffine aff[FVV_MAX_CAMS];
  __shared__ int state[FVV_MAX_CAMS];
  __shared__ int mixed[FVV_MAX_CAMS];
  __shared__ float2 sbound[FVV_MAX_CAMS], mbound[FVV_MAX_CAMS];
  __shared__ int n_mixed, n_fg, culled;
  __shared__ int blk[4];  // grid, tile origin i0 j0 k0 (thread 0, for the block)
  __shared__ fvv_grid s_grid;  // its grid and occupancy word offset
  __shared__ int64_t s_woff;
  const int tl = p.tile_log2, kT = 1 << tl;
  const CarveGrids &T = *p.gt;
  if (threadIdx.x == 0) {
    const int64_t b = blockIdx.x;
    int gg = -1;
    if (b < __ldg(&T.total_tiles)) {  // (device-planned batches launch a capacity)
      gg = 0;  // binary search of the block's grid
      const int ng = __ldg(&T.ngrid);
      for (int step = FVV_MAX_GRIDS / 2; step >= 1; step >>= 1)
        if (gg + step < ng && b >= __ldg(&T.blk_start[gg + step])) gg += step;
      const uint32_t tx = __ldg(&T.tiles_x[gg]), ty = __ldg(&T.tiles_y[gg]);
      const uint32_t tile = (uint32_t)(b - __ldg(&T.blk_start[gg]));  // < 2^32 tiles per grid
      const uint32_t tq = tile / tx;
      blk[1] = (int)((tile - tq * tx) * kT);
      blk[2] = (int)((tq % ty) * kT);
      blk[3] = (int)((tq / ty) * kT);
    }
    blk[0] = gg;
    if (gg >= 0) {
      s_grid = T.grids[gg];
      s_woff = T.word_off[gg];
    }
    culled = 0;
  }
  __syncthreads();
  const int g = blk[0], i0 = blk[1], j0 = blk[2], k0 = blk[3];
  if (g < 0) return;
  const fvv_grid &G = s_grid;
  const int64_t nx = G.dims[0], ny = G.dims[1], nz = G.dims[2];
  const int i1 = (int)min((int64_t)i0 + kT, nx) - 1, j1 = (int)min((int64_t)j0 + kT, ny) - 1,
            k1 = (int)min((int64_t)k0 + kT, nz) - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kCarveThreads / 32;
  {  // this grid's camera coefficients (carve_affine_kernel) into shared memory
    const float4 *src = (const float4 *)(p.affine + (int64_t)g * p.ncam);
    float4 *dst = (float4 *)aff;
    for (int e = threadIdx.x; e < p.ncam * (int)(sizeof(CamAffine) / 16); e += blockDim.x)
      dst[e] = __ldg(src + e);
  }
  __syncthreads();
  // every camera's tile state, four cameras per warp (eight lanes each)
  for (int t0 = 0; t0 < p.ncam; t0 += 4 * kWarps) {
    const int t = t0 + 4 * warp + (lane >> 3);
    const int c = t < p.ncam ? p.order[t] : -1;
    bool box;
    float beu, bev;
    const int st = tile_camera(p, aff, c, i0, i1, j0, j1, k0, k1, lane, box, beu, bev);
    if (c >= 0 && (lane & 7) == 0) {
      state[t] = st;
      sbound[t] = box ? make_float2(beu, bev) : make_float2(-1.0f, -1.0f);
      if (st == kTileBg) culled = 1;
    }
  }
  __syncthreads();
  if (culled) {  // every voxel of the tile is OFF (words pre-zeroed)
    if (threadIdx.x == 0) atomicAdd(p.tile_stats, 1ull);
    return;
  }
  if (threadIdx.x == 0) {
    int nm = 0, nf = 0;
    for (int t = 0; t < p.ncam; ++t) {
      if (state[t] == kTileFg) {
        ++nf;
      } else {
        mbound[nm] = sbound[t];
        mixed[nm++] = p.order[t];
      }
    }
    n_mixed = nm;
    n_fg = nf;
    atomicAdd(p.tile_stats + 1, (unsigned long long)nf);
    atomicAdd(p.tile_stats + 2, (unsigned long long)nm);
  }
  __syncthreads();
  if (kSplit) {  // hand the tile to carve_voxels_kernel
    if (threadIdx.x == 0) {
      const unsigned long long slot = atomicAdd(p.ntiles, 1ull);
      if ((int64_t)slot < p.tile_cap) {
        TileWork &tw = p.tiles[slot];
        tw.g = g;
        tw.i0 = i0;
        tw.j0 = j0;
        tw.k0 = k0;
        tw.n_fg = n_fg;
        tw.nm = n_mixed;
        for (int m = 0; m < n_mixed; ++m) tw.mixed[m] = (uint8_t)mixed[m];
      }
    }
    return;
  }
  const int my_on = carve_voxels(p, aff, G, g, i0, j0, k0, i1, j1, k1, mixed, mbound, n_mixed,
                                 n_fg, 0, 1 << (3 * tl), tl, s_woff);
  if (p.count) {  // per-warp atomics: no block barrier at the end
    const int s = __reduce_add_sync(0xffffffffu, my_on);
    if (lane == 0 && s) atomicAdd((unsigned long long *)&p.count[g], (unsigned long long)s);
  }
}

// Split mode, part 2: one block per 8^3 octant of each surviving 16^3 tile.
// The octant is classified again, for the cameras whose boundary crosses the
// whole tile only (a camera all-foreground over the tile is so over the
// octant), which culls like 8^3 tiles do, then its 512 voxels are carved.
// kLoop (the launch used): one resident wave of blocks takes the octants of
// the surviving tiles from a counter; !kLoop: one block per octant of every
// tile, blocks past the surviving count exit.
template <bool kLoop, int kThreads>
__global__ void __launch_bounds__(kThreads, oct_min_blocks<kThreads>())
    carve_voxels_kernel(const __grid_constant__ CarveParams p) {
  pdl_wait();
  __shared__ CamAffine aff[FVV_MAX_CAMS];
  __shared__ int tmixed[FVV_MAX_CAMS], state[FVV_MAX_CAMS], mixed[FVV_MAX_CAMS];
  __shared__ float2 sbound[FVV_MAX_CAMS], mbound[FVV_MAX_CAMS];
  __shared__ int n_mixed, n_fg, culled;
  __shared__ fvv_grid s_grid;
  __shared__ int64_t s_woff;
  __shared__ int64_t s_next;
  int64_t n = (int64_t)__ldcg(p.ntiles);
  if (n > p.tile_cap) n = p.tile_cap;
  // kLoop: a grid of resident blocks takes the octants from a counter (many
  // tiles, or a capacity launch: one block per octant would spend its time
  // launching empty blocks, and octants differ widely in cost)
  for (int64_t w = blockIdx.x; w < n * 8;) {
  if (kLoop) {
    __syncthreads();  // the previous octant is done with the shared arrays
    if (threadIdx.x == 0) s_next = (int64_t)atomicAdd(p.ntiles + 1, 1ull);
    __syncthreads();
    w = s_next;
    if (w >= n * 8) break;
  }
  const TileWork &tw = p.tiles[w >> 3];
  const int oct = (int)(w & 7);
  const int g = __ldcg(&tw.g), tnm = __ldcg(&tw.nm);
  const int i0 = __ldcg(&tw.i0) + 8 * (oct & 1), j0 = __ldcg(&tw.j0) + 8 * ((oct >> 1) & 1),
            k0 = __ldcg(&tw.k0) + 8 * (oct >> 2);
  if (threadIdx.x == 0) {
    s_grid = p.gt->grids[g];
    s_woff = p.gt->word_off[g];
  }
  const fvv_grid &G = s_grid;
  __syncthreads();
  if (i0 >= G.dims[0] || j0 >= G.dims[1] || k0 >= G.dims[2]) {  // octant off the grid
    if (kLoop) continue;
    return;
  }
  const int i1 = (int)min((int64_t)i0 + 8, G.dims[0]) - 1,
            j1 = (int)min((int64_t)j0 + 8, G.dims[1]) - 1,
            k1 = (int)min((int64_t)k0 + 8, G.dims[2]) - 1;
  {
    const float4 *src = (const float4 *)(p.affine + (int64_t)g * p.ncam);
    float4 *dst = (float4 *)aff;
    for (int e = threadIdx.x; e < p.ncam * (int)(sizeof(CamAffine) / 16); e += blockDim.x)
      dst[e] = __ldg(src + e);
  }
  for (int m = threadIdx.x; m < tnm; m += blockDim.x) tmixed[m] = __ldcg(&tw.mixed[m]);
  if (threadIdx.x == 0) culled = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;
  for (int m0 = 0; m0 < tnm; m0 += 4 * kWarps) {
    if (m0 + 4 * warp >= tnm) break;  // (warp-uniform)
    const int m = m0 + 4 * warp + (lane >> 3);
    const int c = m < tnm ? tmixed[m] : -1;
    bool box;
    float beu, bev;
    const int st = tile_camera(p, aff, c, i0, i1, j0, j1, k0, k1, lane, box, beu, bev);
    if (c >= 0 && (lane & 7) == 0) {
      state[m] = st;
      sbound[m] = box ? make_float2(beu, bev) : make_float2(-1.0f, -1.0f);
      if (st == kTileBg) culled = 1;
    }
  }
  __syncthreads();
  if (culled) {
    if (threadIdx.x == 0) atomicAdd(p.tile_stats + 3, 1ull);  // culled octants
    if (kLoop) continue;
    return;
  }
  if (threadIdx.x == 0) {
    int nm = 0, nf = __ldcg(&tw.n_fg);
    atomicAdd(p.tile_stats + 4, 1ull);  // carved octants
    for (int m = 0; m < tnm; ++m) {
      if (state[m] == kTileFg) {
        ++nf;
      } else {
        mbound[nm] = sbound[m];
        mixed[nm++] = tmixed[m];
      }
    }
    n_mixed = nm;
    n_fg = nf;
    atomicAdd(p.tile_stats + 5, (unsigned long long)nm);  // their mixed cameras
  }
  __syncthreads();
  const int my_on = carve_voxels(p, aff, G, g, i0, j0, k0, i1, j1, k1, mixed, mbound, n_mixed,
                                 n_fg, 0, 512, 3, s_woff);
  if (p.count) {
    const int s = __reduce_add_sync(0xffffffffu, my_on);
    if (lane == 0 && s) atomicAdd((unsigned long long *)&p.count[g], (unsigned long long)s);
  }
  if (!kLoop) return;
  }
}

// Zero the occupancy words of every grid of the batch (tiles only set bits).
__device__ __forceinline__ void carve_zero(const CarveParams &p, int bid, int nblocks) {
  const CarveGrids &T = *p.gt;
  for (int g = 0; g < T.ngrid; ++g) {
    const fvv_grid &G = T.grids[g];
    const int64_t words = (G.dims[0] * G.dims[1] * G.dims[2] + 31) / 32;
    uint32_t *occ_g = p.occ + T.word_off[g];
    for (int64_t w = bid * (int64_t)blockDim.x + threadIdx.x; w < words;
         w += (int64_t)nblocks * blockDim.x)
      occ_g[w] = 0u;
  }
}

// One launch for the per-call preparation: camera coefficients, silhouette
// cell maps, zeroed occupancy words (block ranges of one grid).
__global__ void carve_prep_kernel(const __grid_constant__ CarveParams p, CamAffine *aff,
                                  int nb_aff, int nb_cells, int ncount) {
  pdl_wait();
  const int b = blockIdx.x;
  if (b == 0) {  // the launch's counters (the carve kernels run after this one)
    if (threadIdx.x < 32) p.tile_stats[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
      p.amb[0] = 0ull;
      p.ntiles[0] = p.ntiles[1] = 0ull;
    }
    if (p.count)
      for (int g = threadIdx.x; g < ncount; g += blockDim.x) p.count[g] = 0;
  }
  if (b < nb_aff) carve_affine(p, aff, b, nb_aff);
  else if (b < nb_aff + nb_cells) carve_cells(p, b - nb_aff, nb_cells);
  else carve_zero(p, b - nb_aff - nb_cells, gridDim.x - nb_aff - nb_cells);
}

// Voxels the FP32 pass left undecided: their undecided cameras through the
// float64 chain, then set their bits.
__global__ void __launch_bounds__(kCarveThreads)
    carve_exact_kernel(const __grid_constant__ CarveParams p) {
  pdl_wait();
  // lanes test different cameras: a shared-memory copy (divergent indexing of
  // the parameter block would serialise the constant cache)
  __shared__ fvv_camera cams[FVV_MAX_CAMS];
  int64_t n = (int64_t)__ldcg(p.amb);
  if (n > p.amb_cap) n = p.amb_cap;
  if (blockIdx.x * (int64_t)blockDim.x >= n) return;  // (block-uniform: no entries here)
  {  // copied word by word by the whole block (one thread per camera would
     // serialise ~50 divergent parameter loads per lane)
    static_assert(sizeof(fvv_camera) % 4 == 0, "cameras are copied in 32-bit words");
    const uint32_t *src = reinterpret_cast<const uint32_t *>(p.cams);
    uint32_t *dst = reinterpret_cast<uint32_t *>(cams);
    for (int e = threadIdx.x; e < p.ncam * (int)(sizeof(fvv_camera) / 4); e += blockDim.x)
      dst[e] = src[e];
  }
  __syncthreads();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long e = p.amb[1 + 2 * q], mask = p.amb[2 + 2 * q];
    const int g = (int)((e >> 40) & 0x7f);
    const int seen = (int)((e >> 47) & 0x7f);
    const int64_t l = (int64_t)(e & ((1ull << 40) - 1));
    if (carve_exact(p, cams, p.gt->grids[g], l, mask, seen)) {
      atomicOr(p.occ + p.gt->word_off[g] + (l >> 5), 1u << (l & 31));
      if (p.count) atomicAdd((unsigned long long *)&p.count[g], 1ull);
    }
  }
}

}  // namespace fvv

using namespace fvv;

static size_t affine_bytes() {
  return (sizeof(CamAffine) * FVV_MAX_GRIDS * FVV_MAX_CAMS + 255) & ~(size_t)255;
}

static int64_t cell_words_total(const fvv_camera *cams, int ncam) {
  int64_t n = 0;
  for (int c = 0; c < ncam; ++c)
    n += (int64_t)((cams[c].height + 7) >> 3) * ((((cams[c].width + 7) >> 3) + 31) >> 5);
  return n;
}

static size_t cells_bytes(const fvv_camera *cams, int ncam) {
  return (2 * sizeof(uint32_t) * (size_t)cell_words_total(cams, ncam) + 255) & ~(size_t)255;
}

static size_t grids_bytes() { return (sizeof(CarveGrids) + 255) & ~(size_t)255; }

size_t fvv::carve_grids_offset(const fvv_camera *cams, int ncam) {
  const size_t end = affine_bytes() + 256 + cells_bytes(cams, ncam) +
                     sizeof(unsigned long long) * (1 + 2 * (size_t)kAmbCap) + 512 +
                     sizeof(TileWork) * (size_t)kTileCap;
  return (end + 255) & ~(size_t)255;
}

extern "C" size_t fvv_carve_workspace_bytes(const fvv_camera *cams, int ncam) {
  if (!cams || ncam < 1 || ncam > FVV_MAX_CAMS) return 0;
  return carve_grids_offset(cams, ncam) + grids_bytes();  // (the tile list ends before it)
}

namespace fvv {
static_assert(sizeof(CarveGrids) % 16 == 0, "CarveGrids is copied in 16-byte words");
__global__ void store_carve_grids_kernel(const __grid_constant__ CarveGrids src, CarveGrids *dst) {
  pdl_wait();
  const int4 *a = reinterpret_cast<const int4 *>(&src);
  int4 *b = reinterpret_cast<int4 *>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(CarveGrids) / 16); i += blockDim.x) b[i] = a[i];
}
}  // namespace fvv

int fvv::carve_batch(const fvv_camera *cams, int ncam, const uint32_t *sil_dev,
                     const int64_t *sil_word_off, const CarveGrids *gt_dev, int ngrid_max,
                     int tile_log2, int64_t blocks, int min_views, uint32_t *occ_dev,
                     int64_t *count_dev, void *workspace, size_t ws_bytes, cudaStream_t st,
                     bool reuse_cells) {
  if (ngrid_max == 0 || blocks == 0) {
    if (count_dev && ngrid_max) fill_async(count_dev, 0, sizeof(int64_t) * ngrid_max, st);
    return cuda_check("fvv_carve");
  }
  static thread_local CarveParams p;  // ~13 KB: keep it off the host stack
  memset(&p, 0, sizeof(p));
  p.ncam = ncam;
  p.min_views = min_views;
  p.sil = sil_dev;
  p.occ = occ_dev;
  p.count = count_dev;
  p.gt = gt_dev;
  const size_t need = fvv_carve_workspace_bytes(cams, ncam);
  if (!workspace || ws_bytes < need) {
    set_error("fvv_carve: workspace of %zu bytes needed", need);
    return FVV_E_ARG;
  }
  char *ws = (char *)workspace;
  p.affine = (const CamAffine *)ws;
  p.tile_stats = (unsigned long long *)(ws + affine_bytes());
  p.cell_any = (uint32_t *)(ws + affine_bytes() + 256);
  p.cell_all = p.cell_any + cell_words_total(cams, ncam);
  p.amb = (unsigned long long *)(ws + affine_bytes() + 256 + cells_bytes(cams, ncam));
  p.ntiles = (unsigned long long *)(((uintptr_t)(p.amb + 1 + 2 * kAmbCap) + 255) & ~(uintptr_t)255);
  p.tiles = (TileWork *)((char *)p.ntiles + 256);
  p.tile_cap = kTileCap;
  {
    int64_t off = 0;
    for (int c = 0; c < ncam; ++c) {
      p.cell_off[c] = off;
      p.cell_words[c] = (((cams[c].width + 7) >> 3) + 31) >> 5;
      off += (int64_t)((cams[c].height + 7) >> 3) * p.cell_words[c];
    }
    p.cell_total = off;
  }
  p.amb_cap = kAmbCap;
  // phase-1 cameras: up to 4 spread evenly through the rig order (ring rigs:
  // roughly orthogonal views), then the rest in rig order
  p.k1 = ncam < 4 ? ncam : 4;
  {
    bool used[FVV_MAX_CAMS] = {};
    int t = 0;
    for (int m = 0; m < p.k1; ++m) {
      const int c = (int)((int64_t)m * ncam / p.k1);
      p.order[t++] = c;
      used[c] = true;
    }
    for (int c = 0; c < ncam; ++c)
      if (!used[c]) p.order[t++] = c;
  }
  for (int c = 0; c < ncam; ++c) {
    p.cams[c] = cams[c];
    p.sil_off[c] = sil_word_off[c];
    if (sil_word_off[c] < 0 || sil_word_off[c] > 0x7fffffffll) {
      set_error("fvv_carve: silhouette plane %d at word %lld (the carve addresses < 2^31 words)",
                c, (long long)sil_word_off[c]);
      return FVV_E_LIMIT;
    }
    p.sil_stride[c] = sil_stride_words(cams[c].width);
  }
  p.tile_log2 = tile_log2;
  if (blocks > 0x7fffffff) {
    set_error("fvv_carve: %lld blocks", (long long)blocks);
    return FVV_E_LIMIT;
  }
  const int nb_aff = (ngrid_max * ncam + 255) / 256;
  // (the cell maps depend on the silhouettes only: a batch over the same
  // planes as the previous carve into this workspace reuses them)
  const int nb_cells = reuse_cells ? 0 : (int)((cell_words_total(cams, ncam) + 255) / 256);
  launch_k(carve_prep_kernel, nb_aff + nb_cells + 148 * 2, 256, 0, st, p, (CamAffine *)workspace, nb_aff,
                                                                nb_cells, ngrid_max);
  // large (stage) grids: classify the 16^3 tiles, then carve the surviving
  // tiles' voxels with kParts blocks each; ROI grids: one kernel per 8^3 tile
  const bool split = p.tile_log2 == 4 && blocks <= kTileCap;
  if (split) {
    launch_k(carve_kernel<true>, (unsigned)blocks, kCarveThreads, 0, st, p);
    // one block per octant of every tile (C3 ROI batch: ~70k octants); more
    // octants (C5 512^3: 131k, mostly of culled tiles): a capped grid loops
    // one resident wave of blocks taking octants from a counter (measured
    // against one block per octant of every tile: B-1 56 -> 44 us, B-3 equal)
    if (ngrid_max > 1) {
      launch_k(carve_voxels_kernel<true, 128>,
               (unsigned)std::min<int64_t>(blocks * 8, 148 * oct_min_blocks<128>()), 128, 0, st, p);
    } else {
      launch_k(carve_voxels_kernel<true, 256>,
               (unsigned)std::min<int64_t>(blocks * 8, 148 * oct_min_blocks<256>()), 256, 0, st, p);
    }
  } else {
    launch_k(carve_kernel<false>, (unsigned)blocks, kCarveThreads, 0, st, p);
  }
  launch_k(carve_exact_kernel, 148 * 4, kCarveThreads, 0, st, p);
  note_launches(split ? 4 : 3);
  return cuda_check("fvv_carve");
}

extern "C" int fvv_carve(const fvv_camera *cams, int ncam, const uint32_t *sil_dev,
                         const int64_t *sil_word_off, const fvv_grid *grids, int ngrid,
                         const int64_t *word_off, int min_views, uint32_t *occ_dev,
                         int64_t *count_dev, void *workspace, size_t ws_bytes, void *stream) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("fvv_carve: %d cameras (limit %d)", ncam, FVV_MAX_CAMS);
    return ncam < 1 ? FVV_E_ARG : FVV_E_LIMIT;
  }
  if (ngrid < 0 || ngrid > FVV_MAX_GRIDS) {
    set_error("fvv_carve: %d grids (limit %d)", ngrid, FVV_MAX_GRIDS);
    return FVV_E_LIMIT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = fvv_carve_workspace_bytes(cams, ncam);
  if (ngrid > 0 && (!workspace || ws_bytes < need)) {
    set_error("fvv_carve: workspace of %zu bytes needed", need);
    return FVV_E_ARG;
  }
  static thread_local CarveGrids T;
  memset(&T, 0, sizeof(T));
  T.ngrid = ngrid;
  // Batches of >= 4M voxels: 16^3 tiles, a cheap first classification that
  // culls empty space and fixes the all-foreground cameras, then one block
  // per 8^3 octant of the survivors (C3 ROI grids: 18 + 132 us vs. 162 us
  // for fused 8^3 tiles; stage grid 15 + 56 vs. 120 us). Smaller batches:
  // fused 8^3 tiles (C1 / C2 stage grids: 0.061 / 0.076 ms vs. 0.076 /
  // 0.091 ms split).
  int64_t total_vox = 0;
  for (int g = 0; g < ngrid; ++g)
    total_vox += grids[g].dims[0] * grids[g].dims[1] * grids[g].dims[2];
  T.tile_log2 = total_vox >= ((int64_t)4 << 20) ? 4 : 3;
  for (int g = 0; g < ngrid; ++g) {
    T.grids[g] = grids[g];
    T.word_off[g] = word_off[g];
    int64_t tiles;
    if (!carve_grid_tiles(grids[g], T.tile_log2, T.tiles_x[g], T.tiles_y[g], tiles)) {
      set_error("fvv_carve: grid %d has no voxels", g);
      return FVV_E_ARG;
    }
    T.blk_start[g + 1] = T.blk_start[g] + tiles;
  }
  for (int g = ngrid; g < FVV_MAX_GRIDS; ++g) T.blk_start[g + 1] = T.blk_start[ngrid];
  T.total_tiles = T.blk_start[ngrid];
  CarveGrids *dst = nullptr;
  if (ngrid > 0) {
    dst = (CarveGrids *)((char *)workspace + carve_grids_offset(cams, ncam));
    launch_k(store_carve_grids_kernel, 1, 256, 0, st, T, dst);
    note_launches(1);
  }
  return carve_batch(cams, ncam, sil_dev, sil_word_off, dst, ngrid, T.tile_log2, T.total_tiles,
                     min_views, occ_dev, count_dev, workspace, ws_bytes, st, false);
}
