// Stage C: marching cubes with silhouette-exact edge isovalues
// (mesh.py:131-374), batched over every ROI grid of a frame.
//
// Layout: each grid's occupancy is first transposed into "rows" (one row
// per (i, j), row index q = i*ny + j, C order) of ceil(nz/32) words holding
// consecutive k. In that layout the reference's orderings become word
// scans:
//   * vertices: one per sign-changing grid edge, ordered by (axis, i, j, k)
//     with k fastest (mesh.py:315-327 argwhere order). Edge-flag words
//     along axis 0/1 are XORs of neighbouring rows, along axis 2 an XOR
//     with the row shifted by one bit; an ordered popcount scan over
//     (grid, axis, row, word) gives every vertex its index.
//   * triangles: slot-major (TRI_TABLE triangle 0 of every surface cell in
//     C order, then triangle 1, ...) (mesh.py:351-359), winding reversed
//     (mesh.py:365), degenerate ones (area <= 1e-9 mm^2) dropped in place
//     (mesh.py:372-373): a 5-lane ordered scan over surface cells.
// Phase A (fvv_mesh_prepare) counts vertices and surface cells; the host
// sizes the outputs from those counts; phase B (fvv_mesh_emit) computes
// isovalues, vertices and triangles. All float64 work uses the reference's
// operation order (fvv_common.cuh, -fmad=false).
#include <cstring>
#include <mutex>

#include "mc_cases.cuh"
#include "scan.cuh"

namespace fvv {

__constant__ unsigned long long c_mc_edges[256];
__constant__ unsigned char c_mc_ntri[256];

// mesh.py:31-38 edge -> (base corner offset, axis), packed (di,dj,dk,axis)
__constant__ unsigned char c_edge_base[12][4] = {
    {0, 0, 0, 0}, {1, 0, 0, 1}, {0, 1, 0, 0}, {0, 0, 0, 1}, {0, 0, 1, 0}, {1, 0, 1, 1},
    {0, 1, 1, 0}, {0, 0, 1, 1}, {0, 0, 0, 2}, {1, 0, 0, 2}, {1, 1, 0, 2}, {0, 1, 0, 2}};

struct MeshBufs {
  const uint32_t *occ;
  uint32_t *tw;        // transposed words [tw_total]
  uint32_t *eflags;    // [3*tw_total]
  int32_t *vprefix;    // [3*tw_total]
  uint32_t *sflags;    // [tw_total]
  int32_t *sprefix;    // [tw_total]
  int64_t *sums;       // scan chunk sums
  int64_t *sums2;      // the cell scan's when it runs beside the vertex scan
  int64_t *totals;     // [0] V, [1] S, [2] T
  int64_t *info;       // [ngrid][8]: vbase V sbase S tbase T fallback inconsistent
  // phase B
  int64_t *vert_key;   // [V] V-element*32 + bit
  int32_t *cell_tri;   // [S][5][3] vertex indices of the cell's triangles, emitted order
  int64_t *cell_key;   // [S] S-element*32 + bit (the fused path's cell list)
  int32_t *cell_mask;  // [S] case | keep<<8 | grid<<16
  int32_t *cprefix;    // [S][5]
  int64_t *slot_base;  // [ngrid][5]
  int64_t *cell_sums;
  double *verts;       // [V][3]
  int32_t *tris;       // [T][3] global vertex indices
  int64_t cap_v, cap_s;  // phase-B capacities (emit kernels skip a batch that exceeds them)
  uint4 *zero;           // optional: cleared by the transpose kernel (scan status, totals)
  int64_t zero_n;        // its 16-byte words
};

// phase B runs only when the counts fit the buffers it was given
__device__ __forceinline__ bool emit_fits(const MeshBufs &B) {
  return __ldcg(B.totals) <= B.cap_v && __ldcg(B.totals + 1) <= B.cap_s;
}

enum { kInfoVbase, kInfoV, kInfoSbase, kInfoS, kInfoTbase, kInfoT, kInfoFallback, kInfoIncons };

__device__ __forceinline__ int grid_of(const MeshGrids &G, int64_t e) {
  // last g with tw_start[g] <= e < tw_start[g+1]
  int lo = 0, hi = G.ngrid - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (G.tw_start[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t row_word(const uint32_t *tw, const MeshGridInfo &gi, int64_t q,
                                             int64_t w) {
  return (w < gi.nzw) ? tw[gi.tw_off + q * gi.nzw + w] : 0u;
}

// row word shifted so bit b holds k+1
__device__ __forceinline__ uint32_t row_next(const uint32_t *tw, const MeshGridInfo &gi, int64_t q,
                                             int64_t w) {
  return (row_word(tw, gi, q, w) >> 1) | (row_word(tw, gi, q, w + 1) << 31);
}

// ---- A1: transpose F-order occupancy into k-rows --------------------------
// A warp takes 32 consecutive i of one (grid, j, k-row word w): lane L loads
// the 32 occupancy bits of row (j, k = 32 w + L) starting at i0 (a funnel
// shift of two words), and 32 ballots turn the 32 x 32 bit block around:
// ballot b collects bit b (= i0 + b) over the lanes (= k), i.e. the k-row
// word of column i0 + b. Two loads per 32 output words instead of 32 per word.
__global__ void mesh_transpose_kernel(const MeshGrids *__restrict__ Gp, MeshBufs B) {
  pdl_wait();
  const MeshGrids &G = *Gp;
  if (blockIdx.x == 0)  // the isovalue pass's per-grid counters (device-planned C has
    for (int g = threadIdx.x; g < G.ngrid; g += blockDim.x) {  // no grid-counts launch)
      B.info[8 * g + kInfoFallback] = 0;
      B.info[8 * g + kInfoIncons] = 0;
    }
  for (int64_t z = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; z < B.zero_n;
       z += (int64_t)gridDim.x * blockDim.x)
    B.zero[z] = make_uint4(0u, 0u, 0u, 0u);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = G.tr_total;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < total;
       t += nwarps) {
    int g = 0;  // last grid with tr_off <= t
    for (int step = FVV_MAX_GRIDS / 2; step >= 1; step >>= 1)
      if (g + step < G.ngrid && G.gi[g + step].tr_off <= t) g += step;
    const MeshGridInfo &gi = G.gi[g];
    const uint32_t local = (uint32_t)(t - gi.tr_off);
    const uint32_t rest = local / gi.nzw32, w = local - rest * gi.nzw32;
    const uint32_t ic = rest / gi.ny32, j = rest - ic * gi.ny32;
    const int64_t nx = gi.g.dims[0], ny = gi.g.dims[1], nz = gi.g.dims[2];
    const int64_t i0 = 32 * (int64_t)ic, k = 32 * (int64_t)w + lane;
    const int64_t nvalid = nx - i0 < 32 ? nx - i0 : 32;
    uint32_t bits = 0;
    if (k < nz) {
      const int64_t l0 = i0 + nx * (j + ny * k);
      const uint32_t *p = B.occ + gi.occ_word_off + (l0 >> 5);
      const int sh = (int)(l0 & 31);
      const uint32_t lo = __ldg(p), hi = (sh + nvalid > 32) ? __ldg(p + 1) : 0u;
      bits = __funnelshift_r(lo, hi, sh);
      if (nvalid < 32) bits &= (1u << nvalid) - 1u;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const uint32_t col = __ballot_sync(0xffffffffu, (bits >> b) & 1u);
      if (lane == b) mine = col;
    }
    if (lane < nvalid)
      B.tw[gi.tw_off + ((i0 + lane) * ny + j) * (int64_t)gi.nzw32 + w] = mine;
  }
}

// ---- A2: vertex (edge-flag) scan over (grid, axis, row, word) ---------------
// bits b of word w (of a row of n bits) with 32*w + b < n
__device__ __forceinline__ uint32_t kmask32(uint32_t w, int64_t n) {
  const int64_t r = n - 32 * (int64_t)w;
  return r <= 0 ? 0u : r >= 32 ? 0xffffffffu : (1u << r) - 1u;
}

// grid of element e of a space where grid g starts at mult*tw_start[g]
__device__ __forceinline__ int grid_of_scaled(const MeshGrids &G, int64_t e, int mult) {
  int lo = 0, hi = G.ngrid - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (mult * G.tw_start[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// One scan element = one word; decoded with 32-bit arithmetic (fill_grids
// bounds 3*tw_total below 2^31).
struct EdgeFlags {
  const MeshGrids *Gp;
  const uint32_t *tw;
  uint32_t *eflags;
  int32_t *vprefix;
  typedef uint32_t Item;
  __device__ uint32_t load(int64_t e) const {
    const MeshGrids &G = *Gp;
    // V space: grid g occupies [3*tw_start[g], 3*tw_start[g+1]), axis-major
    const int g = grid_of_scaled(G, e, 3);
    const MeshGridInfo &gi = G.gi[g];
    const uint32_t local = (uint32_t)(e - 3 * G.tw_start[g]);
    const uint32_t per_axis = gi.words32, nzw = gi.nzw32, ny = gi.ny32;
    const uint32_t axis = local / per_axis;
    const uint32_t rw = local - axis * per_axis;
    const uint32_t q = rw / nzw, w = rw - q * nzw;
    const uint32_t i = q / ny, j = q - i * ny;
    const uint32_t *row = tw + gi.tw_off + rw;  // word w of row q
    const uint32_t x = row[0];
    const int64_t nz = gi.g.dims[2];
    if (axis == 0)
      return (i + 1 < (uint32_t)gi.g.dims[0]) ? (x ^ row[ny * nzw]) & kmask32(w, nz) : 0u;
    if (axis == 1) return (j + 1 < ny) ? (x ^ row[nzw]) & kmask32(w, nz) : 0u;
    const uint32_t next = (x >> 1) | ((w + 1 < nzw ? row[1] : 0u) << 31);  // bit b holds k+1
    return (x ^ next) & kmask32(w, nz - 1);
  }
  __device__ int64_t value(uint32_t f) const { return __popc(f); }
  int64_t *vert_key;  // optional: the vertex list (V-element * 32 + bit), at most cap_v
  int64_t cap_v;
  __device__ void emit(int64_t e, int64_t prefix, uint32_t f) const {
    eflags[e] = f;
    vprefix[e] = (int32_t)prefix;
    if (vert_key)
      for (int64_t v = prefix; f && v < cap_v; ++v) {
        vert_key[v] = e * 32 + (__ffs(f) - 1);
        f &= f - 1;
      }
  }
};

// ---- A3: surface-cell scan over (grid, row, word) ---------------------------
struct CellFlags {
  const MeshGrids *Gp;
  const uint32_t *tw;
  uint32_t *sflags;
  int32_t *sprefix;
  typedef uint32_t Item;
  __device__ uint32_t load(int64_t e) const {
    const MeshGrids &G = *Gp;
    const int g = grid_of_scaled(G, e, 1);
    const MeshGridInfo &gi = G.gi[g];
    const uint32_t rw = (uint32_t)(e - G.tw_start[g]);
    const uint32_t nzw = gi.nzw32, ny = gi.ny32;
    const uint32_t q = rw / nzw, w = rw - q * nzw;
    const uint32_t i = q / ny, j = q - i * ny;
    if (i + 1 >= (uint32_t)gi.g.dims[0] || j + 1 >= ny) return 0u;
    const uint32_t *row = tw + gi.tw_off + rw;
    const uint32_t off[4] = {0u, ny * nzw, (ny + 1) * nzw, nzw};  // rows q, q+ny, q+ny+1, q+1
    const bool more = w + 1 < nzw;
    uint32_t any = 0u, all = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t a = row[off[r]];
      const uint32_t b = (a >> 1) | ((more ? row[off[r] + 1] : 0u) << 31);
      any |= a | b;
      all &= a & b;
    }
    return (any & ~all) & kmask32(w, gi.g.dims[2] - 1);
  }
  __device__ int64_t value(uint32_t f) const { return __popc(f); }
  int64_t *cell_key;  // optional: the surface-cell list (S-element * 32 + bit), at most cap_s
  int64_t cap_s;
  __device__ void emit(int64_t e, int64_t prefix, uint32_t f) const {
    sflags[e] = f;
    sprefix[e] = (int32_t)prefix;
    if (cell_key)
      for (int64_t c = prefix; f && c < cap_s; ++c) {
        cell_key[c] = e * 32 + (__ffs(f) - 1);
        f &= f - 1;
      }
  }
};

// per-grid vertex / surface-cell bases and counts (prefix at grid starts)
// grid g's vertex range [vb, ve) and surface-cell range [sb, se) from the
// scans' prefixes (the totals past the last grid)
__device__ __forceinline__ void grid_ranges(const MeshGrids &G, const MeshBufs &B, int g,
                                            int64_t &vb, int64_t &ve, int64_t &sb, int64_t &se) {
  const int64_t s0 = G.tw_start[g], s1 = G.tw_start[g + 1];
  vb = (s0 < G.tw_total) ? __ldcg(B.vprefix + 3 * s0) : __ldcg(B.totals + 0);
  ve = (s1 < G.tw_total) ? __ldcg(B.vprefix + 3 * s1) : __ldcg(B.totals + 0);
  sb = (s0 < G.tw_total) ? __ldcg(B.sprefix + s0) : __ldcg(B.totals + 1);
  se = (s1 < G.tw_total) ? __ldcg(B.sprefix + s1) : __ldcg(B.totals + 1);
}

__global__ void mesh_grid_counts_kernel(const MeshGrids *__restrict__ Gp, MeshBufs B) {
  pdl_wait();
  const MeshGrids &G = *Gp;
  for (int g = threadIdx.x; g < G.ngrid; g += blockDim.x) {
    int64_t vb, ve, sb, se;
    grid_ranges(G, B, g, vb, ve, sb, se);
    int64_t *inf = B.info + 8 * g;
    inf[kInfoVbase] = vb;
    inf[kInfoV] = ve - vb;
    inf[kInfoSbase] = sb;
    inf[kInfoS] = se - sb;
    inf[kInfoTbase] = 0;
    inf[kInfoT] = 0;
    inf[kInfoFallback] = 0;
    inf[kInfoIncons] = 0;
  }
}

// ---- B0: vertex list ----------------------------------------------------------
__global__ void mesh_vertex_list_kernel(const MeshGrids *__restrict__ Gp, MeshBufs B) {
  pdl_wait();
  const MeshGrids &G = *Gp;
  if (!emit_fits(B)) return;
  const int64_t n = 3 * G.tw_total;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t f = B.eflags[e];
    int64_t v = B.vprefix[e];
    while (f) {
      const int b = __ffs(f) - 1;
      f &= f - 1;
      B.vert_key[v++] = e * 32 + b;
    }
  }
}


// decode a V-space key -> grid, axis, (i, j, k)
__device__ __forceinline__ int decode_vkey(const MeshGrids &G, int64_t key, int &axis, int64_t &i,
                                           int64_t &j, int64_t &k) {
  const int64_t e = key >> 5;
  int lo = 0, hi = G.ngrid - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (3 * G.tw_start[mid] <= e) lo = mid; else hi = mid - 1;
  }
  const MeshGridInfo &gi = G.gi[lo];
  const uint32_t local = (uint32_t)(e - 3 * G.tw_start[lo]);  // 32-bit (fill_grids)
  const uint32_t a = local / gi.words32;
  const uint32_t rw = local - a * gi.words32;
  const uint32_t q = rw / gi.nzw32, w = rw - q * gi.nzw32;
  const uint32_t i32 = q / gi.ny32;
  axis = (int)a;
  i = i32;
  j = q - i32 * gi.ny32;
  k = (int64_t)w * 32 + (key & 31);
  return lo;
}


struct MeshCams {
  int ncam;
  int32_t sil_stride[FVV_MAX_CAMS];
  int64_t sil_off[FVV_MAX_CAMS];
  fvv_camera cams[FVV_MAX_CAMS];  // ascending camera id (mesh.py:165-167)
};

// mesh.py:131-162 closed-form Bresenham: pixel t of the segment a -> b.
__device__ __forceinline__ void bresenham_px(int ax, int ay, int bx, int by, int t, int &x,
                                             int &y) {
  const int dx = abs(bx - ax), dy = abs(by - ay);
  const int sx = bx >= ax ? 1 : -1, sy = by >= ay ? 1 : -1;
  const int major = dx > dy ? dx : dy;
  const bool xmajor = dx >= dy;
  const long long dmaj = major > 1 ? major : 1;
  const long long dmin = xmajor ? dy : dx;
  const int tc = t < major ? t : major;
  const int smin = (int)((2ll * tc * dmin + dmaj) / (2ll * dmaj));
  x = ax + sx * (xmajor ? tc : smin);
  y = ay + sy * (xmajor ? smin : tc);
}

// mesh.py:231-272 for one edge: cameras in ascending id order, only those
// seeing both endpoints; Bresenham walk from rint(p_on) to rint(p_off);
// lam_i = |last fg pixel - px_on| / |px_off - px_on| clipped to [0,1], 1 if
// unconstrained, 0 if the start pixel is background; min over cameras
// (strict <: ties keep the lower id). sel = camera slot or -1 (lam = 0.5).
// One camera's term of mesh.py:231-272 for one edge: valid (both endpoints
// in frustum), lam_i, and whether the walk starts on background.
__device__ __forceinline__ bool edge_lambda_cam(const fvv_camera &cam,
                                                const uint32_t *__restrict__ plane, int stride,
                                                const double *pon, const double *poff,
                                                bool gemv, double &lam_i, bool &incons) {
  double uo, vo, zo, uf, vf, zf;
  const bool ino = project_exact(cam, pon[0], pon[1], pon[2], true, gemv, uo, vo, zo);
  const bool inf = project_exact(cam, poff[0], poff[1], poff[2], true, gemv, uf, vf, zf);
  incons = false;
  if (!(ino && inf)) return false;
  const int ax = (int)rint(uo), ay = (int)rint(vo), bx = (int)rint(uf), by = (int)rint(vf);
  // the pixels of bresenham_px for t = 0..major, walked incrementally: the
  // minor offset floor((2 t dmin + dmaj) / (2 dmaj)) advances by at most one
  // per step (dmin <= dmaj), tracked as quotient + remainder
  const int dx = abs(bx - ax), dy = abs(by - ay);
  const int sx = bx >= ax ? 1 : -1, sy = by >= ay ? 1 : -1;
  const bool xmajor = dx >= dy;
  const int major = xmajor ? dx : dy;
  // (both endpoints are in the image: major < 2^16 keeps the remainder
  // arithmetic in 32 bits; loading 2-8 of the walk's pixel words at once
  // measured no faster, 98.5 -> 99 / 115 / 147 us)
  const int two_maj = 2 * (major > 1 ? major : 1), two_min = 2 * (xmajor ? dy : dx);
  int rem = two_maj / 2;
  int smin = 0, first_bg = -1, lx = ax, ly = ay;
  for (int t = 0; t <= major; ++t) {
    const int x = ax + sx * (xmajor ? t : smin), y = ay + sy * (xmajor ? smin : t);
    if (!sil_bit(plane, stride, x, y)) {
      first_bg = t;
      break;
    }
    lx = x;  // last foreground pixel so far
    ly = y;
    rem += two_min;
    if (rem >= two_maj) {
      rem -= two_maj;
      ++smin;
    }
  }
  const double ddx = uf - uo, ddy = vf - vo;
  const double denom = sqrt(ddx * ddx + ddy * ddy);
  lam_i = 1.0;
  if (first_bg == 0) {
    incons = true;
    lam_i = 0.0;
  } else if (first_bg > 0 && denom > 1e-12) {
    const double ex = (double)lx - uo, ey = (double)ly - vo;
    const double qv = sqrt(ex * ex + ey * ey) / denom;
    lam_i = qv > 1.0 ? 1.0 : qv;
  }
  return true;
}

__device__ __forceinline__ double edge_lambda(const MeshCams &C, const uint32_t *__restrict__ sil,
                                              const double *pon, const double *poff, bool gemv,
                                              int &sel, int &incons) {
  double lam = INFINITY;
  sel = -1;
  incons = 0;
  for (int c = 0; c < C.ncam; ++c) {
    double lam_i;
    bool inc;
    if (!edge_lambda_cam(C.cams[c], sil + C.sil_off[c], C.sil_stride[c], pon, poff, gemv, lam_i,
                         inc))
      continue;
    incons += inc;
    if (lam_i < lam) {
      lam = lam_i;
      sel = c;
    }
  }
  return sel < 0 ? 0.5 : lam;
}

// _edge_isovalues_batch (mesh.py:231-272) on explicit endpoint arrays.
__global__ void __launch_bounds__(128)
    edge_isovalues_kernel(const __grid_constant__ MeshCams C, const uint32_t *__restrict__ sil,
                          const double *__restrict__ pon, const double *__restrict__ poff, int64_t n,
                          double *lam_out, int32_t *cam_out, int64_t *stats) {
  pdl_wait();
  const bool gemv = (n == 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int sel, incons;
    const double lam = edge_lambda(C, sil, pon + 3 * e, poff + 3 * e, gemv, sel, incons);
    lam_out[e] = lam;
    cam_out[e] = sel < 0 ? -1 : C.cams[sel].id;
    if (sel < 0) atomicAdd((unsigned long long *)stats, 1ull);
    if (incons) atomicAdd((unsigned long long *)(stats + 1), (unsigned long long)incons);
  }
}

// ---- B1: isovalues + vertices (mesh.py:231-272, 332-337) --------------------
__global__ void __launch_bounds__(128)
    mesh_lambda_kernel(const MeshGrids *__restrict__ Gp, const __grid_constant__ MeshCams C,
                       MeshBufs B, const uint32_t *__restrict__ sil, int exact,
                       double fixed_iso) {
  pdl_wait();
  const MeshGrids &G = *Gp;
  if (!emit_fits(B)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) B.totals[3] = __ldcg(B.totals + 1);  // tri-scan length
  const int64_t nv = __ldcg(B.totals);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    int axis;
    int64_t i, j, k;
    const int g = decode_vkey(G, B.vert_key[v], axis, i, j, k);
    const MeshGridInfo &gi = G.gi[g];
    const int64_t q = i * gi.g.dims[1] + j;
    const bool on = (row_word(B.tw, gi, q, k >> 5) >> (k & 31)) & 1u;
    double p0[3], p1[3];
    voxel_center(gi.g, i, j, k, p0[0], p0[1], p0[2]);
    for (int d = 0; d < 3; ++d) p1[d] = p0[d] + gi.g.spacing * (double)(d == axis);
    const double *pon = on ? p0 : p1, *poff = on ? p1 : p0;
    double lam;
    if (exact) {
      // one-edge batch (numpy's gemv order): the grid's vertex range is this
      // vertex alone, i.e. its neighbours in the (ordered) vertex list lie in
      // other grids' V-element ranges
      const int64_t lo_e = 3 * G.tw_start[g], hi_e = 3 * G.tw_start[g + 1];
      const bool gemv = (v == 0 || (B.vert_key[v - 1] >> 5) < lo_e) &&
                        (v + 1 >= nv || (B.vert_key[v + 1] >> 5) >= hi_e);
      int sel, incons;
      lam = edge_lambda(C, sil, pon, poff, gemv, sel, incons);
      if (sel < 0)
        atomicAdd((unsigned long long *)(B.info + 8 * g + kInfoFallback), 1ull);
      if (incons)
        atomicAdd((unsigned long long *)(B.info + 8 * g + kInfoIncons),
                  (unsigned long long)incons);
    } else {
      lam = fixed_iso;
    }
    for (int d = 0; d < 3; ++d) B.verts[3 * v + d] = pon[d] + lam * (poff[d] - pon[d]);
  }
}

// global vertex index of cell-edge `edge` of cell (i, j, k) in grid gi
__device__ __forceinline__ int64_t edge_vertex(const MeshGrids &G, const MeshBufs &B, int g,
                                               int64_t i, int64_t j, int64_t k, int edge) {
  const MeshGridInfo &gi = G.gi[g];
  const int64_t bi = i + c_edge_base[edge][0], bj = j + c_edge_base[edge][1],
                bk = k + c_edge_base[edge][2];
  const int axis = c_edge_base[edge][3];
  const int64_t e = 3 * G.tw_start[g] + axis * gi.rows * gi.nzw + (bi * gi.g.dims[1] + bj) * gi.nzw +
                    (bk >> 5);
  return B.vprefix[e] + __popc(B.eflags[e] & ((1u << (bk & 31)) - 1u));
}

__device__ __forceinline__ int cell_case(const MeshBufs &B, const MeshGridInfo &gi, int64_t q,
                                         int64_t k) {
  const int64_t ny = gi.g.dims[1];
  const int64_t rows[4] = {q, q + ny, q + ny + 1, q + 1};  // corners v0..v3 (mesh.py:26-29)
  int ci = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t lo = row_word(B.tw, gi, rows[r], k >> 5);
    const uint32_t hi = row_word(B.tw, gi, rows[r], (k + 1) >> 5);
    ci |= ((lo >> (k & 31)) & 1u) << r;
    ci |= ((hi >> ((k + 1) & 31)) & 1u) << (r + 4);
  }
  return ci;
}

// ---- B2: surface-cell list, per-slot keep bits (mesh.py:339-373) ------------
// The case's distinct edges are looked up once each; the triangles' vertex
// indices (reversed winding, mesh.py:365) are kept for the emit pass.
__device__ __forceinline__ void mesh_cell(const MeshGrids &G, const MeshBufs &B, int64_t e,
                                          int b, int64_t c) {
  int lo = 0, hi = G.ngrid - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (G.tw_start[mid] <= e) lo = mid; else hi = mid - 1;
  }
  const int g = lo;
  const MeshGridInfo &gi = G.gi[g];
  const uint32_t rw = (uint32_t)(e - G.tw_start[g]);
  const uint32_t q32 = rw / gi.nzw32, w = rw - q32 * gi.nzw32;
  const uint32_t i32 = q32 / gi.ny32;
  const int64_t q = q32, i = i32, j = q32 - i32 * gi.ny32;
  const int64_t k = (int64_t)w * 32 + b;
  const int ci = cell_case(B, gi, q, k);
  const int ntri = c_mc_ntri[ci];
  const unsigned long long edges = c_mc_edges[ci];
  uint32_t used = 0;
  for (int n = 0; n < 3 * ntri; ++n) used |= 1u << ((edges >> (4 * n)) & 15);
  int32_t ev[12];
  for (uint32_t m = used; m; m &= m - 1) {
    const int ed = __ffs(m) - 1;
    ev[ed] = (int32_t)edge_vertex(G, B, g, i, j, k, ed);
  }
  int keep = 0;
  int32_t *out = B.cell_tri + 15 * c;
  for (int t = 0; t < ntri; ++t) {
    const int32_t v0 = ev[(edges >> (12 * t)) & 15];
    const int32_t v1 = ev[(edges >> (12 * t + 4)) & 15];
    const int32_t v2 = ev[(edges >> (12 * t + 8)) & 15];
    // reversed winding (v2, v1, v0); area as numpy: 0.5*|cross(B-A, C-A)|
    const double *A = B.verts + 3 * (int64_t)v2, *Bv = B.verts + 3 * (int64_t)v1,
                 *Cv = B.verts + 3 * (int64_t)v0;
    const double a0 = Bv[0] - A[0], a1 = Bv[1] - A[1], a2 = Bv[2] - A[2];
    const double b0 = Cv[0] - A[0], b1 = Cv[1] - A[1], b2 = Cv[2] - A[2];
    const double c0 = a1 * b2 - a2 * b1;
    const double c1 = a2 * b0 - a0 * b2;
    const double c2 = a0 * b1 - a1 * b0;
    const double area = 0.5 * sqrt((c0 * c0 + c1 * c1) + c2 * c2);
    if (area > kDegenerateArea) keep |= 1 << t;
    out[3 * t] = v2;
    out[3 * t + 1] = v1;
    out[3 * t + 2] = v0;
  }
  B.cell_mask[c] = ci | (keep << 8) | (g << 16);
}

// Surface cells, warp-cooperatively: a warp loads 32 consecutive surface-cell
// words, scans their popcounts, and hands the cells out one per lane (owner
// word by a shuffle binary search, then the n-th set bit), so sparse words
// do not leave lanes idle.
__global__ void mesh_cells_kernel(const MeshGrids *__restrict__ Gp, MeshBufs B) {
  pdl_wait();
  const MeshGrids &G = *Gp;
  if (!emit_fits(B)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) B.totals[3] = __ldcg(B.totals + 1);  // tri-scan length
  const int lane = threadIdx.x & 31;
  for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; e0 < G.tw_total;
       e0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e0 + lane;
    const uint32_t f = e < G.tw_total ? B.sflags[e] : 0u;
    const int cnt = __popc(f);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int sum = __shfl_sync(0xffffffffu, incl, 31);
    if (sum == 0) continue;
    for (int base = 0; base < sum; base += 32) {
      const int idx = base + lane;
      int own = 0;  // number of lanes whose inclusive count is <= idx
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, own + step - 1);
        if (v <= idx) own += step;
      }
      const int own_incl = __shfl_sync(0xffffffffu, incl, own);
      const int own_cnt = __shfl_sync(0xffffffffu, cnt, own);
      uint32_t of = __shfl_sync(0xffffffffu, f, own);
      if (idx < sum) {
        const int n = idx - (own_incl - own_cnt);
        for (int j = 0; j < n; ++j) of &= of - 1;
        const int bit = __ffs(of) - 1;
        const int64_t ew = e0 + own;
        mesh_cell(G, B, ew, bit, B.sprefix[ew] + n);
      }
    }
  }
}

struct Slot5 {
  int32_t v[5];
  __host__ __device__ Slot5() {  // cub value-initialises scan seeds with T{}
    for (int t = 0; t < 5; ++t) v[t] = 0;
  }
  __host__ __device__ Slot5(int x) {
    for (int t = 0; t < 5; ++t) v[t] = x;
  }
  __host__ __device__ Slot5 operator+(const Slot5 &o) const {
    Slot5 r;
    for (int t = 0; t < 5; ++t) r.v[t] = v[t] + o.v[t];
    return r;
  }
  __host__ __device__ Slot5 &operator+=(const Slot5 &o) {
    for (int t = 0; t < 5; ++t) v[t] += o.v[t];
    return *this;
  }
};

// ---- B3: 5-lane triangle scan over cells ------------------------------------
struct TriScan {
  const int32_t *cell_mask;
  int32_t *cprefix;
  typedef int Item;
  __device__ int load(int64_t c) const { return (cell_mask[c] >> 8) & 31; }
  __device__ Slot5 value(int keep) const {
    Slot5 s;
    for (int t = 0; t < 5; ++t) s.v[t] = (keep >> t) & 1;
    return s;
  }
  __device__ void emit(int64_t c, Slot5 prefix, int) const {
    for (int t = 0; t < 5; ++t) cprefix[5 * c + t] = prefix.v[t];
  }
};

// The fused path: the triangle scan's load evaluates the surface cell itself
// (case, per-slot keep bits, triangle vertex indices) from the cell list the
// cell scan emitted - one pass over the cells instead of two.
struct TriCells {
  const MeshGrids *Gp;
  MeshBufs B;
  typedef int Item;
  static constexpr int kItems = 1;  // a cell's evaluation is a long chain (measured: 57 -> 51 us)
  __device__ int load(int64_t c) const {
    const int64_t key = B.cell_key[c];
    mesh_cell(*Gp, B, key >> 5, (int)(key & 31), c);
    return (B.cell_mask[c] >> 8) & 31;
  }
  __device__ Slot5 value(int keep) const {
    Slot5 s;
    for (int t = 0; t < 5; ++t) s.v[t] = (keep >> t) & 1;
    return s;
  }
  __device__ void emit(int64_t c, Slot5 prefix, int) const {
    for (int t = 0; t < 5; ++t) B.cprefix[5 * c + t] = prefix.v[t];
  }
};

// ---- B4: per-grid slot bases (one warp, a lane per grid) ---------------------
// slot_base[g][t] = first triangle index of slot t of grid g minus the slot
// prefix at the grid's start (grids in order, slots in order inside a grid).
// With `info`, also the per-grid vertex / cell / triangle ranges and the
// triangle total (B.info, B.totals[2]).
__device__ __forceinline__ void slot_bases_warp(const MeshGrids &G, const MeshBufs &B,
                                                const Slot5 *total, int64_t *slot_base,
                                                bool info) {
  const int lane = threadIdx.x & 31;
  const int64_t S = B.totals[1];
  int64_t carry = 0;  // triangles of the grids before this chunk of 32
  for (int g0 = 0; g0 < G.ngrid; g0 += 32) {
    const int g = g0 + lane;
    int64_t p0[5], p1[5], cnt = 0;
    if (g < G.ngrid) {
      int64_t vb, ve, s0, s1;
      grid_ranges(G, B, g, vb, ve, s0, s1);
      if (info) {
        int64_t *inf = B.info + 8 * g;
        inf[kInfoVbase] = vb;
        inf[kInfoV] = ve - vb;
        inf[kInfoSbase] = s0;
        inf[kInfoS] = s1 - s0;
      }
      for (int t = 0; t < 5; ++t) {
        p0[t] = s0 < S ? B.cprefix[5 * s0 + t] : total->v[t];
        p1[t] = s1 < S ? B.cprefix[5 * s1 + t] : total->v[t];
        cnt += p1[t] - p0[t];
      }
    }
    int64_t incl = cnt;  // inclusive scan of the grids' triangle counts
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int64_t tbase = carry + incl - cnt;
    if (g < G.ngrid) {
      int64_t run = tbase;
      for (int t = 0; t < 5; ++t) {
        slot_base[5 * g + t] = run - p0[t];
        run += p1[t] - p0[t];
      }
      if (info) {
        B.info[8 * g + kInfoTbase] = tbase;
        B.info[8 * g + kInfoT] = run - tbase;
      }
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (info && lane == 0) B.totals[2] = carry;
}

__global__ void mesh_slot_bases_kernel(const MeshGrids *__restrict__ Gp, MeshBufs B,
                                       const Slot5 *total) {
  pdl_wait();
  const MeshGrids &G = *Gp;
  if (!emit_fits(B)) return;
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  slot_bases_warp(G, B, total, B.slot_base, true);
}

// ---- B5: triangle emission ----------------------------------------------------
// kSlots: each block first computes the slot bases itself into shared memory
// (warp 0; block 0 also writes the per-grid ranges and the triangle total),
// so no separate slot-bases launch runs between the triangle scan and here.
template <bool kSlots>
__global__ void mesh_emit_kernel(const MeshGrids *__restrict__ Gp, MeshBufs B,
                                 const Slot5 *total) {
  pdl_wait();
  if (!emit_fits(B)) return;
  __shared__ int64_t sbase[kSlots ? 5 * FVV_MAX_GRIDS : 1];
  const int64_t *slot_base = B.slot_base;
  if (kSlots) {
    if (threadIdx.x < 32) slot_bases_warp(*Gp, B, total, sbase, blockIdx.x == 0);
    __syncthreads();
    slot_base = sbase;
  }
  const int64_t S = __ldcg(B.totals + 1);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < S;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int m = B.cell_mask[c];
    const int keep = (m >> 8) & 31;
    if (!keep) continue;
    const int g = m >> 16;
    const int32_t *tv = B.cell_tri + 15 * c;
    for (int t = 0; t < 5; ++t) {
      if (!((keep >> t) & 1)) continue;
      const int64_t idx = slot_base[5 * g + t] + B.cprefix[5 * c + t];
      B.tris[3 * idx] = tv[3 * t];
      B.tris[3 * idx + 1] = tv[3 * t + 1];
      B.tris[3 * idx + 2] = tv[3 * t + 2];
    }
  }
}

constexpr int kMeshGrid = 148 * 8;

static size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

struct PrepLayout {
  size_t tw, eflags, vprefix, sflags, sprefix, sums, sums2, totals, info, slot5, grids, total;
};

// workspace of a batch of up to ngrid grids and tw_total k-row words
static PrepLayout prep_layout(int64_t tw_total, int ngrid) {
  PrepLayout L;
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off += al256(b);
    return o;
  };
  L.tw = take(4 * (size_t)tw_total);
  L.eflags = take(12 * (size_t)tw_total);
  L.vprefix = take(12 * (size_t)tw_total);
  L.sflags = take(4 * (size_t)tw_total);
  L.sprefix = take(4 * (size_t)tw_total);
  L.sums = take(onepass_bytes<int64_t>(3 * tw_total + 1));  // scan status words
  L.sums2 = take(onepass_bytes<int64_t>(tw_total + 1));      // (the concurrent cell scan's)
  L.totals = take(8 * 4);  // V, S, T, S for the triangle scan (0: phase B skipped)
  L.info = take(8 * 8 * (size_t)(ngrid > 0 ? ngrid : 1));
  L.slot5 = take(sizeof(int64_t) * 5 * (size_t)(ngrid > 0 ? ngrid : 1) + sizeof(Slot5));
  L.grids = take(sizeof(MeshGrids));  // the host wrappers' grid table
  L.total = off;
  return L;
}

static MeshBufs bufs_from(void *ws, const PrepLayout &L) {
  char *p = (char *)ws;
  MeshBufs B;
  memset(&B, 0, sizeof(B));
  B.tw = (uint32_t *)(p + L.tw);
  B.eflags = (uint32_t *)(p + L.eflags);
  B.vprefix = (int32_t *)(p + L.vprefix);
  B.sflags = (uint32_t *)(p + L.sflags);
  B.sprefix = (int32_t *)(p + L.sprefix);
  B.sums = (int64_t *)(p + L.sums);
  B.sums2 = (int64_t *)(p + L.sums2);
  B.totals = (int64_t *)(p + L.totals);
  B.info = (int64_t *)(p + L.info);
  B.slot_base = (int64_t *)(p + L.slot5);
  return B;
}

// phase-B scratch: vertex list, cell list, per-cell triangles / case+keep /
// slot prefixes, the triangle scan's status words
struct ScratchLayout {
  int64_t *vert_key, *cell_key;
  int32_t *cell_tri, *cell_mask, *cprefix;
  Slot5 *cell_sums;
  size_t total;
};

static ScratchLayout scratch_layout(void *scratch, int64_t cap_v, int64_t cap_s) {
  ScratchLayout S;
  char *base = (char *)scratch, *s = base;
  S.vert_key = (int64_t *)s;
  s += al256(8 * (size_t)cap_v);
  S.cell_key = (int64_t *)s;
  s += al256(8 * (size_t)cap_s);
  S.cell_tri = (int32_t *)s;
  s += al256(60 * (size_t)cap_s);
  S.cell_mask = (int32_t *)s;
  s += al256(4 * (size_t)cap_s);
  S.cprefix = (int32_t *)s;
  s += al256(20 * (size_t)cap_s);
  S.cell_sums = (Slot5 *)s;
  s += al256(onepass_bytes<Slot5>(cap_s + 1));
  S.total = (size_t)(s - base);
  return S;
}

static_assert(sizeof(MeshGrids) % 16 == 0, "MeshGrids is copied in 16-byte words");
__global__ void store_mesh_grids_kernel(const __grid_constant__ MeshGrids src, MeshGrids *dst) {
  pdl_wait();
  const int4 *a = reinterpret_cast<const int4 *>(&src);
  int4 *b = reinterpret_cast<int4 *>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(MeshGrids) / 16); i += blockDim.x) b[i] = a[i];
}

}  // namespace fvv

using namespace fvv;

// marching-cubes tables into constant memory once per process (executor
// lanes may race here on first use)
static std::once_flag g_tables_once;
static int g_tables_rc = FVV_OK;

static int ensure_tables() {
  std::call_once(g_tables_once, [] {
    if (cudaMemcpyToSymbol(c_mc_edges, FVV_MC_EDGES, sizeof(FVV_MC_EDGES)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_mc_ntri, FVV_MC_NTRI, sizeof(FVV_MC_NTRI)) != cudaSuccess)
      g_tables_rc = cuda_check("mesh tables");
  });
  return g_tables_rc;
}

// host grid table of a wrapper call
static int fill_grids(const fvv_grid *grids, int ngrid, const int64_t *word_off, MeshGrids &G) {
  if (ngrid < 1 || ngrid > FVV_MAX_GRIDS) {
    set_error("mesh: %d grids (1..%d)", ngrid, FVV_MAX_GRIDS);
    return FVV_E_LIMIT;
  }
  memset(&G, 0, sizeof(G));
  G.ngrid = ngrid;
  int64_t acc = 0, tr = 0;
  for (int g = 0; g < ngrid; ++g) {
    G.tw_start[g] = acc;
    acc += mesh_grid_info(grids[g], word_off[g], acc, G.gi[g]);
    G.gi[g].tr_off = tr;
    tr += mesh_grid_tr_items(G.gi[g]);
    if (3 * acc >= (int64_t)1 << 31) {  // 32-bit word indices (and int32 vertex prefixes)
      set_error("mesh: %lld occupancy words over the batch (limit %lld)", (long long)acc,
                (long long)((((int64_t)1 << 31) - 1) / 3));
      return FVV_E_LIMIT;
    }
  }
  for (int g = ngrid; g <= FVV_MAX_GRIDS; ++g) G.tw_start[g] = acc;
  G.tw_total = acc;
  G.tw3 = 3 * acc;
  G.tr_total = tr;
  return FVV_OK;
}

static int64_t words_of(const fvv_grid *grids, int ngrid) {
  int64_t acc = 0;
  for (int g = 0; g < ngrid; ++g) {
    const int64_t nx = grids[g].dims[0], ny = grids[g].dims[1], nz = grids[g].dims[2];
    if (nx >= 2 && ny >= 2 && nz >= 2) acc += nx * ny * ((nz + 31) / 32);
  }
  return acc;
}

size_t fvv::mesh_ws_bytes(int64_t tw_cap, int ngrid_max) {
  return prep_layout(tw_cap, ngrid_max).total;
}

int64_t *fvv::mesh_ws_totals(void *ws, int64_t tw_cap, int ngrid_max) {
  return (int64_t *)((char *)ws + prep_layout(tw_cap, ngrid_max).totals);
}

int64_t *fvv::mesh_ws_info(void *ws, int64_t tw_cap, int ngrid_max) {
  return (int64_t *)((char *)ws + prep_layout(tw_cap, ngrid_max).info);
}

int fvv::mesh_prepare_batch(const MeshGrids *G_dev, int64_t tw_cap, int ngrid_max,
                            const uint32_t *occ_dev, void *ws_dev, size_t ws_bytes,
                            cudaStream_t st, cudaStream_t side, cudaEvent_t fork,
                            cudaEvent_t join, void *scratch_dev, int64_t cap_v, int64_t cap_s) {
  int rc = ensure_tables();
  if (rc) return rc;
  const PrepLayout L = prep_layout(tw_cap, ngrid_max);
  if (ws_bytes < L.total) {
    set_error("fvv_mesh_prepare: workspace %zu < %zu bytes", ws_bytes, L.total);
    return FVV_E_ARG;
  }
  MeshBufs B = bufs_from(ws_dev, L);
  B.occ = occ_dev;
  // one fill clears both scans' status words and the totals (contiguous:
  // sums, sums2, totals) when the two scans run side by side
  // with the scans side by side, the transpose kernel clears both scans'
  // status words and the totals (contiguous: sums, sums2, totals; no fill
  // launch on the chain)
  const bool one_fill = side && tw_cap > 0;
  if (one_fill) {
    B.zero = (uint4 *)B.sums;
    B.zero_n = (int64_t)(((char *)B.totals - (char *)B.sums) + 32 + 15) / 16;
  } else {
    fill_async(B.totals, 0, 32, st);
  }
  if (tw_cap > 0) {
    launch_k(mesh_transpose_kernel, kMeshGrid, 256, 0, st, G_dev, B);
    note_launches(1);
    // the vertex and surface-cell scans read the same k-rows only: with a
    // side stream they run side by side (own scan status words each)
    if (side) {
      cudaEventRecord(fork, st);
      cudaStreamWaitEvent(side, fork, 0);
    }
    // with a phase-B scratch, the scans also write the vertex and cell lists
    const ScratchLayout SL = scratch_layout(scratch_dev, cap_v, cap_s);
    if (side && scratch_dev && cap_s > 0)  // the triangle scan's status words, off the main chain
      fill_async(SL.cell_sums, 0, onepass_bytes<Slot5>(cap_s + 1), side);
    CellFlags cf{G_dev, B.tw, B.sflags, B.sprefix, scratch_dev ? SL.cell_key : nullptr, cap_s};
    onepass_scan(cf, &G_dev->tw_total, 0, tw_cap, (void *)(side ? B.sums2 : B.sums),
                 B.totals + 1, side ? side : st, one_fill);
    if (side) cudaEventRecord(join, side);
    EdgeFlags ef{G_dev, B.tw, B.eflags, B.vprefix, scratch_dev ? SL.vert_key : nullptr, cap_v};
    onepass_scan(ef, &G_dev->tw3, 0, 3 * tw_cap, (void *)B.sums, B.totals + 0, st, one_fill);
    if (side) cudaStreamWaitEvent(st, join, 0);
  }
  if (!scratch_dev) {  // (fvv_mesh_counts reads them; device-planned C: the slot-bases launch)
    launch_k(mesh_grid_counts_kernel, 1, 128, 0, st, G_dev, B);
    note_launches(1);
  }
  return cuda_check("fvv_mesh_prepare");
}

size_t fvv::mesh_emit_scratch(int64_t cap_v, int64_t cap_s) {
  return scratch_layout(nullptr, cap_v, cap_s).total;
}

int fvv::mesh_emit_batch(const fvv_camera *cams_by_id, int ncam, const uint32_t *sil_dev,
                         const int64_t *sil_word_off, const MeshGrids *G_dev, int64_t tw_cap,
                         int ngrid_max, int exact, double fixed_iso, void *ws_dev,
                         size_t ws_bytes, int64_t cap_v, int64_t cap_s, void *scratch_dev,
                         size_t scratch_bytes, double *verts_dev, int32_t *tris_dev,
                         cudaStream_t st, bool fused, bool side_cleared) {
  int rc = ensure_tables();
  if (rc) return rc;
  if (exact && (ncam < 1 || ncam > FVV_MAX_CAMS)) {
    set_error("fvv_mesh_emit: %d cameras (1..%d)", ncam, FVV_MAX_CAMS);
    return FVV_E_LIMIT;
  }
  const PrepLayout L = prep_layout(tw_cap, ngrid_max);
  if (ws_bytes < L.total || scratch_bytes < mesh_emit_scratch(cap_v, cap_s)) {
    set_error("fvv_mesh_emit: workspace/scratch too small");
    return FVV_E_ARG;
  }
  MeshBufs B = bufs_from(ws_dev, L);
  const ScratchLayout SL = scratch_layout(scratch_dev, cap_v, cap_s);
  B.vert_key = SL.vert_key;
  B.cell_key = SL.cell_key;
  B.cell_tri = SL.cell_tri;
  B.cell_mask = SL.cell_mask;
  B.cprefix = SL.cprefix;
  Slot5 *cell_sums = SL.cell_sums;
  B.verts = verts_dev;
  B.tris = tris_dev;
  B.cap_v = cap_v;
  B.cap_s = cap_s;
  static thread_local MeshCams h_cams;
  memset(&h_cams, 0, sizeof(h_cams));
  h_cams.ncam = exact ? ncam : 0;
  for (int c = 0; c < h_cams.ncam; ++c) {
    h_cams.cams[c] = cams_by_id[c];
    h_cams.sil_off[c] = sil_word_off[c];
    h_cams.sil_stride[c] = sil_stride_words(cams_by_id[c].width);
  }
  Slot5 *d_total = (Slot5 *)((char *)ws_dev + L.slot5 + sizeof(int64_t) * 5 * ngrid_max);
  if (cap_v > 0) {
    if (!fused) launch_k(mesh_vertex_list_kernel, kMeshGrid, 256, 0, st, G_dev, B);
    // one vertex per thread, cameras in a loop; measured against (vertex,
    // camera) lane groups and a certified-FP32 endpoint projection with the
    // float64 terms deferred to full warps, both slower
    const int64_t lam_blocks = std::min<int64_t>(cap_v / 128 + 1, 148 * 64);
    launch_k(mesh_lambda_kernel, (unsigned)lam_blocks, 128, 0, st, G_dev, h_cams, B, sil_dev, exact,
                                                              fixed_iso);
    note_launches(fused ? 1 : 2);
  }
  if (cap_s > 0 && fused) {  // the cells evaluated inside the triangle scan
    TriCells tc{G_dev, B};
    // (status words cleared on the side stream during C's scans when
    // mesh_prepare_batch ran with one)
    onepass_scan(tc, B.totals + 3, 0, cap_s, (void *)cell_sums, d_total, st, side_cleared);
  } else if (cap_s > 0) {
    const int64_t cell_blocks = std::min<int64_t>(tw_cap / 256 + 1, 148 * 64);
    launch_k(mesh_cells_kernel, (unsigned)std::max<int64_t>(cell_blocks, kMeshGrid), 256, 0, st, G_dev,
                                                                                          B);
    note_launches(1);
    TriScan ts{B.cell_mask, B.cprefix};
    onepass_scan(ts, B.totals + 3, 0, cap_s, (void *)cell_sums, d_total, st);
  } else {
    fill_async(d_total, 0, sizeof(Slot5), st);
  }
  if (cap_s > 0 && fused) {  // the emit blocks compute the slot bases themselves
    launch_k(mesh_emit_kernel<true>, kMeshGrid, 256, 0, st, G_dev, B, (const Slot5 *)d_total);
    note_launches(1);
  } else {
    launch_k(mesh_slot_bases_kernel, 1, 32, 0, st, G_dev, B, (const Slot5 *)d_total);
    if (cap_s > 0) launch_k(mesh_emit_kernel<false>, kMeshGrid, 256, 0, st, G_dev, B,
                            (const Slot5 *)d_total);
    note_launches(1 + (cap_s > 0 ? 1 : 0));
  }
  return cuda_check("fvv_mesh_emit");
}

extern "C" {

size_t fvv_mesh_workspace_bytes(const fvv_grid *grids, int ngrid) {
  return prep_layout(words_of(grids, ngrid), ngrid).total;
}

int fvv_mesh_prepare(const fvv_grid *grids, int ngrid, const uint32_t *occ_dev,
                     const int64_t *word_off, void *ws_dev, size_t ws_bytes, void *stream) {
  static thread_local MeshGrids G;
  int rc = fill_grids(grids, ngrid, word_off, G);
  if (rc) return rc;
  const PrepLayout L = prep_layout(G.tw_total, ngrid);
  if (ws_bytes < L.total) {
    set_error("fvv_mesh_prepare: workspace %zu < %zu bytes", ws_bytes, L.total);
    return FVV_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  MeshGrids *G_dev = (MeshGrids *)((char *)ws_dev + L.grids);
  launch_k(store_mesh_grids_kernel, 1, 256, 0, st, G, G_dev);
  note_launches(1);
  return mesh_prepare_batch(G_dev, G.tw_total, ngrid, occ_dev, ws_dev, ws_bytes, st, nullptr,
                            nullptr, nullptr, nullptr, 0, 0);
}

// Reads the counts fvv_mesh_prepare left in the workspace: totals[3] = {V, S, T}
// and info[ngrid][8] (vbase V sbase S tbase T fallback inconsistent).
int fvv_mesh_counts(const fvv_grid *grids, int ngrid, const void *ws_dev, int64_t *totals_dev,
                    int64_t *info_dev, void *stream) {
  const PrepLayout L = prep_layout(words_of(grids, ngrid), ngrid);
  cudaStream_t st = (cudaStream_t)stream;
  if (totals_dev)
    cudaMemcpyAsync(totals_dev, (const char *)ws_dev + L.totals, 3 * sizeof(int64_t),
                    cudaMemcpyDeviceToDevice, st);
  if (info_dev)
    cudaMemcpyAsync(info_dev, (const char *)ws_dev + L.info, 8 * sizeof(int64_t) * ngrid,
                    cudaMemcpyDeviceToDevice, st);
  return cuda_check("fvv_mesh_counts");
}

size_t fvv_mesh_emit_scratch_bytes(int64_t num_vertices, int64_t num_cells) {
  return mesh_emit_scratch(num_vertices, num_cells);
}

// Phase B of the batch fvv_mesh_prepare set up in ws_dev (its grid table and
// counts); grids / word_off must be the same as there.
int fvv_mesh_emit(const fvv_camera *cams_by_id, int ncam, const uint32_t *sil_dev,
                  const int64_t *sil_word_off, const fvv_grid *grids, int ngrid,
                  const uint32_t *occ_dev, const int64_t *word_off, int exact, double fixed_iso,
                  void *ws_dev, size_t ws_bytes, int64_t num_vertices, int64_t num_cells,
                  void *scratch_dev, size_t scratch_bytes, double *verts_dev, int32_t *tris_dev,
                  void *stream) {
  (void)occ_dev;
  (void)word_off;
  if (ngrid < 1 || ngrid > FVV_MAX_GRIDS) {
    set_error("mesh: %d grids (1..%d)", ngrid, FVV_MAX_GRIDS);
    return FVV_E_LIMIT;
  }
  const int64_t tw = words_of(grids, ngrid);
  const PrepLayout L = prep_layout(tw, ngrid);
  return mesh_emit_batch(cams_by_id, ncam, sil_dev, sil_word_off,
                         (const MeshGrids *)((char *)ws_dev + L.grids), tw, ngrid, exact,
                         fixed_iso, ws_dev, ws_bytes, num_vertices, num_cells, scratch_dev,
                         scratch_bytes, verts_dev, tris_dev, (cudaStream_t)stream, false);
}

int fvv_edge_isovalues(const fvv_camera *cams_by_id, int ncam, const uint32_t *sil_dev,
                       const int64_t *sil_word_off, const double *p_on_dev,
                       const double *p_off_dev, int64_t n, double *lam_dev, int32_t *cam_dev,
                       int64_t *stats_dev, void *stream) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("fvv_edge_isovalues: %d cameras (1..%d)", ncam, FVV_MAX_CAMS);
    return FVV_E_LIMIT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  fill_async(stats_dev, 0, 2 * sizeof(int64_t), st);
  if (n <= 0) return cuda_check("fvv_edge_isovalues");
  static thread_local MeshCams h_cams;
  memset(&h_cams, 0, sizeof(h_cams));
  h_cams.ncam = ncam;
  for (int c = 0; c < ncam; ++c) {
    h_cams.cams[c] = cams_by_id[c];
    h_cams.sil_off[c] = sil_word_off[c];
    h_cams.sil_stride[c] = sil_stride_words(cams_by_id[c].width);
  }
  int64_t blocks = (n + 127) / 128;
  if (blocks > kMeshGrid) blocks = kMeshGrid;
  launch_k(edge_isovalues_kernel, (int)blocks, 128, 0, st, h_cams, sil_dev, p_on_dev, p_off_dev, n,
                                                      lam_dev, cam_dev, stats_dev);
  note_launches(1);
  return cuda_check("fvv_edge_isovalues");
}

}  // extern "C"
