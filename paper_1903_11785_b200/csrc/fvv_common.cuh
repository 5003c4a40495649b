// Shared device helpers: the reference's float64 projection chain, bit
// lookups, error plumbing. Every kernel TU is compiled with -fmad=false, so
// `a*b + c` below rounds twice exactly like numpy; fma() is written out
// only where the reference goes through OpenBLAS.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../include/fvv.h"

namespace fvv {

constexpr int kCarveChunk = 1 << 20;  // hull.py:20 CARVE_CHUNK
constexpr double kNearClip = 1.0;     // visibility.py:19 NEAR_CLIP_MM
constexpr double kDegenerateArea = 1e-9;  // mesh.py:22

void set_error(const char *fmt, ...);
int cuda_check(const char *what);
// kernels launched by this library (bench.py reports the timed-region delta)
void note_launches(long long n);
// kernels this host thread has launched (lanes capture their frame graphs
// concurrently: a capture counts its own launches with this)
long long thread_launch_count();

// Programmatic dependent launch: every kernel is launched with the
// programmatic-serialisation attribute and waits for its predecessor's
// completion (griddepcontrol.wait, a no-op without one) before it touches
// memory, so a launch's setup and block scheduling overlap the previous
// kernel's tail - inside a captured frame graph too. FVV_PDL=0 turns it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

// fvv_frame_run split for pipelined callers (frame.cu): frame_begin launches
// a graph replay without waiting (*async) or runs the frame to completion;
// frame_end completes a begun frame; frame_launched_event is the event
// recorded after the begun frame's launch.
int frame_begin(fvv_frame *f, const uint8_t *masks_dev, const fvv_camera *virt,
                const int32_t *rank_pos, const uint8_t *frames_dev, const int64_t *frame_off,
                const uint8_t *fallback, void *stream, fvv_frame_stats *out_stats, int *out_stage,
                bool *async);
int frame_end(fvv_frame *f, fvv_frame_stats *out_stats, int *out_stage);
cudaEvent_t frame_launched_event(const fvv_frame *f);

// cudaMemsetAsync(p, value, bytes, st) as a programmatic-dependent kernel (api.cu)
void fill_async(void *p, int value, size_t bytes, cudaStream_t st);

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<Args &&>(args)...);
}

// camera.py:177 `pts @ R.T + t`: OpenBLAS gemm (>= 2 rows) accumulates
// fma(z,R2, fma(y,R1, x*R0)); the 1-row gemv kernel fma(z,R2, fma(x,R0, y*R1)).
// (the two orders differ only in which product is fused: the first factor
// pair of each row is selected, so one product and one fma are evaluated)
__device__ __forceinline__ void world_to_cam(const fvv_camera &c, double x, double y, double z,
                                             bool gemv, double &X, double &Y, double &Z) {
  const double m = gemv ? y : x, f = gemv ? x : y;  // m * R[m-col] first, then fma(f, ...)
  const int cm = gemv ? 1 : 0, cf = gemv ? 0 : 1;
  const double a0 = fma(f, c.R[cf], m * c.R[cm]);
  const double a1 = fma(f, c.R[3 + cf], m * c.R[3 + cm]);
  const double a2 = fma(f, c.R[6 + cf], m * c.R[6 + cm]);
  X = fma(z, c.R[2], a0) + c.t[0];
  Y = fma(z, c.R[5], a1) + c.t[1];
  Z = fma(z, c.R[8], a2) + c.t[2];
}

// camera.py:164-201 project() + camera.py:154-161 distort(), float64, in the
// reference's evaluation order. Returns in_frustum; u, v unrounded pixel.
__device__ __forceinline__ bool project_exact(const fvv_camera &c, double x, double y, double z,
                                              bool use_dist, bool gemv, double &u, double &v,
                                              double &zc) {
  double X, Y, Z;
  world_to_cam(c, x, y, z, gemv, X, Y, Z);
  double sz = (Z != 0.0) ? Z : 1.0;
  double xn = X / sz;
  double yn = Y / sz;
  double xd = xn, yd = yn;
  if (use_dist && c.has_distortion) {
    double r2 = xn * xn + yn * yn;
    double radial = 1.0 + r2 * (c.k1 + r2 * (c.k2 + r2 * c.k3));
    xd = xn * radial + 2.0 * c.p1 * xn * yn + c.p2 * (r2 + 2.0 * xn * xn);
    yd = yn * radial + c.p1 * (r2 + 2.0 * yn * yn) + 2.0 * c.p2 * xn * yn;
  }
  u = c.fx * (xd + c.skew * yd) + c.cx;
  v = c.fy * yd + c.cy;
  zc = Z;
  double iu = rint(u), iv = rint(v);  // np.rint: round half to even
  return (Z > 0.0) && (iu >= 0.0) && (iu <= (double)(c.width - 1)) && (iv >= 0.0) &&
         (iv <= (double)(c.height - 1));
}

// rint(u), rint(v) and the in-frustum flag of project_exact(use_dist=false)
// without the two float64 divisions in the common case: X/sz and Y/sz are
// replaced by products with a Newton-refined reciprocal (a few ulps off),
// and the result is kept only when u and v are farther than a generous bound
// (~1e-12 relative, vs ~1e-15 actual) from a rounding boundary, where it
// cannot differ from the exact chain's rint. Otherwise (and for NaN) the
// exact divisions run. Z is the exact camera-space depth either way.
__device__ __forceinline__ bool project_rint(const fvv_camera &c, double x, double y, double z,
                                             bool gemv, double &iu, double &iv, double &zc) {
  double X, Y, Z;
  world_to_cam(c, x, y, z, gemv, X, Y, Z);
  zc = Z;
  const double sz = (Z != 0.0) ? Z : 1.0;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(sz));
  r = fma(r, fma(-sz, r, 1.0), r);
  r = fma(r, fma(-sz, r, 1.0), r);
  const double xn = X * r, yn = Y * r;
  const double s = xn + c.skew * yn;
  double u = c.fx * s + c.cx;
  double v = c.fy * yn + c.cy;
  const double eu = 1e-12 * (fabs(c.fx) * (fabs(xn) + fabs(c.skew * yn)) + fabs(u) + fabs(c.cx) + 1.0);
  const double ev = 1e-12 * (fabs(c.fy * yn) + fabs(v) + fabs(c.cy) + 1.0);
  iu = rint(u);
  iv = rint(v);
  if (!(fabs(u - iu) < 0.5 - eu && fabs(v - iv) < 0.5 - ev)) {  // near a tie (or NaN): exact
    const double xe = X / sz, ye = Y / sz;
    u = c.fx * (xe + c.skew * ye) + c.cx;
    v = c.fy * ye + c.cy;
    iu = rint(u);
    iv = rint(v);
  }
  return (Z > 0.0) && (iu >= 0.0) && (iu <= (double)(c.width - 1)) && (iv >= 0.0) &&
         (iv <= (double)(c.height - 1));
}

// project_rint with the perspective division in FP32: the float64 chain's
// X, Y, Z (exact Z: the depth test needs it), then u, v from their float
// roundings with one reciprocal, kept when u and v lie farther than a
// rigorous bound from a rounding boundary; the float64 divisions otherwise
// (near a tie, |u| >= 2^22, tiny Z). Bound: with unit roundoff eps = 2^-24,
// X/Y/Z to float (eps each), the refined reciprocal (2 eps), the products
// give xn, yn within 5 eps; skew * yn 7 eps; their sum 8 eps of
// (|xn| + |syn|); fx (float) times it 10 eps of |fx| (|xn| + |syn|); + cx
// (eps |cx|) and the final rounding (eps |u|): |u32 - u| <= 10 eps M with
// M = |fx| (|xn| + |syn|) + |cx| + |u|. 2^-20 M is 1.6x that (the float64
// chain's own ~1e-16 relative error and second-order terms are far below).
__device__ __forceinline__ float recip32(float z) {
  const float r = __fdividef(1.0f, z);
  return fmaf(r, fmaf(-z, r, 1.0f), r);
}

// The FP32 constants of project_rint32 for one camera (once per block).
struct CamF32 {
  float fx, fy, cx, cy, sk;
  int width, height;
};
__device__ __forceinline__ CamF32 cam_f32(const fvv_camera &c) {
  return CamF32{(float)c.fx, (float)c.fy, (float)c.cx, (float)c.cy, (float)c.skew, c.width,
                c.height};
}

// Returns in_frustum; (ix, iy) = the rounded pixel when in frustum.
__device__ __forceinline__ bool project_rint32(const fvv_camera &c, const CamF32 &f, double x,
                                               double y, double z, bool gemv, int &ix, int &iy,
                                               double &zc) {
  double X, Y, Z;
  world_to_cam(c, x, y, z, gemv, X, Y, Z);
  zc = Z;
  if (!(Z > 0.0)) return false;  // (the float64 chain's frustum test needs Z > 0 too)
  const float Zf = (float)Z, Xf = (float)X, Yf = (float)Y;
  bool ok = Zf > 1e-30f;
  const float r = recip32(ok ? Zf : 1.0f);
  const float xn = Xf * r, yn = Yf * r;
  const float syn = f.sk * yn;
  const float su = f.fx * (xn + syn), sv = f.fy * yn;
  const float u = su + f.cx, v = sv + f.cy;
  const float eu = 0x1p-20f * (fabsf(f.fx) * (fabsf(xn) + fabsf(syn)) + fabsf(f.cx) + fabsf(u) + 1.0f);
  const float ev = 0x1p-20f * (fabsf(sv) + fabsf(f.cy) + fabsf(v) + 1.0f);
  const float ru = rintf(u), rv = rintf(v);
  ok = ok && fabsf(u) < 4194304.0f && fabsf(v) < 4194304.0f && fabsf(u - ru) < 0.5f - eu &&
       fabsf(v - rv) < 0.5f - ev;
  if (ok) {  // |ru|, |rv| < 2^22
    ix = (int)ru;
    iy = (int)rv;
    return ix >= 0 && ix < f.width && iy >= 0 && iy < f.height;
  }
  // the float64 chain (project_exact, no distortion)
  const double xe = X / Z, ye = Y / Z;
  const double iu = rint(c.fx * (xe + c.skew * ye) + c.cx), iv = rint(c.fy * ye + c.cy);
  if (!((iu >= 0.0) && (iu <= (double)(c.width - 1)) && (iv >= 0.0) &&
        (iv <= (double)(c.height - 1))))
    return false;
  ix = (int)iu;
  iy = (int)iv;
  return true;
}

// voxels.py:52-56 voxel centre.
__device__ __forceinline__ void voxel_center(const fvv_grid &g, int64_t i, int64_t j, int64_t k,
                                             double &x, double &y, double &z) {
  x = g.origin[0] + g.spacing * ((double)i + 0.5);
  y = g.origin[1] + g.spacing * ((double)j + 0.5);
  z = g.origin[2] + g.spacing * ((double)k + 0.5);
}

__device__ __forceinline__ bool sil_bit(const uint32_t *__restrict__ plane, int stride_words,
                                        int x, int y) {
  uint32_t w = __ldg(plane + (int64_t)y * stride_words + (x >> 5));
  return (w >> (x & 31)) & 1u;
}

__host__ __device__ inline int sil_stride_words(int width) { return (width + 31) >> 5; }

// Element count produced on the device by an earlier launch, else the host
// value. (A `p ? *p : fallback` select on a __grid_constant__ member makes
// nvcc form a generic pointer into parameter space; keep it a value select.)
__device__ __forceinline__ int64_t device_count(const int64_t *p, int64_t fallback) {
  int64_t v = fallback;
  if (p != nullptr) v = __ldcg(p);
  return v;
}

// Per-frame input pointers of a device-planned (graph-captured) frame, read
// by the kernels from device memory so one captured frame serves new inputs:
// the masks (pack) and the colour frames (render), camera c's frame at
// frames + frame_off[c].
struct __align__(16) FrameInputs {
  const uint8_t *masks;
  const uint8_t *frames;
  int64_t frame_off[FVV_MAX_CAMS];
};

// fvv_pack_silhouettes / fvv_render_view_coded with the masks / frames
// pointers taken from *in (device) when in is non-null (masks_dev, frames_dev
// and frame_off then only describe the alignment and the camera set).
int pack_silhouettes_bound(const fvv_camera *cams, int ncam, const uint8_t *masks_dev,
                           const FrameInputs *in, const int64_t *mask_off, uint32_t *sil_dev,
                           const int64_t *sil_word_off, cudaStream_t st);
int render_view_coded_bound(const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                            const int64_t *frame_off, const FrameInputs *in,
                            const fvv_camera *virt, const double *depth_dev,
                            const int32_t *tri_id_dev, const int32_t *tri_src_dev,
                            const uint8_t *fallback, uint8_t *color_dev, int32_t *source_dev,
                            uint8_t *covered_dev, int8_t *code_dev, const int64_t *counts_dev,
                            cudaStream_t st);

// fvv_classify, plus (src_dev non-null) fvv_triangle_sources fused into it:
// src_dev[t] = rank_id[r] of the first r with triangle t visible in rig
// camera rank_pos[r], -1 if none.
int classify_sources(const fvv_camera *cams, int ncam, const double *verts_dev,
                     const int32_t *tris_dev, int64_t nt, const int64_t *nt_dev,
                     const double *depth_dev, const int64_t *plane_off, double t_v,
                     uint32_t *vis_dev, int64_t vis_stride_words, int nrank,
                     const int32_t *rank_pos, const int32_t *rank_id, int32_t *src_dev,
                     cudaStream_t st);

// Grid table of one batched carve launch, in device memory (written by the
// host wrapper's store launch, or on the device by the frame planner):
// block b of the tile kernels carves tile b - blk_start[g] of the grid g
// with blk_start[g] <= b < blk_start[g + 1].
struct __align__(16) CarveGrids {
  int ngrid, tile_log2;
  int64_t total_tiles;  // blk_start[ngrid]
  fvv_grid grids[FVV_MAX_GRIDS];
  int64_t word_off[FVV_MAX_GRIDS];
  int64_t blk_start[FVV_MAX_GRIDS + 1];
  uint32_t tiles_x[FVV_MAX_GRIDS], tiles_y[FVV_MAX_GRIDS];
};

// Tiles of a grid at tile edge 1 << tl; false when the grid has no voxels.
__host__ __device__ inline bool carve_grid_tiles(const fvv_grid &g, int tl, uint32_t &tx,
                                                 uint32_t &ty, int64_t &tiles) {
  const int64_t kT = (int64_t)1 << tl;
  if (g.dims[0] <= 0 || g.dims[1] <= 0 || g.dims[2] <= 0) return false;
  tx = (uint32_t)((g.dims[0] + kT - 1) / kT);
  ty = (uint32_t)((g.dims[1] + kT - 1) / kT);
  tiles = (int64_t)tx * ty * ((g.dims[2] + kT - 1) / kT);
  return true;
}

// B-1 / B-3 carve of the grids in *gt (device) - the body of fvv_carve.
// ngrid_max bounds gt->ngrid and blocks_cap the tile count (device-planned
// batches: capacities; blocks past gt->total_tiles exit).
int carve_batch(const fvv_camera *cams, int ncam, const uint32_t *sil_dev,
                const int64_t *sil_word_off, const CarveGrids *gt_dev, int ngrid_max,
                int tile_log2, int64_t blocks_cap, int min_views, uint32_t *occ_dev,
                int64_t *count_dev, void *workspace, size_t ws_bytes, cudaStream_t st,
                bool reuse_cells = false);  // cell maps left by the previous carve of these planes
size_t carve_grids_offset(const fvv_camera *cams, int ncam);  // table slot in the workspace

// Grid table of one batched polygonize (mesh.cu), in device memory: grid g's
// occupancy transposed into k-rows occupies words [tw_start[g], tw_start[g+1]).
struct MeshGridInfo {
  fvv_grid g;
  int64_t occ_word_off;  // F-order occupancy words of this grid
  int64_t rows, nzw;     // rows = nx*ny (0 when a dim < 2: empty mesh, mesh.py:298-299)
  int64_t tw_off;        // transposed-word offset (S space); V space offset = 3*tw_off
  int64_t tr_off;        // first transpose work item (32 i x one k-row word)
  uint32_t words32, nzw32, ny32, nxw32;  // rows*nzw, nzw, ny, ceil(nx/32) (3*tw_total < 2^31)
};

struct __align__(16) MeshGrids {
  int ngrid, pad;
  int64_t tw_total, tw3;  // k-row words of the batch, and 3x (the edge scan's length)
  int64_t tr_total;       // transpose work items of the batch
  int64_t tw_start[FVV_MAX_GRIDS + 1];  // prefix of rows*nzw
  MeshGridInfo gi[FVV_MAX_GRIDS];
};

// grid info at k-row word offset acc; returns the grid's k-row words
__host__ __device__ inline int64_t mesh_grid_info(const fvv_grid &g, int64_t word_off,
                                                  int64_t acc, MeshGridInfo &gi) {
  gi.g = g;
  gi.occ_word_off = word_off;
  const int64_t nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
  const bool meshable = nx >= 2 && ny >= 2 && nz >= 2;  // mesh.py:298-299
  gi.rows = meshable ? nx * ny : 0;
  gi.nzw = meshable ? (nz + 31) / 32 : 1;
  gi.tw_off = acc;
  gi.words32 = (uint32_t)(gi.rows * gi.nzw);
  gi.nzw32 = (uint32_t)gi.nzw;
  gi.ny32 = (uint32_t)ny;
  gi.nxw32 = meshable ? (uint32_t)((nx + 31) / 32) : 0;
  gi.tr_off = 0;
  return gi.rows * gi.nzw;
}

// transpose work items of a grid (one per 32 i of a k-row word)
__host__ __device__ inline int64_t mesh_grid_tr_items(const MeshGridInfo &gi) {
  return (int64_t)gi.nxw32 * gi.ny32 * gi.nzw32;
}

// C polygonize of the grids in *G_dev (device) - the bodies of
// fvv_mesh_prepare / fvv_mesh_emit. tw_cap / ngrid_max bound the batch's
// k-row words and grids (the workspace layout); cap_v / cap_s the vertex and
// surface-cell counts phase B has room for (a batch beyond them skips phase B).
size_t mesh_ws_bytes(int64_t tw_cap, int ngrid_max);
int64_t *mesh_ws_totals(void *ws, int64_t tw_cap, int ngrid_max);  // V, S, T
int64_t *mesh_ws_info(void *ws, int64_t tw_cap, int ngrid_max);    // [ngrid][8]
int mesh_prepare_batch(const MeshGrids *G_dev, int64_t tw_cap, int ngrid_max,
                       const uint32_t *occ_dev, void *ws_dev, size_t ws_bytes, cudaStream_t st,
                       cudaStream_t side = nullptr, cudaEvent_t fork = nullptr,
                       cudaEvent_t join = nullptr, void *scratch_dev = nullptr,
                       int64_t cap_v = 0, int64_t cap_s = 0);  // scratch: also list keys
size_t mesh_emit_scratch(int64_t cap_v, int64_t cap_s);
int mesh_emit_batch(const fvv_camera *cams_by_id, int ncam, const uint32_t *sil_dev,
                    const int64_t *sil_word_off, const MeshGrids *G_dev, int64_t tw_cap,
                    int ngrid_max, int exact, double fixed_iso, void *ws_dev, size_t ws_bytes,
                    int64_t cap_v, int64_t cap_s, void *scratch_dev, size_t scratch_bytes,
                    double *verts_dev, int32_t *tris_dev, cudaStream_t st,
                    bool fused = false,  // fused: prepare wrote the vertex / cell lists
                    bool side_cleared = false);  // prepare (with a side stream) cleared the
                                                 // triangle scan's status words

}  // namespace fvv
