// Native per-frame executor: the whole hot path of pipeline.py:115-220
// (B-1 .. D-2) plus one render_view colour pass (render.py:64-113) driven
// from C++ on one CUDA stream, with device buffers that persist across
// frames (grown on demand, never freed between frames).
//
// The host work the reference does between its kernels is reproduced here
// with the same IEEE double arithmetic: GridSpec.from_aabb (voxels.py:62-71),
// the noise band filter (hull.py:46-47, 257-269) and extract_rois
// (hull.py:272-284). Three host synchronisations per frame remain, each a
// tiny pinned read: the component table (to size the ROI grids), the mesh
// vertex/cell counts (to size the mesh outputs) and the final counters.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <vector>

#include "fvv_common.cuh"

extern "C" {
int fvv_render_view_coded(const fvv_camera *, int, const uint8_t *, const int64_t *,
                          const fvv_camera *, const double *, const int32_t *, const int32_t *,
                          const uint8_t *, uint8_t *, int32_t *, uint8_t *, int8_t *,
                          const int64_t *, void *);
int fvv_pack_silhouettes(const fvv_camera *, int, const uint8_t *, const int64_t *, uint32_t *,
                         const int64_t *, void *);
int fvv_carve(const fvv_camera *, int, const uint32_t *, const int64_t *, const fvv_grid *, int,
              const int64_t *, int, uint32_t *, int64_t *, void *, size_t, void *);
size_t fvv_carve_workspace_bytes(const fvv_camera *, int);
size_t fvv_ccl_workspace_bytes(const fvv_grid *);
int fvv_ccl26(const uint32_t *, const fvv_grid *, void *, size_t, fvv_component *, int64_t,
              int64_t *, void *);
int fvv_ccl_components(const fvv_grid *, const void *, fvv_component *, int64_t, void *);
size_t fvv_mesh_workspace_bytes(const fvv_grid *, int);
int fvv_mesh_prepare(const fvv_grid *, int, const uint32_t *, const int64_t *, void *, size_t,
                     void *);
int fvv_mesh_counts(const fvv_grid *, int, const void *, int64_t *, int64_t *, void *);
size_t fvv_mesh_emit_scratch_bytes(int64_t, int64_t);
int fvv_mesh_emit(const fvv_camera *, int, const uint32_t *, const int64_t *, const fvv_grid *,
                  int, const uint32_t *, const int64_t *, int, double, void *, size_t, int64_t,
                  int64_t, void *, size_t, double *, int32_t *, void *);
size_t fvv_raster_workspace_bytes(int64_t, int64_t, int);
int fvv_rasterize(const fvv_camera *, int, const double *, int64_t, const int32_t *, int64_t,
                  const int64_t *, double *, const int64_t *, int32_t *, void *, size_t, void *);
int fvv_rasterize_tracked(const fvv_camera *, int, const double *, int64_t, const int64_t *,
                          const int32_t *, int64_t, const int64_t *, double *, const int64_t *,
                          int32_t *, void *, size_t, uint8_t *, int, void *);
int fvv_classify(const fvv_camera *, int, const double *, const int32_t *, int64_t,
                 const int64_t *, const double *, const int64_t *, double, uint32_t *, int64_t,
                 void *);
int fvv_triangle_sources(const int32_t *, const int32_t *, int, const uint32_t *, int64_t, int64_t,
                         const int64_t *, int32_t *, void *);
int fvv_render_count(const fvv_camera *, int, const fvv_camera *, const int32_t *,
                     const int32_t *, int64_t *, void *);
int fvv_render_view(const fvv_camera *, int, const uint8_t *, const int64_t *,
                    const fvv_camera *, const double *, const int32_t *, const int32_t *,
                    const uint8_t *, uint8_t *, int32_t *, uint8_t *, const int64_t *, void *);
}

namespace fvv {

// device buffer that only grows
struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap && p) return FVV_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    // exact (rounded to 256 B): device-planned buffers come sized from
    // capacities that already carry headroom, the others are fixed per rig
    size_t want = (bytes + 255) & ~(size_t)255;
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      set_error("frame executor: cudaMalloc(%zu) failed", want);
      return FVV_E_CUDA;
    }
    cap = want;
    return FVV_OK;
  }
  // grow to >= bytes keeping the first `used` bytes (stream-ordered copy;
  // the cudaFree of the old block waits for it)
  int grow_keep(size_t bytes, size_t used, cudaStream_t st) {
    if (bytes <= cap && p) return FVV_OK;
    void *old = p;
    const size_t want = bytes + bytes / 4 + 256;
    void *np = nullptr;
    if (cudaMalloc(&np, want) != cudaSuccess) {
      cudaGetLastError();
      set_error("frame executor: cudaMalloc(%zu) failed", want);
      return FVV_E_CUDA;
    }
    if (old && used) cudaMemcpyAsync(np, old, used, cudaMemcpyDeviceToDevice, st);
    if (old) cudaFree(old);
    p = np;
    cap = want;
    return FVV_OK;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T *as() const {
    return (T *)p;
  }
};

__global__ void add_count_kernel(int64_t *dst, const int64_t *src, int64_t add) {
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) *dst = *src + add;
}

__global__ void offset_tris_kernel(int32_t *tris, int64_t n3, int32_t add) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n3;
       i += (int64_t)gridDim.x * blockDim.x)
    tris[i] += add;
}

// Small results reach the host without a copy engine: one kernel stores
// them straight into mapped pinned memory. (A cudaMemcpyAsync would queue
// behind the multi-MB frame transfers run_sequence keeps on the copy
// engines, stalling every host synchronisation of the next frame.)
struct ReadPiece {
  const int64_t *src;
  int64_t *dst;          // device alias of mapped host memory
  const int64_t *count;  // optional device element count (clamped to max_elems)
  int64_t words;         // words to copy when count == nullptr
  int64_t elem_words, max_elems;
};
constexpr int kReadPieces = 10;
struct ReadBatch {
  ReadPiece p[kReadPieces];
};

__global__ void readback_kernel(ReadBatch B) {
  pdl_wait();
  const int y = blockIdx.y;
  const int64_t *src = B.p[y].src;
  int64_t *dst = B.p[y].dst;
  int64_t w = B.p[y].words;
  if (B.p[y].count) {
    int64_t c = __ldcg(B.p[y].count);
    c = c < 0 ? 0 : (c > B.p[y].max_elems ? B.p[y].max_elems : c);
    w = c * B.p[y].elem_words;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
}

__global__ void bind_inputs_kernel(const __grid_constant__ FrameInputs v, FrameInputs *dst) {
  pdl_wait();
  const int4 *a = reinterpret_cast<const int4 *>(&v);
  int4 *b = reinterpret_cast<int4 *>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(FrameInputs) / 16); i += blockDim.x) b[i] = a[i];
}

// ---- device-side frame planning -------------------------------------------
// What the host does between B-2 and B-3 (the noise band filter, extract_rois
// and GridSpec.from_aabb, hull.py:46-47, 257-284, voxels.py:62-71), done on
// the device in the same IEEE double arithmetic, plus the B-3 carve and C
// polygonize grid tables, so a frame runs without a host round trip. Batches
// the planner does not take (more than FVV_MAX_GRIDS ROIs or 4096
// components, an ROI error, a capacity overflow) come back with a status and
// the host-planned path redoes the frame.
enum : int32_t { kPlanManyRois = 1, kPlanError = 2, kPlanCapacity = 4 };

struct __align__(16) FramePlan {
  int64_t status, nroi;  // (nroi: all ROIs of the band filter, may exceed FVV_MAX_GRIDS)
  int64_t dense_tests, fine_words;
  int64_t roi_component[FVV_MAX_GRIDS];
  double roi_box[FVV_MAX_GRIDS][6];
  CarveGrids carve;  // B-3 (16^3 tiles)
  MeshGrids mesh;    // C
};

struct PlanArgs {
  fvv_grid coarse;
  double roi_margin, fine_spacing, t_large;
  int64_t t_small, budget;
  int64_t comp_cap;  // component records in comps[]
  int64_t cap_words, cap_tiles, cap_tw;
};

constexpr int kPlanThreads = 1024;

__global__ void __launch_bounds__(kPlanThreads)
    frame_plan_kernel(const __grid_constant__ PlanArgs a, const fvv_component *__restrict__ comps,
                      const int64_t *__restrict__ ccl_counts, FramePlan *plan) {
  pdl_wait();
  __shared__ int s_warp[kPlanThreads / 32];
  __shared__ int s_nroi, s_status;
  __shared__ int64_t s_words[FVV_MAX_GRIDS], s_tiles[FVV_MAX_GRIDS], s_tw[FVV_MAX_GRIDS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ncomp = __ldcg(ccl_counts + 1);
  if (tid == 0) {
    s_nroi = 0;
    s_status = ncomp > a.comp_cap ? kPlanManyRois : 0;
  }
  __syncthreads();
  const fvv_grid &G = a.coarse;
  double extent[3];
  for (int j = 0; j < 3; ++j) extent[j] = G.origin[j] + G.spacing * (double)G.dims[j];
  const int64_t n = ncomp < a.comp_cap ? ncomp : a.comp_cap;
  // band filter + ROI boxes in component order (an ordered block scan per chunk)
  for (int64_t c0 = 0; c0 < n; c0 += kPlanThreads) {
    const int64_t c = c0 + tid;
    bool keep = false;
    if (c < n) {
      const double cnt = (double)comps[c].voxel_count;
      keep = (double)a.t_small <= cnt && cnt <= a.t_large;  // hull.py:46-47
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_warp[warp] = __popc(b);
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += s_warp[w];
    const int base = s_nroi;
    const int r = base + before + __popc(b & ((1u << lane) - 1u));
    if (keep && r < FVV_MAX_GRIDS) {
      const fvv_component &cp = comps[c];
      double lo[3], hi[3];
      bool ok = true;
      for (int j = 0; j < 3; ++j) {  // hull.py:279-282
        lo[j] = G.origin[j] + G.spacing * (double)cp.bbox_min[j] - a.roi_margin;
        hi[j] = G.origin[j] + G.spacing * ((double)cp.bbox_max[j] + 1.0) + a.roi_margin;
        lo[j] = lo[j] >= G.origin[j] ? lo[j] : G.origin[j];  // np.maximum(lo, stage_lo)
        hi[j] = hi[j] <= extent[j] ? hi[j] : extent[j];      // np.minimum(hi, stage_hi)
        ok = ok && lo[j] < hi[j];
      }
      // voxels.py:62-71 GridSpec.from_aabb (+ the budget check, voxels.py:34-37)
      fvv_grid fg;
      int64_t nv = 1;
      for (int j = 0; j < 3; ++j) {
        int64_t d = (int64_t)ceil((hi[j] - lo[j]) / a.fine_spacing - 1e-9);
        d = d < 1 ? 1 : d;
        fg.origin[j] = lo[j];
        fg.dims[j] = d;
        nv *= d;
      }
      fg.spacing = a.fine_spacing;
      if (!ok || nv > a.budget) atomicOr(&s_status, kPlanError);
      plan->roi_component[r] = cp.id;
      for (int j = 0; j < 3; ++j) {
        plan->roi_box[r][j] = lo[j];
        plan->roi_box[r][3 + j] = hi[j];
      }
      plan->carve.grids[r] = fg;
      s_words[r] = (nv + 31) / 32;
      uint32_t tx, ty;
      int64_t tiles;
      carve_grid_tiles(fg, 4, tx, ty, tiles);
      plan->carve.tiles_x[r] = tx;
      plan->carve.tiles_y[r] = ty;
      s_tiles[r] = tiles;
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < kPlanThreads / 32; ++w) tot += s_warp[w];
      s_nroi += tot;
    }
    __syncthreads();
  }
  const int nroi_all = s_nroi;
  if (nroi_all > FVV_MAX_GRIDS && tid == 0) atomicOr(&s_status, kPlanManyRois);
  __syncthreads();
  const int nroi = nroi_all < FVV_MAX_GRIDS ? nroi_all : FVV_MAX_GRIDS;
  // per-grid prefixes (one warp, 32 grids per step): occupancy words, tiles, k-row words
  if (warp == 0) {
    int64_t cw = 0, ct = 0, ck = 0, dense = 0, cr = 0;
    for (int g0 = 0; g0 < nroi; g0 += 32) {  // (grids past nroi add nothing)
      const int g = g0 + lane;
      const bool live = g < nroi;
      int64_t w = live ? s_words[g] : 0, t = live ? s_tiles[g] : 0, k = 0, vox = 0;
      MeshGridInfo gi;
      if (live) {
        const fvv_grid &fg = plan->carve.grids[g];
        vox = fg.dims[0] * fg.dims[1] * fg.dims[2];
        k = mesh_grid_info(fg, 0, 0, gi);  // offsets filled in below
      }
      const int64_t tr = live ? mesh_grid_tr_items(gi) : 0;
      int64_t iw = w, it = t, ik = k, iv = vox, ir = tr;  // inclusive scans
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t xw = __shfl_up_sync(0xffffffffu, iw, o), xt = __shfl_up_sync(0xffffffffu, it, o),
                      xk = __shfl_up_sync(0xffffffffu, ik, o), xv = __shfl_up_sync(0xffffffffu, iv, o),
                      xr = __shfl_up_sync(0xffffffffu, ir, o);
        if (lane >= o) {
          iw += xw;
          it += xt;
          ik += xk;
          iv += xv;
          ir += xr;
        }
      }
      const int64_t ow = cw + iw - w, ot = ct + it - t, ok = ck + ik - k, orr = cr + ir - tr;
      if (live) {
        plan->carve.word_off[g] = ow;
        plan->carve.blk_start[g] = ot;
        mesh_grid_info(plan->carve.grids[g], ow, ok, gi);
        gi.tr_off = orr;
        plan->mesh.gi[g] = gi;
        plan->mesh.tw_start[g] = ok;
      }
      cw += __shfl_sync(0xffffffffu, iw, 31);
      ct += __shfl_sync(0xffffffffu, it, 31);
      ck += __shfl_sync(0xffffffffu, ik, 31);
      dense += __shfl_sync(0xffffffffu, iv, 31);
      cr += __shfl_sync(0xffffffffu, ir, 31);
    }
    int st = s_status;
    if (cw > a.cap_words || ct > a.cap_tiles || ck > a.cap_tw) st |= kPlanCapacity;
    if (3 * ck >= ((int64_t)1 << 31)) st |= kPlanError;
    const bool run = st == 0;  // otherwise the device stages find nothing to do
    const int ng = run ? nroi : 0;
    for (int g = ng + lane; g <= FVV_MAX_GRIDS; g += 32) {  // the tables' tails, lane-parallel
      plan->carve.blk_start[g] = run ? ct : 0;
      plan->mesh.tw_start[g] = run ? ck : 0;
    }
    if (lane == 0) {
      plan->status = st;
      plan->nroi = nroi_all;
      plan->dense_tests = dense;
      plan->fine_words = cw;
      plan->carve.ngrid = ng;
      plan->carve.tile_log2 = 4;
      plan->carve.total_tiles = run ? ct : 0;
      plan->mesh.ngrid = ng;
      plan->mesh.tw_total = run ? ck : 0;
      plan->mesh.tw3 = run ? 3 * ck : 0;
      plan->mesh.tr_total = run ? cr : 0;
    }
  }
}

}  // namespace fvv

using namespace fvv;

// byte offsets inside the mapped host block
constexpr size_t kHsComps = 32;           // up to 4096 components (256 KB)
constexpr size_t kHsInfo = 512 * 1024;    // mesh_info of one ROI batch (64 B x 128)
constexpr size_t kHsCntF = 640 * 1024;    // per-ROI dense counts
constexpr int64_t kHsMaxCntF = 8192;
constexpr size_t kHsRCounts = 768 * 1024;  // colour-pass pixel counts

struct fvv_frame {
  std::vector<fvv_camera> cams, cams_by_id;
  std::vector<int64_t> mask_off, word_off, word_off_by_id, plane_off;
  int ncam = 0;
  int64_t sil_words = 0, planes = 0;
  fvv_frame_config cfg;
  fvv_grid coarse;
  // persistent device buffers
  DevBuf carve_ws, code;
  DevBuf sil, occ_c, cnt_c, ccl_ws, comps, occ_f, cnt_f, mesh_ws, mesh_scratch,
      mesh_totals, mesh_info, verts, tris, ntri, raster_ws, depth, vis, vplane_d, vplane_id,
      vraster_ws, src, rcounts, color, source, covered;
  // 32-pixel dirty-tile maps of the depth planes and of the virtual view's
  // depth/id planes: only tiles written by the previous frame are reset
  DevBuf dirty, vdirty;
  // the planes (and map allocations) the maps describe
  const void *dirty_for[2] = {nullptr, nullptr}, *vdirty_for[3] = {nullptr, nullptr, nullptr};
  int64_t vdirty_px = 0;
  // pinned host staging
  int64_t virt_px = 0;         // pixels of the last colour pass (0: none)
  void *host_small = nullptr;  // mapped pinned block (kHs* layout)
  void *host_small_dev = nullptr;
  size_t host_small_cap = 0;
  // results of the last run
  std::vector<fvv_grid> fine;
  std::vector<int64_t> fine_word_off;
  std::vector<int64_t> roi_component;
  std::vector<double> roi_box;  // 6 per ROI
  std::vector<int64_t> info;    // 8 per ROI
  int64_t nv = 0, nt = 0, vis_stride = 0;
  fvv_frame_stats stats;
  cudaEvent_t ev[9];
  // device-planned frames: capacities from the sizes seen so far
  int64_t seen_words = 0, seen_tiles = 0, seen_tw = 0, seen_v = 0, seen_s = 0;
  bool seen_plannable = false, caps_grown = false;
  struct Caps {
    int64_t words = 0, tiles = 0, tw = 0, v = 0, s = 0;
    bool ready = false;
  } caps;
  DevBuf plan, inputs;  // FramePlan, FrameInputs (device-planned frames)
  cudaStream_t side = nullptr;  // device-planned frames: the virtual view's raster
  cudaEvent_t fork = nullptr, join = nullptr;
  // one CUDA graph of the device-planned frame per input binding
  cudaGraphExec_t graph = nullptr;
  std::vector<char> graph_key, pending_key;
  std::vector<const void *> graph_bufs;  // the device buffers the graph was captured on
  long long graph_launches = 0;
  int last_mode = 0;  // fvv_frame_last_mode
  bool stage_times = true;  // fvv_frame_set_stage_times
  // a graph replay begun by frame_begin and not yet ended: its inputs (for a
  // host-planned redo) and the event recorded after its launch
  struct Pending {
    bool active = false;
    const uint8_t *masks = nullptr, *frames = nullptr;
    bool has_virt = false, has_off = false;
    fvv_camera virt{};
    int32_t rank_pos[FVV_MAX_CAMS] = {};
    int64_t frame_off[FVV_MAX_CAMS] = {};
    uint8_t fallback[3] = {0, 0, 0};
    bool has_fallback = false;
    cudaStream_t st = nullptr;
  } pend;
  cudaEvent_t launched = nullptr;
};

// B-2's ON-voxel and component counts: the first words of the CCL workspace
// (fvv_ccl26's layout), read in place
static int64_t *ccl_counts(fvv_frame *f) { return f->ccl_ws.as<int64_t>(); }

// Stage boundary event; inside a graph capture an external event-record node,
// so the replayed frame still reports its stage times.
static void stage_mark(fvv_frame *f, int e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(f->ev[e], st, cudaEventRecordExternal);
  else
    cudaEventRecord(f->ev[e], st);
}

static int grid_from_aabb(const double lo[3], const double hi[3], double spacing, int64_t budget,
                          fvv_grid &g) {
  // voxels.py:62-71 GridSpec.from_aabb (+ the budget check of voxels.py:34-37)
  for (int j = 0; j < 3; ++j)
    if (!(hi[j] > lo[j])) {
      set_error("AABB must have positive extent on every axis");
      return FVV_E_ARG;
    }
  int64_t n = 1;
  for (int j = 0; j < 3; ++j) {
    double d = std::ceil((hi[j] - lo[j]) / spacing - 1e-9);
    int64_t di = (int64_t)d;
    if (di < 1) di = 1;
    g.origin[j] = lo[j];
    g.dims[j] = di;
    n *= di;
  }
  g.spacing = spacing;
  if (n > budget) {
    set_error("grid of %lld voxels exceeds budget %lld", (long long)n, (long long)budget);
    return FVV_E_ARG;
  }
  return FVV_OK;
}

static int host_small_ensure(fvv_frame *f, size_t bytes) {
  if (bytes <= f->host_small_cap) return FVV_OK;
  if (f->host_small) cudaFreeHost(f->host_small);
  f->host_small = nullptr;
  size_t want = bytes * 2 + 4096;
  if (cudaHostAlloc(&f->host_small, want, cudaHostAllocMapped | cudaHostAllocPortable) !=
          cudaSuccess ||
      cudaHostGetDevicePointer(&f->host_small_dev, f->host_small, 0) != cudaSuccess) {
    cudaGetLastError();
    set_error("frame executor: mapped host allocation failed");
    return FVV_E_CUDA;
  }
  f->host_small_cap = want;
  return FVV_OK;
}

// Queue up to four device->host pieces (dst given as offsets into the
// mapped block) in one launch.
struct HostPiece {
  const void *src;
  size_t dst_off;
  int64_t bytes;            // fixed size, or
  const int64_t *count;     // device element count ...
  int64_t elem_bytes, max;  // ... of elem_bytes each, at most max
};
static void readback(fvv_frame *f, cudaStream_t st, std::initializer_list<HostPiece> pieces) {
  ReadBatch b{};
  int n = 0;
  int64_t most = 0;
  for (const HostPiece &h : pieces) {
    if (n == kReadPieces) break;
    ReadPiece &r = b.p[n++];
    r.src = (const int64_t *)h.src;
    r.dst = (int64_t *)((char *)f->host_small_dev + h.dst_off);
    r.count = h.count;
    r.words = h.bytes / 8;
    r.elem_words = h.elem_bytes / 8;
    r.max_elems = h.max;
    const int64_t w = h.count ? h.max * r.elem_words : r.words;
    most = w > most ? w : most;
  }
  int64_t bx = (most + 255) / 256;
  bx = bx < 1 ? 1 : (bx > 32 ? 32 : bx);
  launch_k(readback_kernel, dim3((unsigned)bx, (unsigned)n), 256, 0, st, b);
  note_launches(1);
}

#define FVV_TRY(stage, expr)                     \
  do {                                           \
    int _rc = (expr);                            \
    if (_rc != FVV_OK) {                         \
      if (out_stage) *out_stage = (stage);       \
      return _rc;                                \
    }                                            \
  } while (0)

extern "C" {

fvv_frame *fvv_frame_create(const fvv_camera *cams, int ncam, const fvv_frame_config *cfg) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("fvv_frame_create: %d cameras (1..%d)", ncam, FVV_MAX_CAMS);
    return nullptr;
  }
  fvv_frame *f = new fvv_frame();
  f->cfg = *cfg;
  f->ncam = ncam;
  f->cams.assign(cams, cams + ncam);
  int64_t m = 0, w = 0, pl = 0;
  for (int c = 0; c < ncam; ++c) {
    f->mask_off.push_back(m);
    f->word_off.push_back(w);
    f->plane_off.push_back(pl);
    m += (int64_t)cams[c].width * cams[c].height;
    w += (int64_t)cams[c].height * sil_stride_words(cams[c].width);
    pl += (int64_t)cams[c].width * cams[c].height;
  }
  f->sil_words = w;
  f->planes = pl;
  // cameras in ascending id order for the isovalue kernel (mesh.py:165-167)
  std::vector<int> order(ncam);
  for (int c = 0; c < ncam; ++c) order[c] = c;
  for (int a = 1; a < ncam; ++a)
    for (int b = a; b > 0 && cams[order[b]].id < cams[order[b - 1]].id; --b)
      std::swap(order[b], order[b - 1]);
  for (int c = 0; c < ncam; ++c) {
    f->cams_by_id.push_back(cams[order[c]]);
    f->word_off_by_id.push_back(f->word_off[order[c]]);
  }
  if (grid_from_aabb(cfg->stage_lo, cfg->stage_hi, cfg->coarse_spacing, cfg->budget,
                     f->coarse) != FVV_OK) {
    delete f;
    return nullptr;
  }
  for (int e = 0; e < 9; ++e) cudaEventCreate(&f->ev[e]);
  cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&f->join, cudaEventDisableTiming);
  if (f->sil.ensure(4 * (size_t)f->sil_words) || f->occ_c.ensure(4 * (size_t)((
          f->coarse.dims[0] * f->coarse.dims[1] * f->coarse.dims[2] + 31) / 32)) ||
      f->cnt_c.ensure(64) ||
      f->ccl_ws.ensure(fvv_ccl_workspace_bytes(&f->coarse)) ||
      f->comps.ensure(sizeof(fvv_component) * 4096) || f->mesh_totals.ensure(64) ||
      f->ntri.ensure(64) || f->carve_ws.ensure(fvv_carve_workspace_bytes(f->cams.data(), f->ncam)) ||
      host_small_ensure(f, 1 << 20)) {
    delete f;
    return nullptr;
  }
  return f;
}

void fvv_frame_destroy(fvv_frame *f) {
  if (!f) return;
  if (f->graph) cudaGraphExecDestroy(f->graph);
  if (f->side) cudaStreamDestroy(f->side);
  if (f->fork) cudaEventDestroy(f->fork);
  if (f->join) cudaEventDestroy(f->join);
  if (f->launched) cudaEventDestroy(f->launched);
  for (int e = 0; e < 9; ++e) cudaEventDestroy(f->ev[e]);
  if (f->host_small) cudaFreeHost(f->host_small);
  delete f;
}

// B-1 sparse carve + B-2 CCL (events 0, 1), common to both paths.
static int enqueue_b12(fvv_frame *f, const uint8_t *masks_dev, const FrameInputs *in,
                       cudaStream_t st, int *out_stage) {
  const fvv_frame_config &cfg = f->cfg;
  const int ncam = f->ncam;
  fvv_frame_stats &S = f->stats;
  stage_mark(f, 0, st);
  // ---- B-1 sparse carve (pipeline.py:154-157) ----
  const fvv_grid &G = f->coarse;
  const int64_t nvox_c = G.dims[0] * G.dims[1] * G.dims[2];
  S.sparse_tests = nvox_c;
  FVV_TRY(1, pack_silhouettes_bound(f->cams.data(), ncam, masks_dev, in, f->mask_off.data(),
                                    f->sil.as<uint32_t>(), f->word_off.data(), st));
  const int64_t zero = 0;
  FVV_TRY(1, fvv_carve(f->cams.data(), ncam, f->sil.as<uint32_t>(), f->word_off.data(), &G, 1,
                       &zero, cfg.min_views, f->occ_c.as<uint32_t>(), f->cnt_c.as<int64_t>(),
                       f->carve_ws.p, f->carve_ws.cap, st));
  stage_mark(f, 1, st);

  // ---- B-2 CCL, noise filter, ROIs (pipeline.py:159-166) ----
  FVV_TRY(2, fvv_ccl26(f->occ_c.as<uint32_t>(), &G, f->ccl_ws.p, f->ccl_ws.cap,
                       f->comps.as<fvv_component>(), 4096, nullptr, st));
  return FVV_OK;
}

// D-1 depth images, D-2 visibility, E colour pass (events 5..7). nv: vertex
// count or capacity (the raster records' stride), *nv_dev the count when
// non-null; nt_ub: triangle-count upper bound, *ntri_dev the count.
static int enqueue_tail(fvv_frame *f, const fvv_camera *virt, const int32_t *rank_pos,
                        const uint8_t *frames_dev, const int64_t *frame_off,
                        const uint8_t *fallback, cudaStream_t st, int *out_stage, int64_t nv,
                        const int64_t *nv_dev, int64_t nt_ub, const int64_t *ntri_dev,
                        bool have_mesh, const FrameInputs *in, cudaStream_t side) {
  const fvv_frame_config &cfg = f->cfg;
  const int ncam = f->ncam;
  // ---- E raster of the virtual view (render.py:64-113): it needs only the
  // mesh, so with a side stream it runs beside D-1 / D-2 (a fork in the
  // captured frame graph), joined before the colour pass ----
  f->virt_px = 0;
  const bool vraster = virt && have_mesh;
  int64_t np = 0;
  if (virt) {
    np = (int64_t)virt->width * virt->height;
    f->virt_px = np;
    FVV_TRY(7, f->color.ensure(3 * (size_t)np));
    FVV_TRY(7, f->source.ensure(4 * (size_t)np));
    FVV_TRY(7, f->covered.ensure((size_t)np));
    FVV_TRY(7, f->code.ensure((size_t)np));
  }
  if (vraster) {
    cudaStream_t vs = side ? side : st;
    if (side) {
      cudaEventRecord(f->fork, st);
      cudaStreamWaitEvent(side, f->fork, 0);
    }
    FVV_TRY(7, f->vplane_d.ensure(8 * (size_t)np));
    FVV_TRY(7, f->vplane_id.ensure(4 * (size_t)np));
    const size_t vwb = fvv_raster_workspace_bytes(nv, nt_ub, 1);
    FVV_TRY(7, f->vraster_ws.ensure(vwb));
    const int64_t off0 = 0;
    FVV_TRY(7, f->vdirty.ensure((size_t)(np + 31) / 32));
    // the map is valid for one plane pair at one image size
    const bool vfresh = f->vdirty_for[0] != f->vplane_d.p || f->vdirty_for[1] != f->vplane_id.p ||
                        f->vdirty_for[2] != f->vdirty.p || f->vdirty_px != np;
    FVV_TRY(7, fvv_rasterize_tracked(virt, 1, f->verts.as<double>(), nv, nv_dev,
                                     f->tris.as<int32_t>(), nt_ub, ntri_dev,
                                     f->vplane_d.as<double>(), &off0, f->vplane_id.as<int32_t>(),
                                     f->vraster_ws.p, f->vraster_ws.cap, f->vdirty.as<uint8_t>(),
                                     vfresh, vs));
    f->vdirty_for[0] = f->vplane_d.p;
    f->vdirty_for[1] = f->vplane_id.p;
    f->vdirty_for[2] = f->vdirty.p;
    f->vdirty_px = np;
    if (side) cudaEventRecord(f->join, side);
  }

  // ---- D-1 depth images, D-2 visibility (pipeline.py:198-207) ----
  if (have_mesh) {
    FVV_TRY(5, f->depth.ensure(8 * (size_t)f->planes));
    FVV_TRY(5, f->dirty.ensure((size_t)(f->planes + 31) / 32));
    const size_t rwb = fvv_raster_workspace_bytes(nv, nt_ub, ncam);
    FVV_TRY(5, f->raster_ws.ensure(rwb));
    const bool fresh = f->dirty_for[0] != f->depth.p || f->dirty_for[1] != f->dirty.p;
    FVV_TRY(5, fvv_rasterize_tracked(f->cams.data(), ncam, f->verts.as<double>(), nv,
                                     nv_dev, f->tris.as<int32_t>(), nt_ub, ntri_dev,
                                     f->depth.as<double>(), f->plane_off.data(), nullptr,
                                     f->raster_ws.p, f->raster_ws.cap, f->dirty.as<uint8_t>(),
                                     fresh, st));
    f->dirty_for[0] = f->depth.p;  // new planes or map: filled once above
    f->dirty_for[1] = f->dirty.p;
  }
  stage_mark(f, 5, st);
  FVV_TRY(6, f->vis.ensure(4 * (size_t)ncam * f->vis_stride));
  fill_async(f->vis.p, 0, 4 * (size_t)ncam * f->vis_stride, st);
  // (with a colour pass, the triangle sources of render.py:35-43 come out of
  // the same launch)
  std::vector<int32_t> rank_id(ncam);
  const bool sources = virt && have_mesh;
  if (sources) {
    for (int r = 0; r < ncam; ++r) rank_id[r] = f->cams[rank_pos[r]].id;
    FVV_TRY(6, f->src.ensure(4 * (size_t)(nt_ub > 0 ? nt_ub : 1)));
  }
  if (have_mesh)
    FVV_TRY(6, classify_sources(f->cams.data(), ncam, f->verts.as<double>(),
                                f->tris.as<int32_t>(), nt_ub, ntri_dev, f->depth.as<double>(),
                                f->plane_off.data(), cfg.t_v, f->vis.as<uint32_t>(),
                                f->vis_stride, ncam, rank_pos, rank_id.data(),
                                sources ? f->src.as<int32_t>() : nullptr, st));
  stage_mark(f, 6, st);

  // ---- E colour pass ----
  if (virt) {
    if (vraster) {
      if (side) cudaStreamWaitEvent(st, f->join, 0);
      FVV_TRY(7, f->rcounts.ensure(8 * (size_t)(1 + ncam)));
      FVV_TRY(7, fvv_render_count(f->cams.data(), ncam, virt, f->vplane_id.as<int32_t>(),
                                  f->src.as<int32_t>(), f->rcounts.as<int64_t>(), st));
      FVV_TRY(7, render_view_coded_bound(f->cams.data(), ncam, frames_dev, frame_off, in, virt,
                                         f->vplane_d.as<double>(), f->vplane_id.as<int32_t>(),
                                         f->src.as<int32_t>(), fallback, f->color.as<uint8_t>(),
                                         f->source.as<int32_t>(), f->covered.as<uint8_t>(),
                                         f->code.as<int8_t>(), f->rcounts.as<int64_t>(), st));
    } else {
      fill_async(f->code.p, 0xfe, (size_t)np, st);  // -2: nothing covered
      fill_async(f->color.p, 0, 3 * (size_t)np, st);
      fill_async(f->source.p, 0xff, 4 * (size_t)np, st);
      fill_async(f->covered.p, 0, (size_t)np, st);
    }
  }
  stage_mark(f, 7, st);

  return FVV_OK;
}

static int run_host_planned(fvv_frame *f, const uint8_t *masks_dev, const fvv_camera *virt,
                  const int32_t *rank_pos, const uint8_t *frames_dev, const int64_t *frame_off,
                  const uint8_t *fallback, void *stream, fvv_frame_stats *out_stats,
                  int *out_stage) {
  cudaStream_t st = (cudaStream_t)stream;
  const fvv_frame_config &cfg = f->cfg;
  const int ncam = f->ncam;
  if (out_stage) *out_stage = 0;
  memset(&f->stats, 0, sizeof(f->stats));
  fvv_frame_stats &S = f->stats;
  FVV_TRY(1, enqueue_b12(f, masks_dev, nullptr, st, out_stage));
  const fvv_grid &G = f->coarse;
  int64_t *hs = (int64_t *)f->host_small;
  readback(f, st, {{ccl_counts(f), 0, 16, nullptr, 0, 0},
                   {f->cnt_c.p, 16, 8, nullptr, 0, 0},
                   {f->comps.p, kHsComps, 0, ccl_counts(f) + 1,
                    (int64_t)sizeof(fvv_component), 4096}});
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    if (out_stage) *out_stage = 2;
    return cuda_check("fvv_frame_run B-2");
  }
  const int64_t ncomp = hs[1];
  S.sparse_occupied = hs[2];
  const fvv_component *comps = (const fvv_component *)(hs + 4);
  std::vector<fvv_component> big;
  if (ncomp > 4096) {
    FVV_TRY(2, f->comps.ensure(sizeof(fvv_component) * ncomp));
    FVV_TRY(2, fvv_ccl_components(&G, f->ccl_ws.p, f->comps.as<fvv_component>(), ncomp, st));
    big.resize(ncomp);
    cudaMemcpyAsync(big.data(), f->comps.p, sizeof(fvv_component) * ncomp,
                    cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    comps = big.data();
  }
  f->fine.clear();
  f->roi_component.clear();
  f->roi_box.clear();
  double extent[3];
  for (int j = 0; j < 3; ++j) extent[j] = G.origin[j] + G.spacing * (double)G.dims[j];
  for (int64_t c = 0; c < ncomp; ++c) {
    const double cnt = (double)comps[c].voxel_count;
    if (!((double)cfg.t_small <= cnt && cnt <= cfg.t_large)) continue;  // hull.py:46-47
    double lo[3], hi[3];
    for (int j = 0; j < 3; ++j) {  // hull.py:279-282
      lo[j] = G.origin[j] + G.spacing * (double)comps[c].bbox_min[j] - cfg.roi_margin;
      hi[j] = G.origin[j] + G.spacing * ((double)comps[c].bbox_max[j] + 1.0) + cfg.roi_margin;
      lo[j] = lo[j] >= G.origin[j] ? lo[j] : G.origin[j];  // np.maximum(lo, stage_lo)
      hi[j] = hi[j] <= extent[j] ? hi[j] : extent[j];      // np.minimum(hi, stage_hi)
    }
    for (int j = 0; j < 3; ++j)
      if (!(lo[j] < hi[j])) {
        set_error("ROI must have positive extent");
        if (out_stage) *out_stage = 2;
        return FVV_E_ARG;
      }
    f->roi_component.push_back(comps[c].id);
    for (int j = 0; j < 3; ++j) f->roi_box.push_back(lo[j]);
    for (int j = 0; j < 3; ++j) f->roi_box.push_back(hi[j]);
  }
  S.components = (int64_t)f->roi_component.size();
  stage_mark(f, 2, st);

  // ---- B-3 dense carve (pipeline.py:168-173) ----
  const int nroi = (int)f->roi_component.size();
  f->fine.resize(nroi);
  f->fine_word_off.resize(nroi);
  int64_t fw = 0;
  for (int r = 0; r < nroi; ++r) {
    FVV_TRY(3, grid_from_aabb(&f->roi_box[6 * r], &f->roi_box[6 * r + 3], cfg.fine_spacing,
                              cfg.budget, f->fine[r]));
    const int64_t n = f->fine[r].dims[0] * f->fine[r].dims[1] * f->fine[r].dims[2];
    S.dense_tests += n;
    f->fine_word_off[r] = fw;
    fw += (n + 31) / 32;
  }
  f->seen_words = fw;
  f->seen_tiles = f->seen_tw = 0;
  for (int r = 0; r < nroi; ++r) {
    uint32_t tx, ty;
    int64_t tiles;
    carve_grid_tiles(f->fine[r], 4, tx, ty, tiles);
    MeshGridInfo gi;
    f->seen_tiles += tiles;
    f->seen_tw += mesh_grid_info(f->fine[r], 0, 0, gi);
  }
  f->seen_plannable = nroi <= FVV_MAX_GRIDS && ncomp <= 4096;
  f->seen_v = f->seen_s = 0;
  FVV_TRY(3, f->occ_f.ensure(4 * (size_t)(fw > 0 ? fw : 1)));
  FVV_TRY(3, f->cnt_f.ensure(8 * (size_t)(nroi > 0 ? nroi : 1)));
  for (int r0 = 0; r0 < nroi; r0 += FVV_MAX_GRIDS) {
    const int nb = nroi - r0 < FVV_MAX_GRIDS ? nroi - r0 : FVV_MAX_GRIDS;
    FVV_TRY(3, fvv_carve(f->cams.data(), ncam, f->sil.as<uint32_t>(), f->word_off.data(),
                         &f->fine[r0], nb, &f->fine_word_off[r0], cfg.min_views,
                         f->occ_f.as<uint32_t>(), f->cnt_f.as<int64_t>() + r0, f->carve_ws.p,
                         f->carve_ws.cap, st));
  }
  stage_mark(f, 3, st);

  // ---- C polygonize every ROI (pipeline.py:175-190) ----
  f->info.assign(8 * (size_t)nroi, 0);
  f->nv = f->nt = 0;
  int64_t v_before = 0, t_before = 0;
  for (int r0 = 0; r0 < nroi; r0 += FVV_MAX_GRIDS) {
    const int nb = nroi - r0 < FVV_MAX_GRIDS ? nroi - r0 : FVV_MAX_GRIDS;
    const size_t wsb = fvv_mesh_workspace_bytes(&f->fine[r0], nb);
    FVV_TRY(4, f->mesh_ws.ensure(wsb));
    FVV_TRY(4, f->mesh_info.ensure(64 * (size_t)nb));
    FVV_TRY(4, fvv_mesh_prepare(&f->fine[r0], nb, f->occ_f.as<uint32_t>(),
                                &f->fine_word_off[r0], f->mesh_ws.p, wsb, st));
    FVV_TRY(4, fvv_mesh_counts(&f->fine[r0], nb, f->mesh_ws.p, f->mesh_totals.as<int64_t>(),
                               nullptr, st));
    readback(f, st, {{f->mesh_totals.p, 0, 24, nullptr, 0, 0}});
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      if (out_stage) *out_stage = 4;
      return cuda_check("fvv_frame_run C");
    }
    const int64_t nv = hs[0], ns = hs[1];
    f->seen_v = nv;  // (single-batch frames: the device planner's capacities)
    f->seen_s = ns;
    const size_t sb = fvv_mesh_emit_scratch_bytes(nv, ns);
    FVV_TRY(4, f->mesh_scratch.ensure(sb));
    // vertices / triangles of all batches share one array; keep prior batches
    if (r0 == 0) {
      FVV_TRY(4, f->verts.ensure(24 * (size_t)(nv > 0 ? nv : 1)));
      FVV_TRY(4, f->tris.ensure(12 * (size_t)(5 * ns > 0 ? 5 * ns : 1)));
    } else {  // later ROI batches append: grow keeping the earlier batches
      FVV_TRY(4, f->verts.grow_keep(24 * (size_t)(v_before + nv), 24 * (size_t)v_before, st));
      FVV_TRY(4, f->tris.grow_keep(12 * (size_t)(t_before + 5 * ns), 12 * (size_t)t_before, st));
    }
    FVV_TRY(4, fvv_mesh_emit(f->cams_by_id.data(), ncam, f->sil.as<uint32_t>(),
                             f->word_off_by_id.data(), &f->fine[r0], nb,
                             f->occ_f.as<uint32_t>(), &f->fine_word_off[r0], cfg.exact,
                             cfg.fixed_isovalue, f->mesh_ws.p, wsb, nv, ns, f->mesh_scratch.p,
                             sb, f->verts.as<double>() + 3 * v_before,
                             f->tris.as<int32_t>() + 3 * t_before, st));
    FVV_TRY(4, fvv_mesh_counts(&f->fine[r0], nb, f->mesh_ws.p, f->mesh_totals.as<int64_t>(),
                               f->mesh_info.as<int64_t>(), st));
    if (r0 + nb < nroi) {  // more batches: need this batch's triangle count now
      readback(f, st, {{f->mesh_totals.p, 0, 24, nullptr, 0, 0},
                       {f->mesh_info.p, kHsInfo, 64 * (int64_t)nb, nullptr, 0, 0}});
      cudaStreamSynchronize(st);
      memcpy(f->info.data() + 8 * (size_t)r0, (char *)f->host_small + kHsInfo, 64 * (size_t)nb);
      const int64_t tb = hs[2];
      if (v_before)
        launch_k(offset_tris_kernel, 148 * 4, 256, 0, st, f->tris.as<int32_t>() + 3 * t_before, 3 * tb,
                                                    (int32_t)v_before);
      for (int r = r0; r < r0 + nb; ++r) {
        f->info[8 * r + 0] += v_before;
        f->info[8 * r + 4] += t_before;
      }
      v_before += nv;
      t_before += tb;
    } else {
      // last (usually only) batch: its triangle count stays on the device
      // for D-1/D-2; the host reads it with the final counters
      if (v_before) {
        readback(f, st, {{f->mesh_totals.p, 0, 24, nullptr, 0, 0}});
        cudaStreamSynchronize(st);
        launch_k(offset_tris_kernel, 148 * 4, 256, 0, st, f->tris.as<int32_t>() + 3 * t_before,
                                                    3 * hs[2], (int32_t)v_before);
      }
      f->nv = v_before + nv;
      f->nt = t_before + 5 * ns;  // upper bound until the final read
    }
  }
  stage_mark(f, 4, st);

  // device-side total triangle count for D-1 / D-2 / E (no host round trip)
  int64_t *ntri_dev = f->ntri.as<int64_t>();
  if (nroi > 0)
    launch_k(add_count_kernel, 1, 32, 0, st, ntri_dev, f->mesh_totals.as<int64_t>() + 2, t_before);
  else
    fill_async(ntri_dev, 0, 8, st);
  const int64_t nt_ub = f->nt;
  f->vis_stride = (nt_ub + 31) / 32 > 0 ? (nt_ub + 31) / 32 : 1;

  const bool have_mesh = f->nv > 0 && nt_ub > 0;
  FVV_TRY(5, enqueue_tail(f, virt, rank_pos, frames_dev, frame_off, fallback, st, out_stage, f->nv,
                          nullptr, nt_ub, ntri_dev, have_mesh, nullptr, nullptr));

  // ---- final counters (one read) ----
  int64_t *h = hs;
  const int last0 = nroi ? ((nroi - 1) / FVV_MAX_GRIDS) * FVV_MAX_GRIDS : 0;
  std::vector<int64_t> cnt_big;
  if (nroi > kHsMaxCntF) {  // rare: more ROIs than the mapped block holds
    cnt_big.resize(nroi);
    cudaMemcpyAsync(cnt_big.data(), f->cnt_f.p, 8 * (size_t)nroi, cudaMemcpyDeviceToHost, st);
  }
  const bool counted = virt && have_mesh;  // rcounts: [covered, per rig camera]
  const HostPiece rc_piece{counted ? f->rcounts.p : ntri_dev, kHsRCounts,
                           counted ? 8 * (int64_t)(1 + ncam) : 0, nullptr, 0, 0};
  if (nroi)
    readback(f, st, {{ntri_dev, 0, 8, nullptr, 0, 0},
                     {f->cnt_f.p, kHsCntF, 8 * (nroi > kHsMaxCntF ? 0 : (int64_t)nroi), nullptr,
                      0, 0},
                     {f->mesh_info.p, kHsInfo, 64 * (int64_t)(nroi - last0), nullptr, 0, 0},
                     rc_piece});
  else
    readback(f, st, {{ntri_dev, 0, 8, nullptr, 0, 0}, rc_piece});
  stage_mark(f, 8, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    if (out_stage) *out_stage = 8;
    return cuda_check("fvv_frame_run");
  }
  const int64_t *cnt_f = nroi > kHsMaxCntF ? cnt_big.data()
                                           : (const int64_t *)((char *)f->host_small + kHsCntF);
  if (nroi) {
    memcpy(f->info.data() + 8 * (size_t)last0, (char *)f->host_small + kHsInfo,
           64 * (size_t)(nroi - last0));
    for (int r = last0; r < nroi; ++r) {
      f->info[8 * r + 0] += v_before;
      f->info[8 * r + 4] += t_before;
    }
  }
  f->nt = h[0];
  S.triangles = h[0];
  if (counted) {
    const int64_t *rcn = (const int64_t *)((char *)f->host_small + kHsRCounts);
    S.covered_px = rcn[0];
    for (int c = 0; c < ncam; ++c) S.sourced_px += rcn[1 + c];
  }
  S.vertices = f->nv;
  S.n_rois = nroi;
  for (int r = 0; r < nroi; ++r) {
    S.dense_occupied += cnt_f[r];
    S.fallback_edges += f->info[8 * r + 6];
    S.inconsistent_edge_starts += f->info[8 * r + 7];
  }
  if (!cfg.exact) S.fallback_edges = S.inconsistent_edge_starts = 0;
  for (int e = 0; e < 8; ++e) cudaEventElapsedTime(&S.ms[e], f->ev[e], f->ev[e + 1]);
  if (out_stats) *out_stats = S;
  return cuda_check("fvv_frame_run");
}

// ---- device-planned frames -------------------------------------------------
// B-1 .. E enqueued without a host round trip: the planner kernel replaces the
// host's ROI step, B-3 / C run over its tables with capacities taken from the
// sizes seen so far (x1.25), and one final read brings back every count. A
// frame the planner does not take, or one that outgrows a capacity, is redone
// by the host-planned path (which also sets the capacities).
constexpr size_t kDs = 800 * 1024;  // mapped-block region of the device-planned read
constexpr size_t kDsRCounts = 128, kDsComp = 1024, kDsBox = 2048, kDsGrid = 8192,
                 kDsCntF = 16384, kDsInfo = 17408;

// FVV_FORK=0: the device-planned frame as one chain (no side-stream
// branches; ncu launch lists then follow the stage order)
static cudaStream_t side_stream(const fvv_frame *f) {
  static const bool on = [] {
    const char *e = getenv("FVV_FORK");
    return !(e && e[0] == '0');
  }();
  return on ? f->side : nullptr;
}

static int enqueue_device_planned(fvv_frame *f, const uint8_t *masks_dev, const fvv_camera *virt,
                                  const int32_t *rank_pos, const uint8_t *frames_dev,
                                  const int64_t *frame_off, const uint8_t *fallback,
                                  cudaStream_t st, int *out_stage) {
  const fvv_frame_config &cfg = f->cfg;
  const int ncam = f->ncam;
  const fvv_frame::Caps &K = f->caps;
  FVV_TRY(1, enqueue_b12(f, masks_dev, f->inputs.as<FrameInputs>(), st, out_stage));
  // ---- B-2 noise filter + ROIs on the device (pipeline.py:159-166) ----
  FVV_TRY(2, f->plan.ensure(sizeof(FramePlan)));
  FramePlan *P = f->plan.as<FramePlan>();
  PlanArgs pa;
  pa.coarse = f->coarse;
  pa.roi_margin = cfg.roi_margin;
  pa.fine_spacing = cfg.fine_spacing;
  pa.t_large = cfg.t_large;
  pa.t_small = cfg.t_small;
  pa.budget = cfg.budget;
  pa.comp_cap = 4096;
  pa.cap_words = K.words;
  pa.cap_tiles = K.tiles;
  pa.cap_tw = K.tw;
  launch_k(frame_plan_kernel, 1, kPlanThreads, 0, st, pa, f->comps.as<fvv_component>(),
                                                ccl_counts(f), P);
  note_launches(1);
  stage_mark(f, 2, st);
  // ---- B-3 dense carve over the planned grids ----
  FVV_TRY(3, f->occ_f.ensure(4 * (size_t)K.words));
  FVV_TRY(3, f->cnt_f.ensure(8 * (size_t)FVV_MAX_GRIDS));
  FVV_TRY(3, carve_batch(f->cams.data(), ncam, f->sil.as<uint32_t>(), f->word_off.data(),
                         &P->carve, FVV_MAX_GRIDS, 4, K.tiles, cfg.min_views,
                         f->occ_f.as<uint32_t>(), f->cnt_f.as<int64_t>(), f->carve_ws.p,
                         f->carve_ws.cap, st, true));  // (B-1 built the cell maps)
  stage_mark(f, 3, st);
  // ---- C polygonize ----
  FVV_TRY(4, f->mesh_ws.ensure(mesh_ws_bytes(K.tw, FVV_MAX_GRIDS)));
  FVV_TRY(4, f->mesh_scratch.ensure(mesh_emit_scratch(K.v, K.s)));
  FVV_TRY(4, mesh_prepare_batch(&P->mesh, K.tw, FVV_MAX_GRIDS, f->occ_f.as<uint32_t>(),
                                f->mesh_ws.p, f->mesh_ws.cap, st, side_stream(f), f->fork,
                                f->join, f->mesh_scratch.p, K.v, K.s));
  FVV_TRY(4, f->verts.ensure(24 * (size_t)K.v));
  FVV_TRY(4, f->tris.ensure(12 * (size_t)(5 * K.s)));
  FVV_TRY(4, mesh_emit_batch(f->cams_by_id.data(), ncam, f->sil.as<uint32_t>(),
                             f->word_off_by_id.data(), &P->mesh, K.tw, FVV_MAX_GRIDS, cfg.exact,
                             cfg.fixed_isovalue, f->mesh_ws.p, f->mesh_ws.cap, K.v, K.s,
                             f->mesh_scratch.p, f->mesh_scratch.cap, f->verts.as<double>(),
                             f->tris.as<int32_t>(), st, true, side_stream(f) != nullptr));
  stage_mark(f, 4, st);
  int64_t *totals = mesh_ws_totals(f->mesh_ws.p, K.tw, FVV_MAX_GRIDS);  // V, S, T
  const int64_t nt_ub = 5 * K.s;
  f->vis_stride = (nt_ub + 31) / 32 > 0 ? (nt_ub + 31) / 32 : 1;
  FVV_TRY(5, enqueue_tail(f, virt, rank_pos, frames_dev, frame_off, fallback, st, out_stage, K.v,
                          totals, nt_ub, totals + 2, true, f->inputs.as<FrameInputs>(),
                          side_stream(f)));
  // ---- every count in one read ----
  const int64_t *nroi = &P->nroi;
  readback(f, st, {{ccl_counts(f), kDs, 16, nullptr, 0, 0},
                   {f->cnt_c.p, kDs + 16, 8, nullptr, 0, 0},
                   {P, kDs + 32, 32, nullptr, 0, 0},  // status, nroi, dense_tests, fine_words
                   {totals, kDs + 64, 24, nullptr, 0, 0},
                   {virt ? f->rcounts.p : totals, kDs + kDsRCounts,
                    virt ? 8 * (int64_t)(1 + ncam) : 0, nullptr, 0, 0},
                   {P->roi_component, kDs + kDsComp, 0, nroi, 8, FVV_MAX_GRIDS},
                   {P->roi_box, kDs + kDsBox, 0, nroi, 48, FVV_MAX_GRIDS},
                   {P->carve.grids, kDs + kDsGrid, 0, nroi, (int64_t)sizeof(fvv_grid),
                    FVV_MAX_GRIDS},
                   {f->cnt_f.p, kDs + kDsCntF, 0, nroi, 8, FVV_MAX_GRIDS},
                   {mesh_ws_info(f->mesh_ws.p, K.tw, FVV_MAX_GRIDS), kDs + kDsInfo, 0, nroi, 64,
                    FVV_MAX_GRIDS}});
  stage_mark(f, 8, st);
  return FVV_OK;
}

// After the frame's synchronisation: host state and stats from the final
// read. False when the host-planned path must redo the frame.
static bool finish_device_planned(fvv_frame *f, bool colour) {
  const char *hb = (const char *)f->host_small + kDs;
  const int64_t *h = (const int64_t *)hb;
  const int64_t status = h[4], nroi = h[5], V = h[8], Sn = h[9], T = h[10];
  if (status != 0 || V > f->caps.v || Sn > f->caps.s) {
    static const bool dbg = getenv("FVV_PLAN_DEBUG") != nullptr;
    if (dbg)
      fprintf(stderr, "fvv: device-planned frame redone on the host: status %lld nroi %lld "
              "V %lld/%lld S %lld/%lld words %lld/%lld\n", (long long)status, (long long)nroi,
              (long long)V, (long long)f->caps.v, (long long)Sn, (long long)f->caps.s,
              (long long)h[7], (long long)f->caps.words);
    return false;
  }
  fvv_frame_stats &S = f->stats;
  S.sparse_occupied = h[2];
  S.components = nroi;
  S.dense_tests = h[6];
  S.n_rois = nroi;
  S.vertices = V;
  S.triangles = T;
  f->nv = V;
  f->nt = T;
  const int64_t *comp = (const int64_t *)(hb + kDsComp);
  const double *box = (const double *)(hb + kDsBox);
  const fvv_grid *grid = (const fvv_grid *)(hb + kDsGrid);
  const int64_t *cnt = (const int64_t *)(hb + kDsCntF);
  const int64_t *info = (const int64_t *)(hb + kDsInfo);
  f->roi_component.assign(comp, comp + nroi);
  f->roi_box.assign(box, box + 6 * nroi);
  f->fine.assign(grid, grid + nroi);
  f->info.assign(info, info + 8 * nroi);
  f->fine_word_off.clear();
  for (int64_t r = 0; r < nroi; ++r) {
    S.dense_occupied += cnt[r];
    S.fallback_edges += info[8 * r + 6];
    S.inconsistent_edge_starts += info[8 * r + 7];
  }
  if (!f->cfg.exact) S.fallback_edges = S.inconsistent_edge_starts = 0;
  if (colour) {
    const int64_t *rcn = (const int64_t *)(hb + kDsRCounts);
    S.covered_px = rcn[0];
    for (int c = 0; c < f->ncam; ++c) S.sourced_px += rcn[1 + c];
  }
  // (eight cudaEventElapsedTime calls cost ~22 us of host time per frame)
  for (int e = 0; e < 8; ++e)
    if (!f->stage_times || cudaEventElapsedTime(&S.ms[e], f->ev[e], f->ev[e + 1]) != cudaSuccess)
      S.ms[e] = 0.0f;
  cudaGetLastError();
  return true;
}

static int64_t with_headroom(int64_t need) { return need + need / 4 + 1024; }

// capacities for the next device-planned frames (grown only: buffers and a
// captured graph stay valid while they hold)
static void update_caps(fvv_frame *f, int64_t words, int64_t tiles, int64_t tw, int64_t v,
                        int64_t sn) {
  fvv_frame::Caps &K = f->caps;
  bool grew = false;
  auto fit = [&grew](int64_t need, int64_t &cap) {
    if (need > cap - cap / 16 || cap == 0) {  // within 6 % of the capacity: grow now
      cap = with_headroom(need > cap ? need : cap);
      grew = true;
    }
  };
  fit(words, K.words);
  fit(tiles, K.tiles);  // (launch size of B-3's tile classification only)
  fit(tw, K.tw);
  fit(v, K.v);
  fit(sn, K.s);
  if (K.tiles > (int64_t)1 << 19) K.tiles = (int64_t)1 << 19;  // carve's split-mode tile cap
  K.ready = true;
  if (grew) f->caps_grown = true;  // buffers re-sized before the next device-planned frame
  if (grew && f->graph) {  // the graph's launches were sized for the old capacities
    cudaGraphExecDestroy(f->graph);
    f->graph = nullptr;
    f->graph_key.clear();
  }
}

// The device-planned frame's buffers at the current capacities, allocated
// before the frame is enqueued (never while a captured graph could use them;
// the previous frame's outputs are dropped, as any new frame drops them).
static void reserve_buffers(fvv_frame *f) {
  const fvv_frame::Caps &K = f->caps;
  {
    const int64_t nt_ub = 5 * K.s;
    f->occ_f.ensure(4 * (size_t)K.words);
    f->cnt_f.ensure(8 * (size_t)FVV_MAX_GRIDS);
    f->mesh_ws.ensure(mesh_ws_bytes(K.tw, FVV_MAX_GRIDS));
    f->mesh_scratch.ensure(mesh_emit_scratch(K.v, K.s));
    f->verts.ensure(24 * (size_t)K.v);
    f->tris.ensure(12 * (size_t)nt_ub);
    f->raster_ws.ensure(fvv_raster_workspace_bytes(K.v, nt_ub, f->ncam));
    f->vraster_ws.ensure(fvv_raster_workspace_bytes(K.v, nt_ub, 1));
    f->vis.ensure(4 * (size_t)f->ncam * ((nt_ub + 31) / 32 > 0 ? (nt_ub + 31) / 32 : 1));
    f->src.ensure(4 * (size_t)(nt_ub > 0 ? nt_ub : 1));
    f->plan.ensure(sizeof(FramePlan));
    f->inputs.ensure(sizeof(FrameInputs));
  }
  f->caps_grown = false;
}

// A device-planned frame that has completed: its counts and tables, and the
// capacities for the next ones. False: the frame must be redone host-planned.
static bool finish_after_sync(fvv_frame *f, bool colour) {
  const bool done = finish_device_planned(f, colour);
  if (done) {
    const int64_t *h = (const int64_t *)((const char *)f->host_small + kDs);
    // (tiles / k-row words of this frame are not read back: their
    // capacities grow through a host-planned frame when the planner reports one)
    update_caps(f, h[7], 0, 0, h[8], h[9]);
  }
  return done;
}

// Every device buffer a captured frame graph may address: a host-planned
// frame (redone or not plannable) can reallocate some of them without
// growing the capacities, and the graph must then not replay.
static std::vector<const void *> bound_buffers(const fvv_frame *f) {
  const DevBuf *b[] = {&f->carve_ws, &f->code, &f->sil, &f->occ_c, &f->cnt_c, &f->ccl_ws,
                       &f->comps, &f->occ_f, &f->cnt_f, &f->mesh_ws, &f->mesh_scratch,
                       &f->mesh_totals, &f->mesh_info, &f->verts, &f->tris, &f->ntri,
                       &f->raster_ws, &f->depth, &f->vis, &f->vplane_d, &f->vplane_id,
                       &f->vraster_ws, &f->src, &f->rcounts, &f->color, &f->source,
                       &f->covered, &f->dirty, &f->vdirty, &f->plan, &f->inputs};
  std::vector<const void *> v;
  v.reserve(sizeof(b) / sizeof(b[0]) + 1);
  for (const DevBuf *d : b) v.push_back(d->p);
  v.push_back(f->host_small_dev);
  return v;
}

// What a captured frame graph bakes in: the virtual camera, ranks, fallback
// colour, stream, capacities and the masks' alignment class (the masks and
// frame pointers are bound per frame through FrameInputs).
static std::vector<char> graph_key(const fvv_frame *f, const uint8_t *masks_dev,
                                   const fvv_camera *virt, const int32_t *rank_pos,
                                   const uint8_t *frames_dev, const int64_t *frame_off,
                                   const uint8_t *fallback, cudaStream_t st) {
  std::vector<char> k;
  auto put = [&k](const void *p, size_t n) {
    const char *c = (const char *)p;
    k.insert(k.end(), c, c + n);
  };
  const char wide = ((uintptr_t)masks_dev & 15) == 0;  // the pack kernel's variant
  put(&wide, 1);
  put(&st, sizeof(st));
  put(&f->caps, sizeof(f->caps));
  const char has_virt = virt != nullptr;
  put(&has_virt, 1);
  if (virt) {
    put(virt, sizeof(*virt));
    put(rank_pos, sizeof(int32_t) * f->ncam);
    put(fallback, 3);
  }
  return k;
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char *e = getenv("FVV_FRAME_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool device_planning_enabled() {
  static const bool on = [] {
    const char *e = getenv("FVV_DEVICE_PLAN");
    return !(e && e[0] == '0');
  }();
  return on;
}

// One device-planned frame: a plain enqueue, a graph capture (the second
// frame with the same bindings) or a graph replay. True when it completed.
// begin_only: launch a graph replay and return without waiting (done stays
// false, *replayed tells whether it was launched); a frame that would not
// replay is left untouched.
static int run_device_planned(fvv_frame *f, const uint8_t *masks_dev, const fvv_camera *virt,
                              const int32_t *rank_pos, const uint8_t *frames_dev,
                              const int64_t *frame_off, const uint8_t *fallback, cudaStream_t st,
                              int *out_stage, bool &done, bool begin_only = false,
                              bool *replayed = nullptr) {
  done = false;
  const bool graphs = graphs_enabled() && st != nullptr && st != cudaStreamLegacy &&
                      st != cudaStreamPerThread;
  std::vector<char> key;
  if (begin_only) {
    *replayed = false;
    if (!graphs || f->caps_grown || !f->graph || bound_buffers(f) != f->graph_bufs) return FVV_OK;
    key = graph_key(f, masks_dev, virt, rank_pos, frames_dev, frame_off, fallback, st);
    if (key != f->graph_key) return FVV_OK;
  }
  memset(&f->stats, 0, sizeof(f->stats));
  if (out_stage) *out_stage = 0;
  if (f->caps_grown) reserve_buffers(f);
  if (graphs && !begin_only)
    key = graph_key(f, masks_dev, virt, rank_pos, frames_dev, frame_off, fallback, st);
  {  // this frame's input pointers, read by the pack and colour kernels
    if (f->inputs.ensure(sizeof(FrameInputs))) return FVV_E_CUDA;
    static thread_local FrameInputs in;
    memset(&in, 0, sizeof(in));
    in.masks = masks_dev;
    in.frames = frames_dev;
    if (virt && frame_off)
      for (int c = 0; c < f->ncam; ++c) in.frame_off[c] = frame_off[c];
    launch_k(bind_inputs_kernel, 1, 32, 0, st, in, f->inputs.as<FrameInputs>());
    note_launches(1);
  }
  f->last_mode = 1;  // device-planned, enqueued
  if (f->graph && bound_buffers(f) != f->graph_bufs) {  // a buffer moved under the graph
    cudaGraphExecDestroy(f->graph);
    f->graph = nullptr;
    f->graph_key.clear();
  }
  if (graphs && f->graph && key == f->graph_key) {
    f->last_mode = 3;  // graph replay
    f->stats.sparse_tests = f->coarse.dims[0] * f->coarse.dims[1] * f->coarse.dims[2];
    f->virt_px = virt ? (int64_t)virt->width * virt->height : 0;
    const int64_t nt_ub = 5 * f->caps.s;
    f->vis_stride = (nt_ub + 31) / 32 > 0 ? (nt_ub + 31) / 32 : 1;
    if (cudaGraphLaunch(f->graph, st) != cudaSuccess) return cuda_check("fvv_frame_run graph");
    note_launches(f->graph_launches);
    if (begin_only) {
      if (!f->launched) cudaEventCreateWithFlags(&f->launched, cudaEventDisableTiming);
      cudaEventRecord(f->launched, st);
      *replayed = true;
      return cuda_check("fvv_frame_run graph");
    }
  } else if (graphs && key == f->pending_key) {
    f->last_mode = 2;  // graph capture + launch
    // second frame with these bindings (buffers and dirty maps settled by the
    // first): capture the frame once, then replay it
    if (f->graph) cudaGraphExecDestroy(f->graph);
    f->graph = nullptr;
    f->graph_key.clear();
    const long long n0 = thread_launch_count();
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return cuda_check("fvv_frame_run capture");
    const int rc = enqueue_device_planned(f, masks_dev, virt, rank_pos, frames_dev, frame_off,
                                          fallback, st, out_stage);
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(st, &g);
    if (rc != FVV_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ec != cudaSuccess || cudaGraphInstantiate(&f->graph, g, 0) != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      f->graph = nullptr;
      return cuda_check("fvv_frame_run graph capture");
    }
    cudaGraphDestroy(g);
    f->graph_key = key;
    f->graph_bufs = bound_buffers(f);
    f->graph_launches = thread_launch_count() - n0;
    if (cudaGraphLaunch(f->graph, st) != cudaSuccess) return cuda_check("fvv_frame_run graph");
  } else {
    FVV_TRY(0, enqueue_device_planned(f, masks_dev, virt, rank_pos, frames_dev, frame_off,
                                      fallback, st, out_stage));
    if (graphs) f->pending_key = key;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    if (out_stage) *out_stage = 8;
    return cuda_check("fvv_frame_run");
  }
  done = finish_after_sync(f, virt != nullptr);
  return cuda_check("fvv_frame_run");
}

int fvv_frame_run(fvv_frame *f, const uint8_t *masks_dev, const fvv_camera *virt,
                  const int32_t *rank_pos, const uint8_t *frames_dev, const int64_t *frame_off,
                  const uint8_t *fallback, void *stream, fvv_frame_stats *out_stats,
                  int *out_stage) {
  cudaStream_t st = (cudaStream_t)stream;
  if (f->caps.ready && device_planning_enabled()) {
    bool done = false;
    const int rc = run_device_planned(f, masks_dev, virt, rank_pos, frames_dev, frame_off,
                                      fallback, st, out_stage, done);
    if (rc != FVV_OK) return rc;
    if (done) {
      if (out_stats) *out_stats = f->stats;
      return FVV_OK;
    }
  }
  f->last_mode = 0;  // host-planned
  const int rc = run_host_planned(f, masks_dev, virt, rank_pos, frames_dev, frame_off, fallback,
                                  stream, out_stats, out_stage);
  if (rc == FVV_OK && f->seen_plannable)
    update_caps(f, f->seen_words, f->seen_tiles, f->seen_tw, f->seen_v, f->seen_s);
  return rc;
}


}  // extern "C"

// fvv_frame_run in two halves for the sequence runner's lanes: a frame that
// replays its graph is launched and left running (*async), so the lane can
// finish its previous frame while this one runs; frame_end waits for it
// (the event recorded after its launch, not the whole stream) and reads its
// results back, or redoes it host-planned when the device planner handed it
// back. Any other frame runs to completion in frame_begin.
int fvv::frame_begin(fvv_frame *f, const uint8_t *masks_dev, const fvv_camera *virt,
                     const int32_t *rank_pos, const uint8_t *frames_dev, const int64_t *frame_off,
                     const uint8_t *fallback, void *stream, fvv_frame_stats *out_stats,
                     int *out_stage, bool *async) {
  *async = false;
  cudaStream_t st = (cudaStream_t)stream;
  if (f->pend.active) {
    set_error("fvv_frame: a begun frame was not ended");
    return FVV_E_ARG;
  }
  if (f->caps.ready && device_planning_enabled()) {
    bool done = false, replayed = false;
    const int rc = run_device_planned(f, masks_dev, virt, rank_pos, frames_dev, frame_off,
                                      fallback, st, out_stage, done, true, &replayed);
    if (rc != FVV_OK) return rc;
    if (replayed) {
      fvv_frame::Pending &P = f->pend;
      P.active = true;
      P.masks = masks_dev;
      P.frames = frames_dev;
      P.has_virt = virt != nullptr;
      if (virt) P.virt = *virt;
      for (int c = 0; c < f->ncam && rank_pos; ++c) P.rank_pos[c] = rank_pos[c];
      P.has_off = frame_off != nullptr;
      for (int c = 0; c < f->ncam && frame_off; ++c) P.frame_off[c] = frame_off[c];
      P.has_fallback = fallback != nullptr;
      if (fallback) memcpy(P.fallback, fallback, 3);
      P.st = st;
      *async = true;
      return FVV_OK;
    }
  }
  return fvv_frame_run(f, masks_dev, virt, rank_pos, frames_dev, frame_off, fallback, stream,
                       out_stats, out_stage);
}

int fvv::frame_end(fvv_frame *f, fvv_frame_stats *out_stats, int *out_stage) {
  fvv_frame::Pending &P = f->pend;
  if (!P.active) {
    set_error("fvv_frame: no begun frame");
    return FVV_E_ARG;
  }
  P.active = false;
  if (out_stage) *out_stage = 0;
  if (cudaEventSynchronize(f->launched) != cudaSuccess) {
    if (out_stage) *out_stage = 8;
    return cuda_check("fvv_frame_run");
  }
  if (finish_after_sync(f, P.has_virt)) {
    if (out_stats) *out_stats = f->stats;
    return cuda_check("fvv_frame_run");
  }
  f->last_mode = 0;  // handed back by the device planner: host-planned
  const fvv_camera *virt = P.has_virt ? &P.virt : nullptr;
  const int rc = run_host_planned(f, P.masks, virt, P.rank_pos, P.frames,
                                  P.has_off ? P.frame_off : nullptr,
                                  P.has_fallback ? P.fallback : nullptr, P.st, out_stats,
                                  out_stage);
  if (rc == FVV_OK && f->seen_plannable)
    update_caps(f, f->seen_words, f->seen_tiles, f->seen_tw, f->seen_v, f->seen_s);
  return rc;
}

cudaEvent_t fvv::frame_launched_event(const fvv_frame *f) { return f->launched; }

extern "C" {

int fvv_frame_last_mode(const fvv_frame *f) { return f ? f->last_mode : -1; }

int fvv_frame_set_stage_times(fvv_frame *f, int on) {
  if (!f) return FVV_E_ARG;
  f->stage_times = on != 0;
  return FVV_OK;
}

int fvv_frame_get_outputs(const fvv_frame *f, fvv_frame_outputs *o) {
  memset(o, 0, sizeof(*o));
  o->verts = f->verts.as<double>();
  o->tris = f->tris.as<int32_t>();
  o->nv = f->nv;
  o->nt = f->nt;
  o->vis = f->vis.as<uint32_t>();
  o->vis_stride = f->vis_stride;
  o->depth = f->depth.as<double>();
  o->color = f->color.as<uint8_t>();
  o->source = f->source.as<int32_t>();
  o->covered = f->covered.as<uint8_t>();
  o->n_rois = (int64_t)f->roi_component.size();
  o->ntri_dev = f->ntri.as<int64_t>();
  return FVV_OK;
}

// flags: bit 0 depth planes, bit 1 compact colour pass (colour + the int8
// code plane instead of source + covered), bit 2 image only (no mesh or
// visibility: a frame-sharded rank ships those to rank 0 over NCCL)
static void readback_layout(const fvv_frame *f, int flags, int64_t *lay) {
  const bool compact = flags & 2;
  const bool mesh = !(flags & 4);
  const int64_t sz[7] = {mesh ? 24 * f->nv : 0,
                         mesh ? 12 * f->nt : 0,
                         mesh ? 4 * (int64_t)f->ncam * f->vis_stride : 0,
                         3 * f->virt_px,
                         (compact ? 1 : 4) * f->virt_px,
                         compact ? 0 : f->virt_px,
                         ((flags & 1) && f->nt > 0) ? 8 * f->planes : 0};
  int64_t off = 0;
  for (int i = 0; i < 7; ++i) {
    lay[i] = off;
    lay[8 + i] = sz[i];
    off += (sz[i] + 255) & ~255ll;
  }
  lay[7] = off;  // total bytes
  lay[15] = 0;
}

int64_t fvv_frame_readback_layout(const fvv_frame *f, int flags, int64_t *layout) {
  int64_t lay[16];
  readback_layout(f, flags, lay);
  if (layout) memcpy(layout, lay, sizeof(lay));
  return lay[7];
}

int fvv_frame_readback(const fvv_frame *f, void *host_dst, int flags, void *stream) {
  int64_t lay[16];
  readback_layout(f, flags, lay);
  const void *src[7] = {f->verts.p, f->tris.p, f->vis.p, f->color.p,
                        (flags & 2) ? f->code.p : f->source.p, f->covered.p, f->depth.p};
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < 7; ++i)
    if (lay[8 + i] > 0)
      cudaMemcpyAsync((char *)host_dst + lay[i], src[i], (size_t)lay[8 + i],
                      cudaMemcpyDeviceToHost, st);
  return cuda_check("fvv_frame_readback");
}

int fvv_frame_get_rois(const fvv_frame *f, int64_t *component_ids, double *boxes, fvv_grid *grids,
                   int64_t *info) {
  const size_t n = f->roi_component.size();
  if (component_ids) memcpy(component_ids, f->roi_component.data(), 8 * n);
  if (boxes) memcpy(boxes, f->roi_box.data(), 48 * n);
  if (grids) memcpy(grids, f->fine.data(), sizeof(fvv_grid) * n);
  if (info) memcpy(info, f->info.data(), 64 * n);
  return FVV_OK;
}

}  // extern "C"
