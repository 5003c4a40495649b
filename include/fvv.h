/*
 * fvv.h — C ABI of the B200 free-viewpoint-video hot path (libfvv.so).
 *
 * Plain pointers and sizes only: no torch types cross this boundary. All
 * array arguments named *_dev are device pointers owned by the caller; all
 * other pointers are host memory read during the call (camera and grid
 * tables are copied into the kernel parameter block, so the call is CUDA
 * graph capturable). `stream` is a cudaStream_t (NULL = legacy default).
 * Every entry point returns 0 on success or a nonzero FVV_E_* code;
 * fvv_last_error() then describes the failure (thread-local).
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/freeview/<file>:<line>). The reference is a
 * Python library with no FFI; INTEGRATION.md shows the ctypes binding a
 * freeview maintainer would add for each entry point.
 *
 * Layouts
 *   occupancy bits : grid g's voxel l = i + nx*(j + ny*k) (voxels.py:74-96)
 *                    is bit (l & 31) of word occ_dev[word_off[g] + (l >> 5)].
 *   silhouette bits: camera c's pixel (row y, column x) is bit (x & 31) of
 *                    word sil_dev[sil_word_off[c] + y*ceil(W/32) + (x >> 5)].
 *   meshes         : vertices float64 (V,3); triangles int32 (T,3).
 */
#ifndef FVV_H
#define FVV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVV_MAX_CAMS 64   /* kernels keep the rig in the parameter block */
#define FVV_MAX_GRIDS 128 /* grids per batched carve / polygonize launch */

#define FVV_OK 0
#define FVV_E_ARG 1   /* invalid argument (message says which) */
#define FVV_E_CUDA 2  /* CUDA launch / runtime error */
#define FVV_E_LIMIT 3 /* exceeds FVV_MAX_CAMS / FVV_MAX_GRIDS / capacity */

/* camera.py:28-101 CameraModel, flattened. R maps world -> camera
 * (x_c = R x_w + t), row-major; dist order k1 k2 p1 p2 k3 (camera.py:156).
 * has_distortion = any(dist != 0) (camera.py:67-68). 192 bytes. */
typedef struct fvv_camera {
    double R[9];
    double t[3];
    double fx, fy, cx, cy, skew;
    double k1, k2, p1, p2, k3;
    int32_t width, height, id, has_distortion;
} fvv_camera;

/* voxels.py:18-71 GridSpec: voxel centre = origin + spacing*(ijk + 0.5). */
typedef struct fvv_grid {
    double origin[3];
    double spacing;
    int64_t dims[3];
} fvv_grid;

/* hull.py:23-28 Component; bbox inclusive voxel indices. */
typedef struct fvv_component {
    int64_t id, voxel_count;
    int64_t bbox_min[3], bbox_max[3];
} fvv_component;

const char *fvv_last_error(void);
int fvv_version(void);
/* Number of kernels this library has launched (all entry points). */
long long fvv_launch_count(void);

/* Stage n host (or device) buffers back to back into dst on `stream`
 * (cudaMemcpyAsync per piece, direction inferred through UVA): one frame's
 * silhouettes or colour frames in a single call (pipeline.py:150-200 hands
 * the reference per-camera arrays). Pinned sources copy asynchronously. */
int fvv_copy_gather(const void *const *src, const int64_t *bytes, int64_t n, void *dst,
                    void *stream);

/* 1 if kernels can dereference host pointer p at the same address (pinned,
 * mapped host memory under unified addressing), else 0. Colour frames that
 * pass this test are sampled in place by the colour pass (zero-copy: only
 * the bilinear taps cross PCIe) instead of being uploaded whole. */
int fvv_host_mapped(const void *p);

/* camera.py:164-201 project(cam, p, use_distortion) for n points (float64
 * (n,3)); writes pixel (n,2), camera-frame z (n,), in_frustum (n,) 0/1.
 * single_point selects numpy's 1-row BLAS order. */
int fvv_project(const fvv_camera *cam, const double *pts_dev, int64_t n, int use_distortion,
                int single_point, double *pixel_dev, double *z_dev, uint8_t *in_dev,
                void *stream);

/* Input side of hull.py:63-75 (_check_sils): uint8/bool masks, camera c's
 * (H,W) row-major mask at masks_dev + mask_off[c], -> silhouette bits. */
int fvv_pack_silhouettes(const fvv_camera *cams, int ncam, const uint8_t *masks_dev,
                         const int64_t *mask_off, uint32_t *sil_dev, const int64_t *sil_word_off,
                         void *stream);

/* hull.py:78-119 carve / hull.py:287-302 dense_carve: one launch carves
 * ngrid grids (the coarse stage grid, or every ROI grid) against the rig.
 * Voxel ON iff in-frustum for >= min_views cameras and every camera that
 * sees it hits foreground. Also writes per-grid ON counts (int64 [ngrid])
 * to count_dev when non-NULL (zeroed by the call). */
int fvv_carve(const fvv_camera *cams, int ncam, const uint32_t *sil_dev,
              const int64_t *sil_word_off, const fvv_grid *grids, int ngrid,
              const int64_t *word_off, int min_views, uint32_t *occ_dev,
              int64_t *count_dev, void *workspace, size_t ws_bytes, void *stream);
/* Device workspace fvv_carve needs for these cameras: per-(grid, camera)
 * FP32 projection coefficients, 8x8-pixel silhouette cell maps, and the
 * queue of voxels its certified FP32 pass leaves to the float64 chain. */
size_t fvv_carve_workspace_bytes(const fvv_camera *cams, int ncam);

/* voxels.py:100-162 save_grid: the bit transitions of an occupancy field
 * (bit l != bit l-1, bit -1 OFF), in ascending order, into pos_dev (capacity
 * nvox) and their number into *count_dev; run lengths are the differences of
 * [0, pos..., nvox]. */
size_t fvv_rle_workspace_bytes(int64_t nvox);
int fvv_rle_transitions(const uint32_t *occ_dev, int64_t nvox, int64_t *pos_dev,
                        int64_t *count_dev, void *ws_dev, size_t ws_bytes, void *stream);

/* ---- B-2: hull.py:122-269 ------------------------------------------------ */

/* Device workspace fvv_ccl26 needs for `grid` (compacted ON-voxel ranks,
 * union-find forest, per-component stats). */
size_t fvv_ccl_workspace_bytes(const fvv_grid *grid);

/* hull.py:218-254 label_components: 26-connected labelling of occ_dev.
 * Labels 1..n ascend with each component's minimum linear index (the
 * reference's canonical numbering). Writes min(n, comp_cap) component
 * records (id, count, inclusive bbox) to comps_dev and {n_on, n} to
 * counts_dev[0..1]; the labelling itself stays in the workspace. */
int fvv_ccl26(const uint32_t *occ_dev, const fvv_grid *grid, void *ws_dev, size_t ws_bytes,
              fvv_component *comps_dev, int64_t comp_cap, int64_t *counts_dev, void *stream);

/* Re-export component records from a labelled workspace (larger buffer). */
int fvv_ccl_components(const fvv_grid *grid, const void *ws_dev, fvv_component *comps_dev,
                       int64_t comp_cap, void *stream);

/* Dense int32 labels (0 = background) of a labelled workspace: the
 * reference's Labeling.labels (hull.py:31-34). */
int fvv_ccl_labels(const fvv_grid *grid, const void *ws_dev, int32_t *labels_dev, void *stream);

/* hull.py:257-269 filter_noise on a labelled workspace: keep_dev[label]
 * (uint8, indexed 0..n) selects survivors, ids unchanged. Writes the
 * filtered dense labels and/or occupancy bits (either may be NULL) and the
 * surviving voxel count. */
int fvv_filter_labels(const fvv_grid *grid, const void *ws_dev, const uint8_t *keep_dev,
                      int32_t *labels_dev, uint32_t *occ_dev, int64_t *kept_dev, void *stream);

/* The same filter for a caller-supplied dense label array (nkeep entries
 * in keep_dev). */
int fvv_filter_dense(const int32_t *labels_in_dev, int64_t nvox, const uint8_t *keep_dev,
                     int64_t nkeep, int32_t *labels_dev, uint32_t *occ_dev, int64_t *kept_dev,
                     void *stream);

/* ---- C: mesh.py:131-374 --------------------------------------------------- */

/* Workspace of fvv_mesh_prepare / fvv_mesh_emit for a batch of grids. */
size_t fvv_mesh_workspace_bytes(const fvv_grid *grids, int ngrid);

/* Phase A of mesh.py:275-374 polygonize, batched over ngrid grids (their
 * occupancy bits at occ_dev + word_off[g]): transposes occupancy into
 * k-rows and scans intersected grid edges (vertices, in the reference's
 * (axis, i, j, k) order) and surface cells. Grids with a dimension < 2
 * yield empty meshes (mesh.py:298-299). Counts are read with
 * fvv_mesh_counts. */
int fvv_mesh_prepare(const fvv_grid *grids, int ngrid, const uint32_t *occ_dev,
                     const int64_t *word_off, void *ws_dev, size_t ws_bytes, void *stream);

/* Copies totals {V, S, T} (int64[3]) and per-grid info int64[ngrid][8] =
 * {vbase, V, sbase, S, tbase, T, fallback_edges, inconsistent_starts}
 * (IsovalueStats, mesh.py:225-228) out of the workspace. T fields are valid
 * after fvv_mesh_emit. */
int fvv_mesh_counts(const fvv_grid *grids, int ngrid, const void *ws_dev, int64_t *totals_dev,
                    int64_t *info_dev, void *stream);

/* Scratch fvv_mesh_emit needs for V vertices and S surface cells. */
size_t fvv_mesh_emit_scratch_bytes(int64_t num_vertices, int64_t num_cells);

/* Phase B: per-edge isovalues (exact: mesh.py:231-272 with cameras given in
 * ascending id order; else fixed_iso), vertices p_on + lam*(p_off - p_on)
 * (float64 [V][3], grid-major), triangles (int32 [<=5S][3], indices into
 * verts_dev, slot-major per grid, winding reversed, area <= 1e-9 dropped). */
int fvv_mesh_emit(const fvv_camera *cams_by_id, int ncam, const uint32_t *sil_dev,
                  const int64_t *sil_word_off, const fvv_grid *grids, int ngrid,
                  const uint32_t *occ_dev, const int64_t *word_off, int exact, double fixed_iso,
                  void *ws_dev, size_t ws_bytes, int64_t num_vertices, int64_t num_cells,
                  void *scratch_dev, size_t scratch_bytes, double *verts_dev, int32_t *tris_dev,
                  void *stream);

/* mesh.py:231-272 _edge_isovalues_batch on explicit endpoints (n,3):
 * lam (n,), contributing camera id (n,) (-1 = fallback 0.5), stats int64[2]
 * = {fallback_edges, inconsistent_starts}. */
int fvv_edge_isovalues(const fvv_camera *cams_by_id, int ncam, const uint32_t *sil_dev,
                       const int64_t *sil_word_off, const double *p_on_dev,
                       const double *p_off_dev, int64_t n, double *lam_dev, int32_t *cam_dev,
                       int64_t *stats_dev, void *stream);

/* ---- D-1 / D-2: visibility.py:34-140 --------------------------------------- */

/* Scratch for fvv_rasterize: projected vertices of every camera (float64
 * records + float-rounded (u, v) for the FP32 filter), the FP32 filter's
 * per-warp (item, pixel) pair lists and sweep-item lists, and the queue of
 * large-bbox triangles (~40 B per camera-vertex + 20 B per camera-triangle). */
size_t fvv_raster_workspace_bytes(int64_t num_vertices, int64_t num_triangles, int ncam);

/* visibility.py:34-98 rasterize for ncam cameras at once (zero-distortion
 * projection, near clip 1 mm, top-left rule, perspective-correct depth).
 * Camera c's float64 depth plane (+inf background) is depth_dev +
 * plane_off[c]; when tri_id_dev is non-NULL its int32 winning-triangle
 * plane (-1 background; lowest id on exact depth ties) is tri_id_dev +
 * plane_off[c]. The triangle count is *nt_dev when nt_dev is non-NULL
 * (nt is then an upper bound), else nt. Limits: nt * ncam < 2^32 - 1 and
 * image sides <= 65535 (FVV_E_LIMIT otherwise). */
int fvv_rasterize(const fvv_camera *cams, int ncam, const double *verts_dev, int64_t nv,
                  const int32_t *tris_dev, int64_t nt, const int64_t *nt_dev, double *depth_dev,
                  const int64_t *plane_off, int32_t *tri_id_dev, void *ws_dev, size_t ws_bytes,
                  void *stream);

/* fvv_rasterize for planes that persist across calls (the frame executor's):
 * depth (and tri_id) planes contiguous from plane_off[0], already holding the
 * background except the 32-pixel tiles flagged in dirty_dev (one byte per
 * tile of plane 0's element index / 32, ceil(total_px / 32) bytes), which
 * are reset first; the call flags the tiles it writes. The vertex count is
 * *nv_dev when nv_dev is non-NULL (nv: the capacity, the records' stride),
 * like nt / nt_dev. full_reset != 0 fills
 * the planes and clears the map instead (first use, or new buffers). Same
 * results as fvv_rasterize; only the background writes differ. */
int fvv_rasterize_tracked(const fvv_camera *cams, int ncam, const double *verts_dev, int64_t nv,
                          const int64_t *nv_dev, const int32_t *tris_dev, int64_t nt,
                          const int64_t *nt_dev,
                          double *depth_dev, const int64_t *plane_off, int32_t *tri_id_dev,
                          void *ws_dev, size_t ws_bytes, uint8_t *dirty_dev, int full_reset,
                          void *stream);

/* visibility.py:106-129 classify_visibility for ncam cameras: triangle t
 * visible in camera c iff its centroid projects in-frustum and
 * z - depth[rint v, rint u] <= t_v. Bit t of vis_dev + c*vis_stride_words. */
int fvv_classify(const fvv_camera *cams, int ncam, const double *verts_dev,
                 const int32_t *tris_dev, int64_t nt, const int64_t *nt_dev,
                 const double *depth_dev, const int64_t *plane_off, double t_v,
                 uint32_t *vis_dev, int64_t vis_stride_words, void *stream);

/* ---- E: render.py:29-113, camera.py:204-220 --------------------------------- */

/* render.py:35-43 triangle_sources: first ranked camera (rig position
 * rank_pos[r], id rank_id[r]) whose visibility bit is set; -1 if none. */
int fvv_triangle_sources(const int32_t *rank_pos, const int32_t *rank_id, int nrank,
                         const uint32_t *vis_dev, int64_t vis_stride_words, int64_t nt,
                         const int64_t *nt_dev, int32_t *src_dev, void *stream);

/* render.py:96-110 bookkeeping of render_view: int64 counts_dev[1 + ncam] =
 * {covered pixels, pixels sourced from rig camera c ...} of the virtual view
 * (tri_id_dev from fvv_rasterize, tri_src_dev from fvv_triangle_sources).
 * A count of 1 selects numpy's one-row BLAS order downstream, and the
 * non-zero entries say which cameras' frames the colour pass reads. */
int fvv_render_count(const fvv_camera *rig, int ncam, const fvv_camera *virt,
                     const int32_t *tri_id_dev, const int32_t *tri_src_dev, int64_t *counts_dev,
                     void *stream);

/* render.py:64-113 render_view colour pass, given the virtual view's depth /
 * triangle-id planes, per-triangle source ids and fvv_render_count's counts:
 * back-projects each covered pixel, projects it (with distortion) into its
 * source camera and samples that camera's (H,W,3) uint8 frame (frames_dev +
 * frame_off[c], rig order; only cameras with a non-zero count are read)
 * bilinearly; fallback colour where no camera sees the triangle. */
int fvv_render_view(const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                    const int64_t *frame_off, const fvv_camera *virt, const double *depth_dev,
                    const int32_t *tri_id_dev, const int32_t *tri_src_dev, const uint8_t *fallback,
                    uint8_t *color_dev, int32_t *source_dev, uint8_t *covered_dev,
                    const int64_t *counts_dev, void *stream);
/* The same, also writing an int8 code per pixel (-2 uncovered, -1 fallback,
 * else the source camera's rig position; code_dev may be NULL). */
int fvv_render_view_coded(const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                          const int64_t *frame_off, const fvv_camera *virt,
                          const double *depth_dev, const int32_t *tri_id_dev,
                          const int32_t *tri_src_dev, const uint8_t *fallback,
                          uint8_t *color_dev, int32_t *source_dev, uint8_t *covered_dev,
                          int8_t *code_dev, const int64_t *counts_dev, void *stream);

/* camera.py:204-220 back_project for n pixels (n,2) at depths (n,) -> (n,3). */
int fvv_back_project(const fvv_camera *cam, const double *pixel_dev, const double *depth_dev,
                     int64_t n, double *out_dev, void *stream);

/* ---- silhouettes: silhouette.py:59-109 (upstream of the hot path) ---- */

/* silhouette.py:59-69 distance_map of one (H, W) uint8 proposal: exact
 * squared Euclidean distance to the nearest proposal pixel (int32,
 * INT32_MAX when the proposal is empty) and, when dm_dev != NULL, its
 * float64 sqrt (+inf when empty) = scipy distance_transform_edt(~prop).
 * ws_dev: int32 scratch of H*W. */
int fvv_distance_map(const uint8_t *prop_dev, int64_t H, int64_t W, int32_t *sqdist_dev,
                     double *dm_dev, int32_t *ws_dev, void *stream);

/* silhouette.py:72-87 build_background: per element of n = H*W*C, mean and
 * population std (floor 2.0) over K uint8 frames stacked frame-major. */
int fvv_background(const uint8_t *frames_dev, int64_t K, int64_t n, double *mean_dev,
                   double *std_dev, void *stream);

/* silhouette.py:90-109 extract_silhouette with AdaptiveParams.threshold:
 * uint8 mask = max_c |frame - mean| / std > theta(distance). Distances from
 * dm_dev (float64) when non-NULL, else from fvv_distance_map's sqdist_dev. */
int fvv_extract_silhouette(const uint8_t *frame_dev, const double *mean_dev,
                           const double *std_dev, int64_t npx, int C, const int32_t *sqdist_dev,
                           const double *dm_dev, double theta_near, double theta_far,
                           double d_max, uint8_t *mask_dev, void *stream);

/* ---- native frame executor: pipeline.py:115-220 run_frame + render.py:64-113 ---- */

typedef struct fvv_frame fvv_frame;

/* PipelineConfig (pipeline.py:41-101) with derived defaults resolved
 * (roi_margin, t_v); t_large may be +inf; budget = GridSpec voxel budget. */
typedef struct fvv_frame_config {
    double stage_lo[3], stage_hi[3];
    double coarse_spacing, fine_spacing, roi_margin, t_v, t_large, fixed_isovalue;
    int64_t t_small, budget;
    int32_t min_views, exact;
} fvv_frame_config;

/* run_frame's stats dict (pipeline.py:152-196) + sizes + device stage times
 * (ms: B-1, B-2, B-3, C, D-1, D-2, E, readback). */
typedef struct fvv_frame_stats {
    int64_t sparse_tests, sparse_occupied, components, dense_tests, dense_occupied,
        fallback_edges, inconsistent_edge_starts, triangles, vertices, n_rois;
    float ms[8];
    /* colour pass: covered virtual pixels, pixels sampled from a rig camera */
    int64_t covered_px, sourced_px;
} fvv_frame_stats;

/* How the last fvv_frame_run ran: 0 host-planned (first frame, or a frame
 * the device planner handed back), 1 device-planned enqueue, 2 device-planned
 * graph capture + launch, 3 graph replay. */
int fvv_frame_last_mode(const fvv_frame *f);

/* Whether device-planned frames read their per-stage device times back into
 * fvv_frame_stats.ms (default 1; the readout costs ~22 us of host time per
 * frame). 0: ms is zero-filled. */
int fvv_frame_set_stage_times(fvv_frame *f, int on);

/* Device outputs of the last fvv_frame_run (valid until the next run):
 * merged-order triangles indexing verts (per-ROI slices via fvv_frame_rois),
 * visibility bits (ncam x vis_stride words), depth planes (rig order,
 * H*W each), virtual-view colour/source/covered. */
typedef struct fvv_frame_outputs {
    double *verts;
    int32_t *tris;
    int64_t nv, nt;
    uint32_t *vis;
    int64_t vis_stride;
    double *depth;
    uint8_t *color;
    int32_t *source;
    uint8_t *covered;
    int64_t n_rois;
    int64_t *ntri_dev;
} fvv_frame_outputs;

/* Executor for a fixed rig and config; device buffers persist across runs. */
fvv_frame *fvv_frame_create(const fvv_camera *cams, int ncam, const fvv_frame_config *cfg);
void fvv_frame_destroy(fvv_frame *frame);

/* One frame: silhouette masks (uint8, rig order, camera c at
 * masks_dev + sum of previous H*W) -> B-1 .. D-2, and when virt != NULL the
 * colour pass from frames_dev + frame_off[c] (bytes; device memory or
 * mapped pinned host memory, see fvv_host_mapped) with the
 * camera ranking rank_pos (rig positions, render.py:29-32). On failure
 * *out_stage names the stage (1 B-1, 2 B-2, 3 B-3, 4 C, 5 D-1, 6 D-2, 7 E). */
int fvv_frame_run(fvv_frame *frame, const uint8_t *masks_dev, const fvv_camera *virt,
                  const int32_t *rank_pos, const uint8_t *frames_dev, const int64_t *frame_off,
                  const uint8_t *fallback, void *stream, fvv_frame_stats *out_stats,
                  int *out_stage);
int fvv_frame_get_outputs(const fvv_frame *frame, fvv_frame_outputs *out);
/* Host copy of the last run's outputs in one pinned block: layout[0..6] =
 * byte offsets of verts, tris, visibility bits, colour, source, covered,
 * depth planes (depth only with flag bit 0), layout[8..14] their sizes,
 * layout[7] the total; returns the total. fvv_frame_readback queues the
 * device->host copies into host_dst (pinned, >= total bytes) on stream. */
int64_t fvv_frame_readback_layout(const fvv_frame *frame, int flags, int64_t *layout);
int fvv_frame_readback(const fvv_frame *frame, void *host_dst, int flags, void *stream);
/* flags: bit 0 = depth planes; bit 1 = compact colour pass: slot 4 holds an
 * int8 code per virtual pixel (-2 uncovered, -1 fallback colour, else the
 * source camera's rig position) and slot 5 is empty, instead of int32
 * source ids + uint8 coverage (render.py:64-113's outputs follow from it);
 * bit 2 = image only: slots 0-2 (mesh, visibility) are empty, for a
 * frame-sharded rank that sends those to rank 0 from device memory. */
/* Per ROI: component id, box lo/hi (6 doubles), fine grid, mesh info
 * {vbase, V, sbase, S, tbase, T, fallback_edges, inconsistent_starts}. */
int fvv_frame_get_rois(const fvv_frame *frame, int64_t *component_ids, double *boxes,
                   fvv_grid *grids, int64_t *info);

/* ---- native sequence runner: pipeline.run_sequence's engine ------------------ */
/* `lanes` host threads, each with its own CUDA streams and two frame
 * executors, run frames n = lane (mod lanes) of a video sequence: the
 * silhouette upload, fvv_frame_run and one fvv_frame_readback into a pooled
 * pinned block per frame (pipeline.py:115-220 + render.py:64-113 per frame,
 * pipelined over threads as PAPER.md:561 describes). Results come back in
 * submission order and own their outputs until fvv_seq_result_free. */
typedef struct fvv_seq fvv_seq;
typedef struct fvv_seq_result fvv_seq_result;

typedef struct fvv_seq_config {
    int32_t lanes;
    int32_t readback_flags;   /* fvv_frame_readback flags (bit 1: compact colour) */
    int32_t has_virtual;      /* run the colour pass for virt */
    int32_t export_payload;   /* mesh + visibility into a device payload, not read back */
    fvv_camera virt;
    int32_t rank_pos[FVV_MAX_CAMS];  /* render.py:29-32 ranking (rig positions) */
    uint8_t fallback[4];             /* render.py:19 FALLBACK_COLOR */
} fvv_seq_config;

typedef struct fvv_seq_result_info {
    int64_t id;
    int32_t status, stage;    /* fvv_frame_run status; stage as its out_stage */
    const char *err;
    fvv_frame_stats stats;
    int64_t nv, nt, vis_stride, n_rois;
    const int64_t *component_ids;  /* n_rois */
    const double *boxes;           /* n_rois x 6 */
    const fvv_grid *grids;         /* n_rois */
    const int64_t *roi_info;       /* n_rois x 8, as fvv_frame_get_rois */
    int64_t layout[16];            /* fvv_frame_readback_layout of the pinned block */
    const void *host;              /* the pinned block */
    void *payload_dev;             /* export: verts | tris | visibility bits (256-aligned) */
    int64_t payload_bytes;
} fvv_seq_result_info;

fvv_seq *fvv_seq_create(const fvv_camera *cams, int ncam, const fvv_frame_config *cfg,
                        const fvv_seq_config *seq_cfg);
void fvv_seq_destroy(fvv_seq *seq);
/* Queue frame `id`: nmask silhouette buffers (one rig-order buffer or one per
 * camera; host pageable/pinned or device) with their byte sizes, and per
 * camera colour frames (H, W, 3) uint8 or NULL. Inputs must stay alive until
 * the frame's result is returned. Blocks while the lane holds 2 queued frames. */
int fvv_seq_submit(fvv_seq *seq, int64_t id, const void *const *mask_src,
                   const int64_t *mask_bytes, int nmask, const void *const *frame_src);
/* Next result in submission order (its copies complete): 1 = *out set, 0 =
 * none pending (or, with wait = 0, none ready yet). */
int fvv_seq_next(fvv_seq *seq, int wait, fvv_seq_result **out);
int fvv_seq_result_get(const fvv_seq_result *res, fvv_seq_result_info *info);
void fvv_seq_result_free(fvv_seq_result *res);
/* sizeof of the ABI records (fvv_camera, fvv_grid, fvv_component,
 * fvv_frame_config, fvv_frame_stats, fvv_frame_outputs, fvv_seq_config,
 * fvv_seq_result_info) into out[0..n): bindings check their layouts. */
int fvv_abi_sizes(int64_t *out, int n);

/* ---- harness (not hot path): synthetic scene inputs ------------------------- */

/* synthetic.py:165-218 for the reference's Sphere/Box scenes: per pixel of
 * `cam` (zero distortion) the centre ray (camera.py:223-235), the nearest hit
 * over objs_dev (nobj records of 10 doubles: sphere {0, centre[3], r^2,
 * colour[3], 0, 0}, box {1, lo[3], hi[3], colour[3]}), the analytic
 * silhouette (uint8 (H,W), optional) and the Lambertian frame (uint8
 * (H,W,3), optional; shading = {ambient, 1 - ambient, background rgb},
 * light = unit light direction, noise_dev = optional (H,W,3) float64 added
 * before rounding). */
int fvv_synth_render(const fvv_camera *cam, const double *light, const double *shading,
                     const double *objs_dev, int nobj, const double *noise_dev,
                     uint8_t *sil_dev, uint8_t *rgb_dev, void *stream);
/* synthetic.py:221-226: binary erosion with the 3x3 cross, `iterations`
 * times, outside pixels 0 (scipy.ndimage.binary_erosion defaults). */
int fvv_erode_cross(const uint8_t *in_dev, uint8_t *tmp_dev, uint8_t *out_dev, int width,
                    int height, int iterations, void *stream);

/* Ray-cast nparts ellipsoids (float64 records: centre[3], orientation[9]
 * row-major (columns = ellipsoid axes), semi-axes[3], rgb[3]) into camera
 * `cam`: silhouette uint8 (H,W) and Lambertian frame uint8 (H,W,3); either
 * output may be NULL. shading = {ambient, light dir xyz, background rgb}.
 * GPU twin of synthetic.py render_camera (reference synthetic.py:165-218). */
int fvv_render_ellipsoids(const fvv_camera *cam, const double *parts_dev, int nparts,
                          uint8_t *sil_dev, uint8_t *rgb_dev, const double *shading,
                          void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FVV_H */
