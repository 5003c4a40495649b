// B-1 sparse carve / B-3 dense carve (hull.py:78-119, hull.py:287-302).
//
// One thread per voxel, 32 consecutive voxels (consecutive i, so their
// projections land in neighbouring silhouette words) per warp; a warp ballot
// packs the 32 ON flags into one occupancy word. Every grid of the batch
// (the coarse stage grid, or all ROI grids) is carved by one launch: blocks
// are assigned to grids by a prefix table in the parameter block.
//
// Exactness: each (voxel, camera) test runs the reference's float64 chain
// (fvv_common.cuh project_exact). A voxel stops at the first camera that
// sees it on background: it is OFF whatever the remaining cameras say
// (hull.py:91 ANDs them), so the early exit cannot change the result.
#include <cstring>

#include "fvv_common.cuh"

namespace fvv {

constexpr int kCarveThreads = 256;
constexpr int kCarveWordsPerBlock = 32;  // 1024 voxels per block

struct CarveParams {
  int ncam, ngrid, min_views, pad;
  const uint32_t *sil;
  uint32_t *occ;
  int64_t *count;
  int64_t sil_off[FVV_MAX_CAMS];
  int32_t sil_stride[FVV_MAX_CAMS];
  fvv_camera cams[FVV_MAX_CAMS];
  fvv_grid grids[FVV_MAX_GRIDS];
  int64_t word_off[FVV_MAX_GRIDS];
  int64_t blk_start[FVV_MAX_GRIDS + 1];
};

__global__ void __launch_bounds__(kCarveThreads)
    carve_kernel(const __grid_constant__ CarveParams p) {
  __shared__ int block_on;
  const int64_t b = blockIdx.x;
  int g = 0;
  while (b >= p.blk_start[g + 1]) ++g;  // uniform across the block
  const fvv_grid &G = p.grids[g];
  const int64_t nx = G.dims[0], ny = G.dims[1];
  const int64_t nvox = nx * ny * G.dims[2];
  const int64_t gemv_voxel = (nvox % kCarveChunk == 1) ? nvox - 1 : -1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) block_on = 0;
  __syncthreads();
  int my_on = 0;
  const int64_t word0 = (b - p.blk_start[g]) * kCarveWordsPerBlock;
#pragma unroll 1
  for (int it = 0; it < kCarveWordsPerBlock / (kCarveThreads / 32); ++it) {
    const int64_t word = word0 + it * (kCarveThreads / 32) + warp;
    const int64_t l = word * 32 + lane;
    bool on = false;
    if (l < nvox) {
      const int64_t i = l % nx, j = (l / nx) % ny, k = l / (nx * ny);
      double x, y, z;
      voxel_center(G, i, j, k, x, y, z);
      const bool gemv = (l == gemv_voxel);
      int seen = 0;
      bool keep = true;
      for (int c = 0; c < p.ncam; ++c) {
        const fvv_camera &cam = p.cams[c];
        double u, v, zc;
        if (!project_exact(cam, x, y, z, true, gemv, u, v, zc)) continue;
        ++seen;
        if (!sil_bit(p.sil + p.sil_off[c], p.sil_stride[c], (int)rint(u), (int)rint(v))) {
          keep = false;
          break;
        }
      }
      on = keep && seen >= p.min_views;
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, on);
    if (lane == 0 && word * 32 < nvox) {
      p.occ[p.word_off[g] + word] = bits;
      my_on += __popc(bits);
    }
  }
  if (p.count) {
    if (lane == 0 && my_on) atomicAdd(&block_on, my_on);
    __syncthreads();
    if (threadIdx.x == 0 && block_on)
      atomicAdd((unsigned long long *)&p.count[g], (unsigned long long)block_on);
  }
}

}  // namespace fvv

using namespace fvv;

extern "C" int fvv_carve(const fvv_camera *cams, int ncam, const uint32_t *sil_dev,
                         const int64_t *sil_word_off, const fvv_grid *grids, int ngrid,
                         const int64_t *word_off, int min_views, uint32_t *occ_dev,
                         int64_t *count_dev, void *stream) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("fvv_carve: %d cameras (limit %d)", ncam, FVV_MAX_CAMS);
    return ncam < 1 ? FVV_E_ARG : FVV_E_LIMIT;
  }
  if (ngrid < 0 || ngrid > FVV_MAX_GRIDS) {
    set_error("fvv_carve: %d grids (limit %d)", ngrid, FVV_MAX_GRIDS);
    return FVV_E_LIMIT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (count_dev && ngrid) {
    cudaMemsetAsync(count_dev, 0, sizeof(int64_t) * ngrid, st);
  }
  if (ngrid == 0) return FVV_OK;
  static thread_local CarveParams p;  // ~22 KB: keep it off the host stack
  memset(&p, 0, sizeof(p));
  p.ncam = ncam;
  p.ngrid = ngrid;
  p.min_views = min_views;
  p.sil = sil_dev;
  p.occ = occ_dev;
  p.count = count_dev;
  for (int c = 0; c < ncam; ++c) {
    p.cams[c] = cams[c];
    p.sil_off[c] = sil_word_off[c];
    p.sil_stride[c] = sil_stride_words(cams[c].width);
  }
  p.blk_start[0] = 0;
  for (int g = 0; g < ngrid; ++g) {
    p.grids[g] = grids[g];
    p.word_off[g] = word_off[g];
    int64_t nvox = grids[g].dims[0] * grids[g].dims[1] * grids[g].dims[2];
    if (nvox <= 0) {
      set_error("fvv_carve: grid %d has no voxels", g);
      return FVV_E_ARG;
    }
    int64_t words = (nvox + 31) / 32;
    p.blk_start[g + 1] = p.blk_start[g] + (words + kCarveWordsPerBlock - 1) / kCarveWordsPerBlock;
  }
  for (int g = ngrid; g < FVV_MAX_GRIDS; ++g) p.blk_start[g + 1] = p.blk_start[ngrid];
  int64_t blocks = p.blk_start[ngrid];
  if (blocks > 0x7fffffff) {
    set_error("fvv_carve: %lld blocks", (long long)blocks);
    return FVV_E_LIMIT;
  }
  carve_kernel<<<(unsigned)blocks, kCarveThreads, 0, st>>>(p);
  note_launches(1);
  return cuda_check("fvv_carve");
}
