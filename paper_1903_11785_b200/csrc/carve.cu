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

// FP32 image of a camera for the certified fast path (see project_fast).
struct Cam32 {
  float R[9], t[3];
  float fx, fy, cx, cy, skew, askew;
  float eX, eY, eZ;  // bounds on |X32 - X64| etc. over the batch's voxel centres
  int fast;          // 0 when the camera has distortion: always the exact path
};

// per-camera constants staged in shared memory (lanes index different
// cameras in the run classification; divergent parameter-space loads would
// serialise)
struct CamShared {
  Cam32 f;
  int W, H, stride, pad;
  int64_t sil_off;
};

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
  Cam32 c32[FVV_MAX_CAMS];
};

constexpr float kU32 = 5.9604645e-8f;  // 2^-24

// Certified FP32 filter for one (voxel, camera) test. Returns 0 when the
// voxel is certainly outside the camera's frustum, 1 when it is certainly
// inside with rounded pixel (iu, iv), and 2 when the float64 reference chain
// must decide (u or v within the error bound of a half-integer, z near 0).
// The bound: the float32 camera coordinates differ from the float64 ones by
// at most eX/eY/eZ (6 roundings of |R||p| + |t|, host-computed with margin);
// division, scaling and the rounding of fx, cx add <= 7 u32 relative; the
// result is doubled. rint(u) is decided iff u stays farther than the bound
// from every half-integer, which also settles the image-bound tests (the
// bounds -0.5 and W-0.5 are half-integers).
__device__ __forceinline__ int project_fast(const Cam32 &c, float x, float y, float z, int W,
                                            int H, int &iu, int &iv) {
  const float X = fmaf(z, c.R[2], fmaf(y, c.R[1], x * c.R[0])) + c.t[0];
  const float Y = fmaf(z, c.R[5], fmaf(y, c.R[4], x * c.R[3])) + c.t[1];
  const float Z = fmaf(z, c.R[8], fmaf(y, c.R[7], x * c.R[6])) + c.t[2];
  if (Z < -c.eZ) return 0;  // z64 < 0: never in frustum
  if (!(Z > 4.0f * c.eZ + 1e-3f)) return 2;
  const float inv = __frcp_rn(Z);
  const float xn = X * inv, yn = Y * inv;
  const float u = fmaf(c.fx, fmaf(c.skew, yn, xn), c.cx);
  const float v = fmaf(c.fy, yn, c.cy);
  const float axn = fabsf(xn), ayn = fabsf(yn);
  const float exn = (c.eX + axn * c.eZ) * inv + 3.0f * kU32 * axn;
  const float eyn = (c.eY + ayn * c.eZ) * inv + 3.0f * kU32 * ayn;
  const float eu = 2.0f * (c.fx * (exn + c.askew * eyn) +
                           7.0f * kU32 * (c.fx * (axn + c.askew * ayn) + fabsf(u) + fabsf(c.cx))) +
                   1e-6f;
  const float ev = 2.0f * (c.fy * eyn + 7.0f * kU32 * (c.fy * ayn + fabsf(v) + fabsf(c.cy))) +
                   1e-6f;
  if (!(fabsf(u) < 4.0e6f && fabsf(v) < 4.0e6f)) return 2;
  const float ru = (u + 12582912.0f) - 12582912.0f;  // round half to even (1.5 * 2^23)
  const float rv = (v + 12582912.0f) - 12582912.0f;
  if (fabsf(u - ru) > 0.5f - eu || fabsf(v - rv) > 0.5f - ev) return 2;
  iu = (int)ru;
  iv = (int)rv;
  return (iu >= 0 && iu <= W - 1 && iv >= 0 && iv <= H - 1) ? 1 : 0;
}

enum { kSegMixed = 0, kSegFg = 1, kSegBg = 2, kSegOut = 3 };

// Certified float32 projection of a point, with its error bounds (see
// project_fast). False when z is not certainly > 0.
__device__ __forceinline__ bool project_bounds(const Cam32 &c, float x, float y, float z,
                                               float &u, float &v, float &eu, float &ev,
                                               bool &behind) {
  const float X = fmaf(z, c.R[2], fmaf(y, c.R[1], x * c.R[0])) + c.t[0];
  const float Y = fmaf(z, c.R[5], fmaf(y, c.R[4], x * c.R[3])) + c.t[1];
  const float Z = fmaf(z, c.R[8], fmaf(y, c.R[7], x * c.R[6])) + c.t[2];
  behind = Z < -c.eZ;
  if (!(Z > 4.0f * c.eZ + 1e-3f)) return false;
  const float inv = __frcp_rn(Z);
  const float xn = X * inv, yn = Y * inv;
  u = fmaf(c.fx, fmaf(c.skew, yn, xn), c.cx);
  v = fmaf(c.fy, yn, c.cy);
  const float axn = fabsf(xn), ayn = fabsf(yn);
  const float exn = (c.eX + axn * c.eZ) * inv + 3.0f * kU32 * axn;
  const float eyn = (c.eY + ayn * c.eZ) * inv + 3.0f * kU32 * ayn;
  eu = 2.0f * (c.fx * (exn + c.askew * eyn) +
               7.0f * kU32 * (c.fx * (axn + c.askew * ayn) + fabsf(u) + fabsf(c.cx))) +
       1e-5f;
  ev = 2.0f * (c.fy * eyn + 7.0f * kU32 * (c.fy * ayn + fabsf(v) + fabsf(c.cy))) + 1e-5f;
  return fabsf(u) < 4.0e6f && fabsf(v) < 4.0e6f;
}

// Status of one camera for a run of voxels along i (same j, k) whose first
// and last centres are a and b. The projection of a segment in front of the
// camera is the segment between the projected endpoints (u, v are monotone
// along it), so every voxel's rounded pixel lies in the bounding rectangle
// of the two projections widened by their error bounds:
//   kSegFg  : rectangle inside the image and all foreground -> every voxel
//             is seen by this camera and passes it;
//   kSegBg  : rectangle inside the image and all background -> every voxel
//             is seen and fails (the whole run is OFF);
//   kSegOut : run entirely behind the camera or entirely off one image side
//             -> no voxel is seen by this camera;
//   kSegMixed: anything else -> per-voxel tests.
__device__ __forceinline__ int segment_status(const Cam32 &c, int W, int H,
                                              const uint32_t *__restrict__ plane, int stride,
                                              const float *a, const float *b) {
  if (!c.fast) return kSegMixed;
  float ua, va, eua, eva, ub, vb, eub, evb;
  bool behind_a, behind_b;
  const bool ok_a = project_bounds(c, a[0], a[1], a[2], ua, va, eua, eva, behind_a);
  const bool ok_b = project_bounds(c, b[0], b[1], b[2], ub, vb, eub, evb, behind_b);
  if (behind_a && behind_b) return kSegOut;  // z affine along the run: all behind
  if (!(ok_a && ok_b)) return kSegMixed;
  const float eu = fmaxf(eua, eub), ev = fmaxf(eva, evb);
  const float fx0 = floorf(fminf(ua, ub) - eu), fx1 = ceilf(fmaxf(ua, ub) + eu);
  const float fy0 = floorf(fminf(va, vb) - ev), fy1 = ceilf(fmaxf(va, vb) + ev);
  if (fx1 < 0.0f || fy1 < 0.0f || fx0 > (float)(W - 1) || fy0 > (float)(H - 1)) return kSegOut;
  if (fx0 < 0.0f || fy0 < 0.0f || fx1 > (float)(W - 1) || fy1 > (float)(H - 1)) return kSegMixed;
  const int x0 = (int)fx0, x1 = (int)fx1, y0 = (int)fy0, y1 = (int)fy1;
  if ((x1 - x0 + 1) * (y1 - y0 + 1) > 192 || y1 - y0 > 15) return kSegMixed;
  bool any_fg = false, any_bg = false;
  const int w0 = x0 >> 5, w1 = x1 >> 5;
  for (int y = y0; y <= y1 && !(any_fg && any_bg); ++y) {
    const uint32_t *row = plane + (int64_t)y * stride;
    for (int w = w0; w <= w1; ++w) {
      uint32_t m = 0xffffffffu;
      if (w == w0) m &= 0xffffffffu << (x0 & 31);
      if (w == w1) m &= 0xffffffffu >> (31 - (x1 & 31));
      const uint32_t bits = __ldg(row + w);
      any_fg |= (bits & m) != 0u;
      any_bg |= (~bits & m) != 0u;
    }
  }
  if (!any_bg) return kSegFg;
  if (!any_fg) return kSegBg;
  return kSegMixed;
}

__global__ void __launch_bounds__(kCarveThreads)
    carve_kernel(const __grid_constant__ CarveParams p) {
  __shared__ int block_on;
  __shared__ CamShared cs[16];
  const int64_t b = blockIdx.x;
  if (threadIdx.x < 16 && threadIdx.x < p.ncam) {
    const int c = threadIdx.x;
    cs[c].f = p.c32[c];
    cs[c].W = p.cams[c].width;
    cs[c].H = p.cams[c].height;
    cs[c].stride = p.sil_stride[c];
    cs[c].sil_off = p.sil_off[c];
  }
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
    // ---- warp-level camera classification of this word's voxel runs ----
    // lanes 8q..8q+7 (run q) are consecutive voxels along i; a run that
    // crosses a row end is left unclassified. Task t = 16*q + cam (64 tasks,
    // two per lane) classifies one camera for one run.
    unsigned long long seg_fg = 0ull, seg_bg = 0ull, seg_out = 0ull;
    const int64_t lw = word * 32;
    const bool seg_ok = p.ncam <= 16 && lw < nvox && !(gemv_voxel >= lw && gemv_voxel < lw + 32);
    if (seg_ok) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int task = lane + 32 * half;
        const int q = task >> 4, cam = task & 15;
        const int64_t la = lw + 8 * q;
        int64_t lb = la + 7;
        if (lb >= nvox) lb = nvox - 1;
        int st = kSegMixed;
        if (cam < p.ncam && la < nvox && la / nx == lb / nx) {
          const int64_t key = la / nx, jj = key % ny, kk = key / ny;
          double ax, ay, az, bx, by, bz;
          voxel_center(G, la - key * nx, jj, kk, ax, ay, az);
          voxel_center(G, lb - key * nx, jj, kk, bx, by, bz);
          const float a[3] = {(float)ax, (float)ay, (float)az};
          const float bb[3] = {(float)bx, (float)by, (float)bz};
          const CamShared &k = cs[cam];
          st = segment_status(k.f, k.W, k.H, p.sil + k.sil_off, k.stride, a, bb);
        }
        seg_fg |= (unsigned long long)__ballot_sync(0xffffffffu, st == kSegFg) << (32 * half);
        seg_bg |= (unsigned long long)__ballot_sync(0xffffffffu, st == kSegBg) << (32 * half);
        seg_out |= (unsigned long long)__ballot_sync(0xffffffffu, st == kSegOut) << (32 * half);
      }
    }
    if (l < nvox) {
      const int64_t i = l % nx, j = (l / nx) % ny, k = l / (nx * ny);
      uint32_t my_fg = 0u, my_bg = 0u, my_done = 0u;
      if (seg_ok) {
        const int sh = 16 * (lane >> 3);
        my_fg = (uint32_t)(seg_fg >> sh) & 0xffffu;
        my_bg = (uint32_t)(seg_bg >> sh) & 0xffffu;
        my_done = my_fg | my_bg | ((uint32_t)(seg_out >> sh) & 0xffffu);
      }
      double x, y, z;
      voxel_center(G, i, j, k, x, y, z);
      const bool gemv = (l == gemv_voxel);
      const float xf = (float)x, yf = (float)y, zf = (float)z;
      int seen = __popc(my_fg | my_bg);
      bool keep = my_bg == 0u;
      // pass 1: certified float32 tests for the cameras the run left undecided;
      // undecided voxels are deferred so a rare float64 fallback does not
      // serialise the whole warp every camera
      unsigned long long pending = 0ull;
      for (int c = 0; c < p.ncam && keep; ++c) {
        if (c < 32 && ((my_done >> c) & 1u)) continue;
        int iu = 0, iv = 0;
        const int r = (p.c32[c].fast && !gemv)
                          ? project_fast(p.c32[c], xf, yf, zf, p.cams[c].width,
                                         p.cams[c].height, iu, iv)
                          : 2;
        if (r == 0) continue;
        if (r == 2) {
          pending |= 1ull << c;
          continue;
        }
        ++seen;
        if (!sil_bit(p.sil + p.sil_off[c], p.sil_stride[c], iu, iv)) {
          keep = false;
          break;
        }
      }
      // pass 2: the reference's float64 chain for the deferred cameras (only
      // voxels still ON need them: one background camera already decides)
      while (keep && pending) {
        const int c = __ffsll((long long)pending) - 1;
        pending &= pending - 1;
        double u, v, zc;
        if (!project_exact(p.cams[c], x, y, z, true, gemv, u, v, zc)) continue;
        ++seen;
        if (!sil_bit(p.sil + p.sil_off[c], p.sil_stride[c], (int)rint(u), (int)rint(v)))
          keep = false;
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
  // FP32 filter constants: P_j bounds |voxel centre coordinate j| over the batch
  double P[3] = {0, 0, 0};
  for (int g = 0; g < ngrid; ++g)
    for (int j = 0; j < 3; ++j) {
      const double a = fabs(grids[g].origin[j]);
      const double b = fabs(grids[g].origin[j] + grids[g].spacing * (double)grids[g].dims[j]);
      P[j] = fmax(P[j], fmax(a, b));
    }
  for (int c = 0; c < ncam; ++c) {
    const fvv_camera &k = cams[c];
    Cam32 &f = p.c32[c];
    for (int q = 0; q < 9; ++q) f.R[q] = (float)k.R[q];
    for (int q = 0; q < 3; ++q) f.t[q] = (float)k.t[q];
    f.fx = (float)k.fx;
    f.fy = (float)k.fy;
    f.cx = (float)k.cx;
    f.cy = (float)k.cy;
    f.skew = (float)k.skew;
    f.askew = fabsf((float)k.skew);
    float e[3];
    for (int r = 0; r < 3; ++r) {
      const double S = fabs(k.R[3 * r]) * P[0] + fabs(k.R[3 * r + 1]) * P[1] +
                       fabs(k.R[3 * r + 2]) * P[2] + fabs(k.t[r]);
      e[r] = (float)(8.0 * 5.9604645e-8 * S);
    }
    f.eX = e[0];
    f.eY = e[1];
    f.eZ = e[2];
    // exact path for distorted cameras and for parameters float32 cannot hold
    f.fast = !k.has_distortion && k.fx > 0 && k.fy > 0 && k.fx < 1e7 && k.fy < 1e7 &&
             fabs(k.cx) < 1e6 && fabs(k.cy) < 1e6 && fabs(k.skew) < 1e3 &&
             (P[0] + P[1] + P[2]) < 1e7 && k.width < (1 << 22) && k.height < (1 << 22);
  }
  int64_t blocks = p.blk_start[ngrid];
  if (blocks > 0x7fffffff) {
    set_error("fvv_carve: %lld blocks", (long long)blocks);
    return FVV_E_LIMIT;
  }
  carve_kernel<<<(unsigned)blocks, kCarveThreads, 0, st>>>(p);
  note_launches(1);
  return cuda_check("fvv_carve");
}
