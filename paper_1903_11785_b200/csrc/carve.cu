// B-1 sparse carve / B-3 dense carve (hull.py:78-119, hull.py:287-302).
//
// One thread per voxel, 32 consecutive voxels (consecutive i, so their
// projections land in neighbouring silhouette words) per warp; a warp ballot
// packs the 32 ON flags into one occupancy word. Every grid of the batch
// (the coarse stage grid, or all ROI grids) is carved by one launch: blocks
// are assigned to grids by a prefix table in the parameter block.
//
// Exactness: each (voxel, camera) test is decided either by a certified
// FP32 evaluation (below) or by the reference's float64 chain
// (fvv_common.cuh project_exact); both give the reference's pixel. A voxel
// stops at the first camera that sees it on background: it is OFF whatever
// the remaining cameras say (hull.py:91 ANDs them), so the early exit
// cannot change the result.
#include <cstring>

#include "fvv_common.cuh"

namespace fvv {

constexpr int kCarveThreads = 256;
constexpr int kCarveWordsPerBlock = 128;  // 4096 voxels per block
constexpr int64_t kAmbCap = 1 << 20;     // deferred-voxel queue entries

struct CarveParams {
  int ncam, ngrid, min_views, pad;
  const uint32_t *sil;
  uint32_t *occ;
  int64_t *count;
  unsigned long long *amb;  // [0] = queued voxels, then (grid << 40 | voxel) entries
  int64_t amb_cap;
  int k1;                    // cameras order[0 .. k1) are tested in phase 1
  int order[FVV_MAX_CAMS];   // camera test order (a permutation of 0 .. ncam-1)
  int64_t sil_off[FVV_MAX_CAMS];
  int32_t sil_stride[FVV_MAX_CAMS];
  fvv_camera cams[FVV_MAX_CAMS];
  fvv_grid grids[FVV_MAX_GRIDS];
  int64_t word_off[FVV_MAX_GRIDS];
  int64_t blk_start[FVV_MAX_GRIDS + 1];
};

// ---- FP32 pre-classification --------------------------------------------
// Without distortion, u = U/Z and v = V/Z with (U, V, Z) affine in the voxel
// indices (i, j, k): U = U0 + i Ui + j Uj + k Uk (K [R|t] applied to the
// voxel centre). Each (voxel, camera) test is first evaluated in FP32 from
// these per-(grid, camera) coefficients together with a rigorous bound E on
// |u32 - u| (and on v, Z). When u32 (v32) is farther than E from every
// half-integer, rint(u) of the reference's float64 chain equals rintf(u32),
// so the test's outcome (frustum, silhouette bit) is decided exactly in
// FP32. Otherwise the camera is "ambiguous"; a voxel with an ambiguous
// camera and no camera that rejects it is re-run through the float64 chain.
// Bound: with eps = 2^-24 and S = |U0| + i|Ui| + j|Uj| + k|Uk| (bounded by
// its value at the far grid corner), coefficient rounding plus the three
// fmaf roundings give |U32 - U| <= 4 eps S_U (same for Z); then
// |U32/Z32 - U/Z| <= 4 eps (S_U + |u| S_Z) / Z32, plus 8.5 eps |u| for the
// approximate reciprocal (__fdividef: <= 2 ulp) and the product; the float64
// chain's own error (< 1e-9 px at these magnitudes) is covered by an
// absolute 2^-12; the whole bound is doubled (and the per-camera constants
// inflated by 1%). The sign of Z is certain once |Z32| > ez; when every
// voxel of the grid has Z beyond that (Z is affine, its minimum is at a
// grid corner) the sign checks are skipped. A |u32| beyond ulim lies outside
// the image whatever its rounding. Cameras with lens distortion always take
// the float64 chain (ez = inf).
struct __align__(16) CamAffine {
  float u[4], v[4], z[4];  // constant, i, j, k coefficients
  float su, sv, sz, ez;    // magnitude sums at the far corner; |Z32 - Z| bound
  float zsafe, ulim, bu, bv;  // fast path (Z32 >= zsafe): eu = (|u|+1)(A rz + C) + bu rz + 2^-12
  float A;                 // 8 eps sz
  int w, h, pad0;
};

constexpr float kEps = 5.9604645e-8f;  // 2^-24

__device__ __forceinline__ void cam_affine(const fvv_camera &c, const fvv_grid &g, CamAffine &a) {
  const double hs = 0.5 * g.spacing;
  const double ox = g.origin[0] + hs, oy = g.origin[1] + hs, oz = g.origin[2] + hs;
  // rows of K [R|t] (no distortion): U = fx X + fx skew Y + cx Z, V = fy Y + cy Z
  double ku[4], kv[4], kz[4];
  for (int m = 0; m < 3; ++m) {
    const double rx = c.R[m], ry = c.R[3 + m], rz = c.R[6 + m];  // column m of R
    ku[1 + m] = g.spacing * (c.fx * rx + c.fx * c.skew * ry + c.cx * rz);
    kv[1 + m] = g.spacing * (c.fy * ry + c.cy * rz);
    kz[1 + m] = g.spacing * rz;
  }
  const double X = c.R[0] * ox + c.R[1] * oy + c.R[2] * oz + c.t[0];
  const double Y = c.R[3] * ox + c.R[4] * oy + c.R[5] * oz + c.t[1];
  const double Z = c.R[6] * ox + c.R[7] * oy + c.R[8] * oz + c.t[2];
  ku[0] = c.fx * X + c.fx * c.skew * Y + c.cx * Z;
  kv[0] = c.fy * Y + c.cy * Z;
  kz[0] = Z;
  const double n[3] = {(double)(g.dims[0] - 1), (double)(g.dims[1] - 1), (double)(g.dims[2] - 1)};
  double su = fabs(ku[0]), sv = fabs(kv[0]), sz = fabs(kz[0]), zmin = kz[0];
  for (int m = 0; m < 3; ++m) {
    su += n[m] * fabs(ku[1 + m]);
    sv += n[m] * fabs(kv[1 + m]);
    sz += n[m] * fabs(kz[1 + m]);
    zmin += fmin(0.0, n[m] * kz[1 + m]);
  }
  for (int m = 0; m < 4; ++m) {
    a.u[m] = (float)ku[m];
    a.v[m] = (float)kv[m];
    a.z[m] = (float)kz[m];
  }
  // the double-side sums above carry ~1e-16 relative error; inflate slightly
  su *= 1.0001;
  sv *= 1.0001;
  sz *= 1.0001;
  a.su = (float)su;
  a.sv = (float)sv;
  a.sz = (float)sz;
  const double e4 = 4.0 * (double)kEps;
  const double ez = 2.0 * e4 * sz + 1e-6;
  a.ez = c.has_distortion ? INFINITY : (float)ez;
  a.w = c.width;
  a.h = c.height;
  const double ulim = (double)(c.width > c.height ? c.width : c.height) + 2.0;
  a.ulim = (float)ulim;
  // every voxel has Z >= zmin, so Z32 >= zmin - ez; below zsafe the per-test
  // sign checks run first
  const double zsafe = (zmin - 2.0 * ez) * (1.0 - 1e-6);
  a.zsafe = (!c.has_distortion && zsafe > ez) ? (float)zsafe : INFINITY;
  a.A = (float)(8.0 * (double)kEps * sz * 1.01);
  a.bu = (float)(8.0 * (double)kEps * su * 1.01);
  a.bv = (float)(8.0 * (double)kEps * sv * 1.01);
}

enum : int { kOut = 0, kIn = 1, kAmb = 2 };

// FP32 classification of one (voxel, camera): kOut (not in frustum), kIn
// (in frustum at pixel (px, py)), kAmb (undecided in FP32).
__device__ __forceinline__ int classify32(const CamAffine &a, float fi, float fj, float fk,
                                          int &px, int &py) {
  const float Z = fmaf(fk, a.z[3], fmaf(fj, a.z[2], fmaf(fi, a.z[1], a.z[0])));
  const float U = fmaf(fk, a.u[3], fmaf(fj, a.u[2], fmaf(fi, a.u[1], a.u[0])));
  const float V = fmaf(fk, a.v[3], fmaf(fj, a.v[2], fmaf(fi, a.v[1], a.v[0])));
  // E = 2 (4 eps (|u| S_Z + S_U) / Z + 8.5 eps |u|) + 2^-12, |u| -> |u32| + 1
  if (!(Z >= a.zsafe)) {
    if (Z <= -a.ez) return kOut;  // Z < 0 for certain
    if (Z < a.ez) return kAmb;
  }
  const float rz = __fdividef(1.0f, Z);
  const float k = fmaf(a.A, rz, 17.0f * kEps);
  const float eu = fmaf(fabsf(U * rz) + 1.0f, k, fmaf(a.bu, rz, 2.44140625e-4f));
  const float ev = fmaf(fabsf(V * rz) + 1.0f, k, fmaf(a.bv, rz, 2.44140625e-4f));
  const float u = U * rz, v = V * rz;
  const float ru = rintf(u), rv = rintf(v);
  px = (int)ru;
  py = (int)rv;
  const bool in = (unsigned)px < (unsigned)a.w && (unsigned)py < (unsigned)a.h;
  // beyond ulim the point is off the image whatever its rounding
  const bool amb = (fabsf(u - ru) >= 0.5f - eu && fabsf(u) <= a.ulim) ||
                   (fabsf(v - rv) >= 0.5f - ev && fabsf(v) <= a.ulim);
  return amb ? kAmb : (in ? kIn : kOut);
}

// The reference's float64 chain for one voxel (hull.py:83-91).
__device__ __forceinline__ bool carve_exact(const CarveParams &p, const fvv_grid &G, int64_t l) {
  const int64_t nx = G.dims[0], ny = G.dims[1];
  const int64_t nvox = nx * ny * G.dims[2];
  const int64_t i = l % nx, j = (l / nx) % ny, k = l / (nx * ny);
  double x, y, z;
  voxel_center(G, i, j, k, x, y, z);
  const bool gemv = (nvox % kCarveChunk == 1) && l == nvox - 1;  // 1-row BLAS chunk
  int seen = 0;
  for (int c = 0; c < p.ncam; ++c) {
    double u, v, zc;
    if (!project_exact(p.cams[c], x, y, z, true, gemv, u, v, zc)) continue;
    ++seen;
    if (!sil_bit(p.sil + p.sil_off[c], p.sil_stride[c], (int)rint(u), (int)rint(v)))
      return false;
  }
  return seen >= p.min_views;
}

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

// Cameras order[t0 .. t1) against one voxel in FP32: sets off on a
// background view, counts in-frustum views, flags undecided tests.
__device__ __forceinline__ void test_cams(const CarveParams &p, const CamAffine *aff, int t0,
                                          int t1, float fi, float fj, float fk, int &seen,
                                          bool &off, bool &amb) {
  for (int t = t0; t < t1; ++t) {
    const int c = p.order[t];
    int px, py;
    const int st = classify32(aff[c], fi, fj, fk, px, py);
    if (st == kOut) continue;
    if (st == kAmb) {
      amb = true;
      continue;
    }
    ++seen;
    if (!sil_bit(p.sil + p.sil_off[c], p.sil_stride[c], px, py)) {
      off = true;  // hull.py:91: one background view removes the voxel
      return;
    }
  }
}

// A voxel no FP32 camera rejected: ON/OFF from the counts, or, when a test
// was undecided, the float64 chain (deferred to carve_exact_kernel).
__device__ __forceinline__ bool settle(const CarveParams &p, const fvv_grid &G, int g, int64_t l,
                                       int seen, bool amb) {
  if (!amb) return seen >= p.min_views;
  if (p.amb) {
    const unsigned long long slot = atomicAdd(p.amb, 1ull);
    if ((int64_t)slot < p.amb_cap) {
      p.amb[1 + slot] = ((unsigned long long)g << 40) | (unsigned long long)l;
      return false;  // its bit is set by carve_exact_kernel
    }
  }
  return carve_exact(p, G, l);
}

// Two phases per block of 4096 voxels. Phase 1: every voxel against the
// first p.k1 cameras of p.order (spread around the rig, so most voxels
// outside the hull are rejected here); survivors are compacted into a
// shared-memory queue with their partial view count. Phase 2: the block's
// threads take the queue densely against the remaining cameras, so a few ON
// voxels no longer hold whole warps for all cameras. The AND over cameras
// and the view count do not depend on the order cameras are tested in.
__global__ void __launch_bounds__(kCarveThreads)
    carve_kernel(const __grid_constant__ CarveParams p) {
  constexpr int kVox = kCarveWordsPerBlock * 32;
  __shared__ CamAffine aff[FVV_MAX_CAMS];
  __shared__ uint32_t occw[kCarveWordsPerBlock];
  __shared__ uint32_t queue[kVox];  // local index | seen << 12 | amb << 19
  __shared__ int qn, block_on;
  const int64_t b = blockIdx.x;
  int g = 0;
  while (b >= p.blk_start[g + 1]) ++g;  // uniform across the block
  const fvv_grid &G = p.grids[g];
  const int64_t nx = G.dims[0], ny = G.dims[1];
  const int64_t nvox = nx * ny * G.dims[2];
  const bool small = nvox < (int64_t)0xffffffff;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kCarveThreads / 32;
  if (threadIdx.x == 0) {
    qn = 0;
    block_on = 0;
  }
  for (int w = threadIdx.x; w < kCarveWordsPerBlock; w += blockDim.x) occw[w] = 0;
  for (int c = threadIdx.x; c < p.ncam; c += blockDim.x) cam_affine(p.cams[c], G, aff[c]);
  __syncthreads();
  const int64_t word0 = (b - p.blk_start[g]) * kCarveWordsPerBlock;
  const int64_t l0 = word0 * 32;
#pragma unroll 1
  for (int it = 0; it < kCarveWordsPerBlock / kWarps; ++it) {
    const int lw = it * kWarps + warp;
    const int64_t l = l0 + lw * 32 + lane;
    bool on = false, survivor = false;
    uint32_t code = 0;
    if (l < nvox) {
      int64_t i, j, k;
      voxel_ijk(l, nx, ny, small, i, j, k);
      int seen = 0;
      bool off = false, amb = false;
      test_cams(p, aff, 0, p.k1, (float)i, (float)j, (float)k, seen, off, amb);
      if (!off) {
        if (p.k1 < p.ncam) {
          survivor = true;
          code = (uint32_t)(lw * 32 + lane) | ((uint32_t)seen << 12) | ((uint32_t)amb << 19);
        } else {
          on = settle(p, G, g, l, seen, amb);
        }
      }
    }
    const uint32_t sv = __ballot_sync(0xffffffffu, survivor);
    if (sv) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&qn, __popc(sv));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (survivor) queue[base + __popc(sv & ((1u << lane) - 1u))] = code;
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, on);
    if (lane == 0 && bits) atomicOr(&occw[lw], bits);
  }
  __syncthreads();
  const int n = qn;
#pragma unroll 1
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const uint32_t code = queue[q];
    const int li = (int)(code & 0xfffu);
    int seen = (int)((code >> 12) & 0x7fu);
    bool amb = (code >> 19) & 1u, off = false;
    const int64_t l = l0 + li;
    int64_t i, j, k;
    voxel_ijk(l, nx, ny, small, i, j, k);
    test_cams(p, aff, p.k1, p.ncam, (float)i, (float)j, (float)k, seen, off, amb);
    if (!off && settle(p, G, g, l, seen, amb)) atomicOr(&occw[li >> 5], 1u << (li & 31));
  }
  __syncthreads();
  int my_on = 0;
  for (int w = threadIdx.x; w < kCarveWordsPerBlock; w += blockDim.x) {
    if ((word0 + w) * 32 < nvox) {
      p.occ[p.word_off[g] + word0 + w] = occw[w];
      my_on += __popc(occw[w]);
    }
  }
  if (p.count) {
    my_on = __reduce_add_sync(0xffffffffu, my_on);
    if (lane == 0 && my_on) atomicAdd(&block_on, my_on);
    __syncthreads();
    if (threadIdx.x == 0 && block_on)
      atomicAdd((unsigned long long *)&p.count[g], (unsigned long long)block_on);
  }
}

// Voxels the FP32 pass left undecided: float64 chain, set their bits.
__global__ void __launch_bounds__(kCarveThreads)
    carve_exact_kernel(const __grid_constant__ CarveParams p) {
  int64_t n = (int64_t)__ldcg(p.amb);
  if (n > p.amb_cap) n = p.amb_cap;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long e = p.amb[1 + q];
    const int g = (int)(e >> 40);
    const int64_t l = (int64_t)(e & ((1ull << 40) - 1));
    if (carve_exact(p, p.grids[g], l)) {
      atomicOr(p.occ + p.word_off[g] + (l >> 5), 1u << (l & 31));
      if (p.count) atomicAdd((unsigned long long *)&p.count[g], 1ull);
    }
  }
}

}  // namespace fvv

using namespace fvv;

extern "C" size_t fvv_carve_workspace_bytes(void) {
  return sizeof(unsigned long long) * (1 + (size_t)kAmbCap);
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
  const bool deferred = workspace && ws_bytes >= fvv_carve_workspace_bytes();
  p.amb = deferred ? (unsigned long long *)workspace : nullptr;
  p.amb_cap = deferred ? kAmbCap : 0;
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
  if (deferred) cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), st);
  carve_kernel<<<(unsigned)blocks, kCarveThreads, 0, st>>>(p);
  note_launches(1);
  if (deferred) {
    carve_exact_kernel<<<148 * 4, kCarveThreads, 0, st>>>(p);
    note_launches(1);
  }
  return cuda_check("fvv_carve");
}
