// D-1 depth images, D-2 visibility, E view-dependent colour
// (visibility.py:34-140, render.py:35-113, camera.py:204-220).
//
// Rasterisation: one thread per (camera, triangle) sets the triangle up
// exactly as visibility.py:48-78 does (zero-distortion projection, near
// clip, clamped bbox, signed area / swap, top-left flags) and walks its
// bbox when it is small (the norm at C3: ~1-4 px); triangles with a larger
// bbox go to a queue that whole blocks sweep pixel-parallel. The reference
// keeps, per pixel, the first triangle (ascending id) reaching the minimum
// depth (strict `<`): lexicographic min of (depth, id). Depth is positive,
// so its IEEE bits order like the value: pass 1 is a 64-bit atomicMin of
// the depth bits; pass 2 (only when ids are wanted) re-evaluates the
// identical depth and atomicMin's the id where it equals the stored depth.
// Integer atomics only; results do not depend on scheduling.
#include <cstdlib>
#include <cstring>

#include "fvv_common.cuh"

namespace fvv {

constexpr int kSmallBBox = 64;       // pixels walked by one thread
constexpr int kRasterThreads = 128;
constexpr int kBigThreads = 256;

struct RasterCams {
  int ncam;
  int64_t depth_off[FVV_MAX_CAMS];  // element offset of camera c's (H, W) planes
  fvv_camera cams[FVV_MAX_CAMS];
};

struct TriSetup {
  double x0, y0, x1, y1, x2, y2, za, zb, zc, area;
  int lox, loy, hix, hiy;
  bool tl0, tl1, tl2;
};

__device__ __forceinline__ bool top_left(double ax, double ay, double bx, double by) {
  const double dy = by - ay, dx = bx - ax;  // visibility.py:28-31
  return dy < 0.0 || (dy == 0.0 && dx < 0.0);
}

// visibility.py:50: every vertex projected once per camera (zero distortion,
// gemm order; gemv when the mesh has one vertex) -> (u, v, z, pad) records,
// plus the float-rounded (u, v) the FP32 filter reads; NaN there when the
// reference culls every triangle using the vertex (z <= NEAR_CLIP or NaN u/v).
__device__ __forceinline__ void project_vertex(const RasterCams &C, const double *__restrict__ V,
                                               int64_t nv, int64_t w, bool gemv,
                                               double4 *__restrict__ proj,
                                               float2 *__restrict__ q) {
  const int c = (int)(w / nv);
  const int64_t i = w - (int64_t)c * nv;
  double u, v, z;
  project_exact(C.cams[c], V[3 * i], V[3 * i + 1], V[3 * i + 2], false, gemv, u, v, z);
  proj[w] = make_double4(u, v, z, 0.0);
  q[w] = (z > kNearClip && !isnan(u) && !isnan(v)) ? make_float2((float)u, (float)v)
                                                   : make_float2(__int_as_float(0x7fffffff),
                                                                 __int_as_float(0x7fffffff));
}

// (camera, vertex) records for vertices i < nvd of a [ncam][nv] layout
__device__ __forceinline__ void project_vertices(const RasterCams &C, const double *__restrict__ V,
                                                 int64_t nv, int64_t nvd, int64_t tid,
                                                 int64_t stride, double4 *__restrict__ proj,
                                                 float2 *__restrict__ q) {
  const bool gemv = nvd == 1;
  const int64_t total = nv * C.ncam;
  for (int64_t w = tid; w < total; w += stride)
    if (w - (w / nv) * nv < nvd) project_vertex(C, V, nv, w, gemv, proj, q);
}

__global__ void raster_vertex_kernel(const __grid_constant__ RasterCams C,
                                     const double *__restrict__ V, int64_t nv,
                                     const int64_t *nv_dev, double4 *__restrict__ proj,
                                     float2 *__restrict__ q) {
  pdl_wait();
  project_vertices(C, V, nv, device_count(nv_dev, nv), blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                   (int64_t)gridDim.x * blockDim.x, proj, q);
}

__device__ __forceinline__ double dmin3(double a, double b, double c) {
  const double m = a < b ? a : b;
  return m < c ? m : c;
}
__device__ __forceinline__ double dmax3(double a, double b, double c) {
  const double m = a > b ? a : b;
  return m > c ? m : c;
}

// visibility.py:48-78 for triangle t from its projected vertices. False = skipped.
__device__ __forceinline__ bool tri_setup(int width, int height, const double4 *__restrict__ P,
                                          const int32_t *__restrict__ T, int64_t t,
                                          TriSetup &s) {
  const double4 pa = P[T[3 * t]], pb = P[T[3 * t + 1]], pc = P[T[3 * t + 2]];
  const double u[3] = {pa.x, pb.x, pc.x}, v[3] = {pa.y, pb.y, pc.y}, z[3] = {pa.z, pb.z, pc.z};
  if (!(z[0] > kNearClip && z[1] > kNearClip && z[2] > kNearClip)) return false;
  if (isnan(u[0]) || isnan(u[1]) || isnan(u[2]) || isnan(v[0]) || isnan(v[1]) || isnan(v[2]))
    return false;
  // (no NaN past this point: plain compares instead of fmin/fmax)
  const double mnx = dmin3(u[0], u[1], u[2]), mxx = dmax3(u[0], u[1], u[2]);
  const double mny = dmin3(v[0], v[1], v[2]), mxy = dmax3(v[0], v[1], v[2]);
  const double flx = floor(mnx), fly = floor(mny), chx = ceil(mxx), chy = ceil(mxy);
  const double W1 = (double)(width - 1), H1 = (double)(height - 1);
  if (flx > W1 || fly > H1 || chx < 0.0 || chy < 0.0) return false;
  s.lox = flx > 0.0 ? (int)flx : 0;
  s.loy = fly > 0.0 ? (int)fly : 0;
  s.hix = chx < W1 ? (int)chx : width - 1;
  s.hiy = chy < H1 ? (int)chy : height - 1;
  if (s.hix < s.lox || s.hiy < s.loy) return false;
  const double x0 = u[0], y0 = v[0], za = z[0];
  const double area0 = (u[1] - x0) * (v[2] - y0) - (v[1] - y0) * (u[2] - x0);
  if (area0 == 0.0) return false;
  // swap v1 <-> v2 when the area is negative (visibility.py:63-66), branch-free
  const bool sw = area0 < 0.0;
  const double x1 = sw ? u[2] : u[1], y1 = sw ? v[2] : v[1], zb = sw ? z[2] : z[1];
  const double x2 = sw ? u[1] : u[2], y2 = sw ? v[1] : v[2], zc = sw ? z[1] : z[2];
  const double area = sw ? -area0 : area0;
  s.x0 = x0; s.y0 = y0; s.x1 = x1; s.y1 = y1; s.x2 = x2; s.y2 = y2;
  s.za = za; s.zb = zb; s.zc = zc; s.area = area;
  s.tl0 = top_left(x1, y1, x2, y2);
  s.tl1 = top_left(x2, y2, x0, y0);
  s.tl2 = top_left(x0, y0, x1, y1);
  return true;
}

// visibility.py:67-91 at pixel (x, y): inside test and perspective depth.
__device__ __forceinline__ bool tri_depth(const TriSetup &s, int x, int y, double &d) {
  const double gx = (double)x, gy = (double)y;
  const double w0 = (s.x2 - s.x1) * (gy - s.y1) - (s.y2 - s.y1) * (gx - s.x1);
  const double w1 = (s.x0 - s.x2) * (gy - s.y2) - (s.y0 - s.y2) * (gx - s.x2);
  const double w2 = (s.x1 - s.x0) * (gy - s.y0) - (s.y1 - s.y0) * (gx - s.x0);
  const bool in = (w0 > 0.0 || (w0 == 0.0 && s.tl0)) && (w1 > 0.0 || (w1 == 0.0 && s.tl1)) &&
                  (w2 > 0.0 || (w2 == 0.0 && s.tl2));
  if (!in) return false;
  const double b0 = w0 / s.area, b1 = w1 / s.area, b2 = w2 / s.area;
  const double zinv = b0 / s.za + b1 / s.zb + b2 / s.zc;
  d = 1.0 / zinv;
  return d < INFINITY;  // only finite depths can beat the +inf background
}

// p: the pixel's element index in the depth buffer (its dirty tile is p / 32)
__device__ __forceinline__ void pixel_update(int pass, double d, int64_t t,
                                             unsigned long long *depth, unsigned *ids,
                                             uint8_t *dirty, int64_t p) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
  if (pass == 0) {
    atomicMin(depth, bits);  // result unused -> RED.MIN (no round trip)
    if (dirty) dirty[p >> 5] = 1;
  } else if (bits == __ldcg(depth)) {
    atomicMin(ids, (unsigned)t);
  }
}

// (item, pixel) pair entries carry the camera in the top bits of the
// triangle index (no division to split a camera-major item index)
constexpr int kPairCamShift = 26;
constexpr uint32_t kPairTriMask = (1u << kPairCamShift) - 1u;

struct RasterArgs {
  const double4 *P;  // [ncam][nv] projected vertices (u, v, z, 0)
  const float2 *Q;   // [ncam][nv] (u, v) rounded to float; NaN: the vertex culls its triangles
  const int32_t *T;
  int64_t nt;
  const int64_t *nt_dev;
  int64_t nv;
  double *depth;
  int32_t *ids;
  int64_t *queue;     // big (camera, triangle) entries
  int64_t *qcount;
  int64_t qcap;
  // work lists of the FP32 filter: one pair list and one item list per
  // filter warp (appends need no atomics); wl_items bounds the items one
  // filter warp sees, so the item lists cannot overflow; a full pair list
  // sets *overflow and the sweep kernel then redoes every item
  int64_t nwl, wl_items, wl_pairs;
  uint8_t *dirty;     // optional: per 32-pixel tile of the planes, set when a depth is written
  // ids wanted: pass 0 also records every depth write (pixel, triangle, depth
  // bits); one pass over that list then finds each pixel's lowest id at the
  // final depth (pass 1 re-runs the raster only if the list overflowed)
  uint4 *hits;
  unsigned long long *hit_count;
  int64_t hit_cap;
  uint32_t *slow;     // items the FP32 filter leaves to the warp-sweep kernel
  uint2 *pairs;       // (item, y << 16 | x): candidate pixels from the FP32 filter
  int *wcount;        // [nwl][2]: pairs, items
  int *overflow;
  int pass;
};

// Warp-aggregated append of this lane's depth write (hit) to the hit list;
// called by every lane of the warp.
__device__ __forceinline__ void record_hit(const RasterArgs &A, bool hit, int64_t p, int64_t t,
                                           double d) {
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if (!m) return;
  const int lane = threadIdx.x & 31, lead = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == lead) base = atomicAdd(A.hit_count, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, lead);
  if (hit) {
    const unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
    const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
    if ((int64_t)slot < A.hit_cap)
      A.hits[slot] = make_uint4((uint32_t)p, (uint32_t)t, (uint32_t)bits, (uint32_t)(bits >> 32));
  }
}

// pass 1 kernels: nothing to do when the hit list holds every depth write
__device__ __forceinline__ bool pass1_covered(const RasterArgs &A) {
  return A.pass == 1 && A.hits != nullptr && (int64_t)__ldcg(A.hit_count) <= A.hit_cap;
}

// Triangle setup as kept in shared memory for the warp's pixel sweep.
struct TriSmem {
  double x0, y0, x1, y1, x2, y2, za, zb, zc, area;
  unsigned long long mask;       // candidate bbox pixels (bit k = pixel k), 0 = all
  int t, cam, lox, loy, bw, tl;  // tl: top-left flags bits 0..2
};

// Candidate filter for a bbox of <= 64 pixels: a pixel centre is kept unless
// an FP32 evaluation of some edge function, in bbox-local coordinates, is
// below minus an error margin that dominates the FP32 error by orders of
// magnitude. A rejected pixel therefore has a strictly negative real-valued
// edge function, and the exact float64 test (tri_depth) would reject it too:
// the filter changes how many pixels are tested, never the result. At C3 the
// bboxes sweep ~8 pixel centres per triangle for ~0.25 inside.
__device__ __forceinline__ unsigned long long candidate_mask(const TriSetup &s) {
  const int bw = s.hix - s.lox + 1, bh = s.hiy - s.loy + 1;
  const double ox = (double)s.lox, oy = (double)s.loy;
  const float X0 = (float)(s.x0 - ox), Y0 = (float)(s.y0 - oy);
  const float X1 = (float)(s.x1 - ox), Y1 = (float)(s.y1 - oy);
  const float X2 = (float)(s.x2 - ox), Y2 = (float)(s.y2 - oy);
  // w = a (gy - Y) - b (gx - X) = a gy - b gx + c   (edge order of tri_depth)
  const float a0 = X2 - X1, b0 = Y2 - Y1, c0 = b0 * X1 - a0 * Y1;
  const float a1 = X0 - X2, b1 = Y0 - Y2, c1 = b1 * X2 - a1 * Y2;
  const float a2 = X1 - X0, b2 = Y1 - Y0, c2 = b2 * X0 - a2 * Y0;
  const float ext = (float)(bw + bh + 2);
  const float k = 1.0f / 16384.0f;
  const float m0 = ((fabsf(a0) + fabsf(b0)) * ext + fabsf(c0) + 1.0f) * k;
  const float m1 = ((fabsf(a1) + fabsf(b1)) * ext + fabsf(c1) + 1.0f) * k;
  const float m2 = ((fabsf(a2) + fabsf(b2)) * ext + fabsf(c2) + 1.0f) * k;
  // per row gy, edge i keeps gx with b_i gx <= r_i(gy) + m_i: an interval
  // of gx per edge, intersected, widened by 1e-3 px (the reciprocal's error
  // is ~1e-7 relative over |gx| <= 64), turned into a run of mask bits
  const float ib0 = __fdividef(1.0f, b0), ib1 = __fdividef(1.0f, b1), ib2 = __fdividef(1.0f, b2);
  unsigned long long mask = 0;
  const float top = (float)(bw - 1);
  for (int yy = 0; yy < bh; ++yy) {
    const float gy = (float)yy;
    float lo = 0.0f, hi = top;
    bool empty = false;
    const float sv0 = fmaf(a0, gy, c0) + m0, sv1 = fmaf(a1, gy, c1) + m1,
                sv2 = fmaf(a2, gy, c2) + m2;
    // branchless: b > 0 bounds gx from above, b < 0 from below, b == 0 keeps
    // the whole row iff sv >= 0
    const float t0 = sv0 * ib0, t1 = sv1 * ib1, t2 = sv2 * ib2;
    hi = fminf(hi, b0 > 0.0f ? t0 + 1e-3f : INFINITY);
    lo = fmaxf(lo, b0 < 0.0f ? t0 - 1e-3f : -INFINITY);
    hi = fminf(hi, b1 > 0.0f ? t1 + 1e-3f : INFINITY);
    lo = fmaxf(lo, b1 < 0.0f ? t1 - 1e-3f : -INFINITY);
    hi = fminf(hi, b2 > 0.0f ? t2 + 1e-3f : INFINITY);
    lo = fmaxf(lo, b2 < 0.0f ? t2 - 1e-3f : -INFINITY);
    empty = ((b0 == 0.0f) & (sv0 < 0.0f)) | ((b1 == 0.0f) & (sv1 < 0.0f)) |
            ((b2 == 0.0f) & (sv2 < 0.0f));
    const int x0 = (int)ceilf(lo), x1 = (int)floorf(hi);  // NaN bounds -> empty below
    if (!empty && x0 <= x1 && lo <= hi) {
      const unsigned long long run = (x1 - x0 >= 63) ? ~0ull : ((2ull << (x1 - x0)) - 1ull);
      mask |= run << (yy * bw + x0);
    }
  }
  return mask;
}

__device__ __forceinline__ void setup_to_smem(const TriSetup &s, int64_t t, int cam, TriSmem &m,
                                              unsigned long long mask) {
  m.mask = mask;
  m.x0 = s.x0; m.y0 = s.y0; m.x1 = s.x1; m.y1 = s.y1; m.x2 = s.x2; m.y2 = s.y2;
  m.za = s.za; m.zb = s.zb; m.zc = s.zc; m.area = s.area;
  m.t = (int)t;
  m.cam = cam;
  m.lox = s.lox;
  m.loy = s.loy;
  m.bw = s.hix - s.lox + 1;
  m.tl = (int)s.tl0 | ((int)s.tl1 << 1) | ((int)s.tl2 << 2);
}

__device__ __forceinline__ void smem_to_setup(const TriSmem &m, TriSetup &s) {
  s.x0 = m.x0; s.y0 = m.y0; s.x1 = m.x1; s.y1 = m.y1; s.x2 = m.x2; s.y2 = m.y2;
  s.za = m.za; s.zb = m.zb; s.zc = m.zc; s.area = m.area;
  s.tl0 = m.tl & 1; s.tl1 = (m.tl >> 1) & 1; s.tl2 = (m.tl >> 2) & 1;
}

// ---- FP32 filter: which (camera, triangle) items can cover which pixels ----
//
// At C3 the projected triangles are ~1 px: 10.4 M (camera, triangle) items
// per frame cover 2.5 M pixels, and three quarters of the items cover none.
// raster_filter_kernel decides each item from the float-rounded vertices
// (Q, rounded from the exact float64 projections) with certified margins and
// emits (item, pixel) pairs for the pixels that may be inside; the float64
// test of the reference then runs only on those (raster_pair_kernel).
// Items it cannot decide go to the warp-sweep kernel (raster_small_kernel),
// which rasterises them exactly as before.
//
// Certification (vertices u_j exact float64, U_j = float(u_j)):
//  * |U_j - u_j| <= 2^-24 max|U|, and the local coordinates X_j = U_j - ox
//    (ox = floor of the float min, |X_j| <= 65) add <= 2^-24 * 65; dd =
//    2^-22 (max|U| + 128) bounds the sum twice over.
//  * the float area's error is bounded by aerr; |area32| > aerr fixes the
//    orientation (the reference's v1 <-> v2 swap, visibility.py:63-66, which
//    negates the three edge functions). Uncertain orientation -> sweep kernel.
//  * candidate pixels: the tight integer range of the float extent widened by
//    mt = 2 dd + 2^-12 when |area32| > aerr + A (A = 2^-6), else the whole
//    widened bounding box. A pixel centre outside the tight range lies >=
//    2^-12 outside the exact extent; with exact |area| >= A and an extent
//    <= 64 px its barycentric coordinates give some edge function
//    w <= -2^-12 A / 128 = -2^-25 in exact arithmetic, while the float64
//    evaluation of w in the reference (|terms| <= 65 * 64) errs by < 2^-36:
//    the reference rejects the pixel.
//  * a candidate is dropped when some float edge function (oriented) is below
//    -m, m twice the bound of the float rounding plus the effect of the vertex
//    perturbation dd: its exact w is < -m/2 < 0 and the float64 rounding
//    (< 2^-36) cannot lift it to >= 0.
//  * ranges larger than 2 x 2 pixels (4 % of the C3 items), extents above
//    60 px and coordinates beyond 2^20 px go to the sweep kernel.
// Every emitted pixel is re-tested in float64 exactly as the reference does,
// so the filter decides how much work runs, never a result.
__device__ __forceinline__ float2 ldq(const float2 *__restrict__ q) { return __ldg(q); }

__global__ void __launch_bounds__(256)
    raster_filter_kernel(const __grid_constant__ RasterCams C, RasterArgs A) {
  pdl_wait();
  const int64_t nt = device_count(A.nt_dev, A.nt);
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  uint2 *pl = A.pairs + wid * A.wl_pairs;
  uint32_t *sl = A.slow + wid * A.wl_items;
  int np = 0, ns = 0;  // this warp's list lengths
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // a thread takes one triangle through every camera: its vertex indices are
  // read once and the next camera's vertices are fetched while this one runs
  for (int64_t t0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; t0 < nt;
       t0 += stride) {
    const int64_t t = t0 + lane;
    const bool valid = t < nt;
    const float2 *q0 = A.Q, *q1 = A.Q, *q2 = A.Q;  // this triangle's vertices, camera c
    float2 n0 = make_float2(0.f, 0.f), n1 = n0, n2 = n0;
    if (valid) {
      q0 += __ldg(A.T + 3 * t);
      q1 += __ldg(A.T + 3 * t + 1);
      q2 += __ldg(A.T + 3 * t + 2);
      n0 = ldq(q0);
      n1 = ldq(q1);
      n2 = ldq(q2);
    }
    for (int c = 0; c < C.ncam; ++c) {
    const float2 p0 = n0, p1 = n1, p2 = n2;
    q0 += A.nv;
    q1 += A.nv;
    q2 += A.nv;
    if (valid && c + 1 < C.ncam) {
      n0 = ldq(q0);
      n1 = ldq(q1);
      n2 = ldq(q2);
    }
    const int W = C.cams[c].width, H = C.cams[c].height;
    const uint32_t w = (uint32_t)(c * nt + t);  // camera-major item index
    const uint32_t pw = ((uint32_t)c << kPairCamShift) | (uint32_t)t;  // pair entries: (camera, t)
    int state = 0;          // 0 nothing, 1 pixels in `bits`, 2 slow path
    unsigned bits = 0;      // candidate pixels of the tight range, row-major
    int gx0 = 0, gy0 = 0, rw = 1;
    if (valid) {
      const bool culled = isnan(p0.x) | isnan(p1.x) | isnan(p2.x);  // near clip / NaN vertex
      const float mnx = fminf(fminf(p0.x, p1.x), p2.x), mxx = fmaxf(fmaxf(p0.x, p1.x), p2.x);
      const float mny = fminf(fminf(p0.y, p1.y), p2.y), mxy = fmaxf(fmaxf(p0.y, p1.y), p2.y);
      const float mx = fmaxf(fmaxf(fabsf(mnx), fabsf(mxx)), fmaxf(fabsf(mny), fabsf(mxy)));
      const float ext = fmaxf(mxx - mnx, mxy - mny);
      if (culled) {
        state = 0;
      } else if (!(mx <= 1048576.0f) || !(ext <= 60.0f)) {
        state = 2;  // inf / huge coordinates, or a large triangle
      } else {
        const float dd = 0x1p-22f * (mx + 128.0f);
        const float ox = floorf(mnx), oy = floorf(mny);
        const float X0 = p0.x - ox, Y0 = p0.y - oy, X1 = p1.x - ox, Y1 = p1.y - oy,
                    X2 = p2.x - ox, Y2 = p2.y - oy;
        const float area = (X1 - X0) * (Y2 - Y0) - (Y1 - Y0) * (X2 - X0);
        // |X1-X0| + |Y2-Y0| + |Y1-Y0| + |X2-X0| <= 4 ext, |q1| + |q2| <= 2 ext^2
        const float aerr = 2.0f * (8.0f * dd * ext + 4.0f * dd * dd + 0x1p-20f * ext * ext);
        const float mt = 2.0f * dd + 0x1p-12f;
        // pixel range: the tight integer range of the extent when |area| >= A
        // is certain, else the whole (widened) bounding box
        const bool tight = fabsf(area) > aerr + 0x1p-6f;
        const float lx = mnx - mt, hx = mxx + mt, ly = mny - mt, hy = mxy + mt;
        const int tx0 = max((int)(tight ? ceilf(lx) : floorf(lx)), 0);
        const int tx1 = min((int)(tight ? floorf(hx) : ceilf(hx)), W - 1);
        const int ty0 = max((int)(tight ? ceilf(ly) : floorf(ly)), 0);
        const int ty1 = min((int)(tight ? floorf(hy) : ceilf(hy)), H - 1);
        rw = tx1 - tx0 + 1;
        const int rh = ty1 - ty0 + 1;
        if (rw > 0 && rh > 0) {
          if (rw > 2 || rh > 2 || !(fabsf(area) > aerr)) {
            state = 2;  // (4 % of the C3 items) the warp-sweep kernel takes it
          } else {
            // edge functions in the reference's vertex order (tri_depth); the
            // v1 <-> v2 swap of visibility.py:63-66 negates all three, so with
            // the sign s of the (certain) orientation a pixel is kept iff
            // min(s w) >= -m. One margin for the three edges (|a| + |b| <=
            // 2 ext, |g - X| <= ext + 2, a few more roundings for the 2 x 2
            // block stepped from its corner). Branch-free over the block; bit
            // yy * rw + xx for the pixels inside the range.
            const float s = area > 0.0f ? 1.0f : -1.0f;
            const float a0 = s * (X2 - X1), b0 = s * (Y2 - Y1), a1 = s * (X0 - X2),
                        b1 = s * (Y0 - Y2), a2 = s * (X1 - X0), b2 = s * (Y1 - Y0);
            const float m = -2.0f * (dd * (6.0f * ext + 9.0f) +
                                     0x1p-20f * (2.0f * ext * (ext + 2.0f) + 1.0f));
            gx0 = tx0;
            gy0 = ty0;
            const float gx = (float)tx0 - ox, gy = (float)ty0 - oy;
            const float r0 = a0 * (gy - Y1) - b0 * (gx - X1);
            const float r1 = a1 * (gy - Y2) - b1 * (gx - X2);
            const float r2 = a2 * (gy - Y0) - b2 * (gx - X0);
#pragma unroll
            for (int yy = 0; yy < 2; ++yy) {
#pragma unroll
              for (int xx = 0; xx < 2; ++xx) {
                const float w0 = (yy ? r0 + a0 : r0) - (xx ? b0 : 0.0f);
                const float w1 = (yy ? r1 + a1 : r1) - (xx ? b1 : 0.0f);
                const float w2 = (yy ? r2 + a2 : r2) - (xx ? b2 : 0.0f);
                if (fminf(fminf(w0, w1), w2) >= m && xx < rw && yy < rh)
                  bits |= 1u << (yy * rw + xx);
              }
            }
            state = bits ? 1 : 0;
          }
        }
      }
    }
    // appends to this warp's own lists (no atomics): pixel pairs, then the
    // items left to the sweep kernel
    const int npx = __popc(bits);
    int incl = npx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int sum = __shfl_sync(0xffffffffu, incl, 31);
    if (sum) {
      if (np + sum > A.wl_pairs) {
        if (lane == 0) atomicOr(A.overflow, 1);  // the sweep kernel redoes every item
      } else {
        if (bits) {
        uint2 *slot = pl + np + (incl - npx);
        const int sh = rw == 2;  // k / rw for rw in {1, 2}
        unsigned b = bits;
        while (b) {
          const int k = __ffs(b) - 1;
          b &= b - 1;
          const int qy = k >> sh;
          *slot++ = make_uint2(pw, ((uint32_t)(gy0 + qy) << 16) | (uint32_t)(gx0 + k - qy * rw));
        }
        }
        np += sum;  // = entries written
      }
    }
    const unsigned slow = __ballot_sync(0xffffffffu, state == 2);
    if (state == 2) sl[ns + __popc(slow & ((1u << lane) - 1u))] = w;
    ns += __popc(slow);
    }
  }
  if (lane == 0) {
    A.wcount[2 * wid] = np;
    A.wcount[2 * wid + 1] = ns;
  }
}

// The float64 test of one emitted (item, pixel) pair, exactly as the
// reference evaluates that pixel for that triangle (visibility.py:48-91):
// the same setup, the pixel must lie in the clamped bounding box, then the
// inside test with top-left ties and the perspective-correct depth. One
// warp per filter-warp list.
template <bool kRec>
__global__ void __launch_bounds__(256)
    raster_pair_kernel(const __grid_constant__ RasterCams C, RasterArgs A) {
  pdl_wait();
  if (pass1_covered(A)) return;
  const int64_t nt = device_count(A.nt_dev, A.nt);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t wl = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); wl < A.nwl;
       wl += nwarps) {
    const int n = __ldcg(A.wcount + 2 * wl);
    const uint2 *pl = A.pairs + wl * A.wl_pairs;
    if (!kRec) {
      for (int i = lane; i < n; i += 32) {
        const uint2 e = pl[i];
        const int c = (int)(e.x >> kPairCamShift);
        const int64_t t = (int64_t)(e.x & kPairTriMask);
        const int x = (int)(e.y & 0xffffu), y = (int)(e.y >> 16);
        const int width = C.cams[c].width;
        TriSetup s;
        if (!tri_setup(width, C.cams[c].height, A.P + (int64_t)c * A.nv, A.T, t, s)) continue;
        if (x < s.lox || x > s.hix || y < s.loy || y > s.hiy) continue;
        double d;
        if (!tri_depth(s, x, y, d)) continue;
        const int64_t p = C.depth_off[c] + (int64_t)y * width + x;
        pixel_update(A.pass, d, t, (unsigned long long *)A.depth + p,
                     A.ids ? (unsigned *)A.ids + p : nullptr, A.dirty, p);
      }
      continue;
    }
    // kRec (pass 0 of an id raster): warp-uniform trip count, since the
    // depth writes are appended to the hit list warp-aggregated
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      bool hit = false;
      double d = 0.0;
      int64_t p = 0, t = 0;
      if (i < n) {
        const uint2 e = pl[i];
        const int c = (int)(e.x >> kPairCamShift);
        t = (int64_t)(e.x & kPairTriMask);
        const int x = (int)(e.y & 0xffffu), y = (int)(e.y >> 16);
        const int width = C.cams[c].width;
        TriSetup s;
        if (tri_setup(width, C.cams[c].height, A.P + (int64_t)c * A.nv, A.T, t, s) &&
            !(x < s.lox || x > s.hix || y < s.loy || y > s.hiy) && tri_depth(s, x, y, d)) {
          p = C.depth_off[c] + (int64_t)y * width + x;
          pixel_update(A.pass, d, t, (unsigned long long *)A.depth + p,
                       A.ids ? (unsigned *)A.ids + p : nullptr, A.dirty, p);
          hit = true;
        }
      }
      record_hit(A, hit, p, t, d);
    }
  }
}

// Warp-cooperative small-triangle raster for the items the FP32 filter could
// not decide (raster_filter_kernel: near-degenerate or large triangles,
// coordinates beyond 2^20 px): the 32 lanes set up 32 (camera, triangle)
// items, publish them in shared memory, then sweep the union of their
// bounding-box pixels 32 at a time (each lane finds its pixel's owner by a
// shuffle binary search over the warp's inclusive pixel-count scan), so uneven
// bounding boxes and culled triangles do not leave lanes idle.
__global__ void __launch_bounds__(kRasterThreads, 8)
    raster_small_kernel(const __grid_constant__ RasterCams C, RasterArgs A) {
  pdl_wait();
  __shared__ TriSmem sm[kRasterThreads];
  if (pass1_covered(A)) return;
  const bool rec = A.hits != nullptr && A.pass == 0;
  const int lane = threadIdx.x & 31;
  TriSmem *wsm = sm + (threadIdx.x & ~31);
  const int64_t nt = device_count(A.nt_dev, A.nt);
  const bool overflow = A.pass == 1 && __ldcg(A.qcount) > A.qcap;
  // work: the filter warps' item lists, or (pair list overflow) every item
  const bool all = __ldcg(A.overflow) != 0;
  const int64_t total_all = nt * C.ncam;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t cur = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);  // list or chunk
  int off = 0;
  for (;;) {
    bool valid;
    uint32_t w;
    if (all) {
      if (cur * 32 >= total_all) break;
      valid = cur * 32 + lane < total_all;
      w = (uint32_t)(cur * 32 + lane);
      cur += nw;
    } else {
      int n = 0;
      while (cur < A.nwl && off >= (n = __ldcg(A.wcount + 2 * cur + 1))) {
        cur += nw;
        off = 0;
      }
      if (cur >= A.nwl) break;
      valid = off + lane < n;
      w = valid ? __ldcg(A.slow + cur * A.wl_items + off + lane) : 0u;
      off += 32;
    }
    int npx = 0;
    if (valid) {
      const int c = (int)(w / (uint32_t)nt);  // camera-major item index
      const int64_t t = (int64_t)w - (int64_t)c * nt;
      TriSetup s;
      if (tri_setup(C.cams[c].width, C.cams[c].height, A.P + (int64_t)c * A.nv, A.T, t, s)) {
        const int64_t n = (int64_t)(s.hix - s.lox + 1) * (s.hiy - s.loy + 1);
        bool mine = true;
        if (n > kSmallBBox) {
          if (A.pass == 0) {
            const unsigned long long slot = atomicAdd((unsigned long long *)A.qcount, 1ull);
            mine = (int64_t)slot >= A.qcap;  // queue full: sweep it here
            if (!mine) A.queue[slot] = w;
          } else {
            mine = overflow;  // pass 1: the big kernel replays the queue
          }
        }
        if (mine) {
          unsigned long long mask = 0;
          if (n <= 64) {
            mask = candidate_mask(s);
            npx = __popcll(mask);
          } else {
            npx = (int)n;  // (queue overflow) sweep the whole bbox
          }
          if (npx) setup_to_smem(s, t, c, wsm[lane], mask);
        }
      }
    }
    // inclusive scan of the pixel counts across the warp
    int incl = npx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int sum = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    for (int base = 0; base < sum; base += 32) {
      const int idx = base + lane;
      // owner = number of lanes whose inclusive count is <= idx
      int own = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, own + step - 1);
        if (v <= idx) own += step;
      }
      const int own_incl = __shfl_sync(0xffffffffu, incl, own);
      const int own_cnt = __shfl_sync(0xffffffffu, npx, own);
      bool hit = false;
      double hd = 0.0;
      int64_t hp = 0, ht = 0;
      if (idx < sum) {
        const TriSmem &m = wsm[own];
        int k = idx - (own_incl - own_cnt);
        unsigned long long mk = m.mask;
        if (mk) {  // k-th candidate -> its bbox pixel index
          for (int j = 0; j < k; ++j) mk &= mk - 1;
          k = __ffsll((long long)mk) - 1;
        }
        // k / bw without an integer divide: exact for k < 2^12 (the fraction
        // of (k + 0.5) / bw is >= 0.5 / bw, far above the float error)
        int qy = (k < 4096) ? __float2int_rz(((float)k + 0.5f) * __frcp_rn((float)m.bw))
                            : k / m.bw;
        const int y = m.loy + qy, x = m.lox + (k - qy * m.bw);
        TriSetup s;
        smem_to_setup(m, s);
        if (tri_depth(s, x, y, hd)) {
          const int W = C.cams[m.cam].width;
          unsigned long long *dp = (unsigned long long *)(A.depth + C.depth_off[m.cam]);
          unsigned *ip = (unsigned *)(A.ids ? A.ids + C.depth_off[m.cam] : nullptr);
          const int64_t pxl = (int64_t)y * W + x;
          pixel_update(A.pass, hd, m.t, dp + pxl, ip ? ip + pxl : nullptr, A.dirty,
                       C.depth_off[m.cam] + pxl);
          hit = true;
          hp = C.depth_off[m.cam] + pxl;
          ht = m.t;
        }
      }
      if (rec) record_hit(A, hit, hp, ht, hd);
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kBigThreads)
    raster_big_kernel(const __grid_constant__ RasterCams C, RasterArgs A) {
  pdl_wait();
  if (pass1_covered(A)) return;
  const bool rec = A.hits != nullptr && A.pass == 0;
  const int64_t nt = device_count(A.nt_dev, A.nt);
  int64_t nq = __ldcg(A.qcount);
  if (nq > A.qcap) nq = A.qcap;
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    const int64_t w = A.queue[q];
    const int c = (int)(w / nt);
    const int64_t t = w - (int64_t)c * nt;
    const int width = C.cams[c].width, height = C.cams[c].height;
    TriSetup s;
    if (!tri_setup(width, height, A.P + (int64_t)c * A.nv, A.T, t, s)) continue;  // uniform
    const int bw = s.hix - s.lox + 1;
    const int64_t npx = (int64_t)bw * (s.hiy - s.loy + 1);
    unsigned long long *dp = (unsigned long long *)(A.depth + C.depth_off[c]);
    unsigned *ip = (unsigned *)(A.ids ? A.ids + C.depth_off[c] : nullptr);
    for (int64_t k0 = 0; k0 < npx; k0 += blockDim.x) {  // (block-uniform trip count)
      const int64_t k = k0 + threadIdx.x;
      bool hit = false;
      double d = 0.0;
      int64_t hp = 0;
      if (k < npx) {
        const int y = s.loy + (int)(k / bw), x = s.lox + (int)(k % bw);
        if (tri_depth(s, x, y, d)) {
          const int64_t p = (int64_t)y * width + x;
          pixel_update(A.pass, d, t, dp + p, ip ? ip + p : nullptr, A.dirty, C.depth_off[c] + p);
          hit = true;
          hp = C.depth_off[c] + p;
        }
      }
      if (rec) record_hit(A, hit, hp, t, d);
    }
  }
}

// The id pass over the hit list: the lowest triangle id among the writes
// that reached the pixel's final depth (visibility.py:80-91 keeps the first
// triangle, in id order, with the minimum depth).
__global__ void raster_hits_kernel(RasterArgs A) {
  pdl_wait();
  const unsigned long long n = __ldcg(A.hit_count);
  if ((int64_t)n > A.hit_cap) return;  // overflow: the pass-1 raster does it
  const unsigned long long *depth = (const unsigned long long *)A.depth;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint4 h = A.hits[i];
    const unsigned long long bits = (unsigned long long)h.z | ((unsigned long long)h.w << 32);
    if (bits == __ldcg(depth + h.x)) atomicMin((unsigned *)A.ids + h.x, h.y);
  }
}

__device__ __forceinline__ void fill_u64(unsigned long long *p, int64_t n, unsigned long long v,
                                         int64_t tid, int64_t stride) {
  const int64_t head = ((uintptr_t)p & 15) ? 1 : 0;
  if (tid == 0 && head && n > 0) p[0] = v;
  const int64_t n2 = (n - head) / 2;
  ulonglong2 *q = (ulonglong2 *)(p + head);
  const ulonglong2 vv = make_ulonglong2(v, v);
  for (int64_t i = tid; i < n2; i += stride) q[i] = vv;
  if (tid == 0 && head + 2 * n2 < n) p[head + 2 * n2] = v;
}

// Background reset of tracked planes: every 32-pixel tile whose flag the
// previous raster into these planes set goes back to +inf depth (and -1 ids),
// and its flag is cleared. The other tiles still hold the background, so
// only the pixels written last time are rewritten.
__device__ __forceinline__ void reset_dirty(unsigned long long *depth, int32_t *ids,
                                            uint8_t *dirty, int64_t npx, int64_t tid,
                                            int64_t stride) {
  const int64_t ntile = (npx + 31) >> 5;
  for (int64_t f = tid; f < ntile; f += stride) {
    if (!dirty[f]) continue;
    const int64_t p0 = f << 5, n = npx - p0 < 32 ? npx - p0 : 32;
    if (n == 32 && ((uintptr_t)(depth + p0) & 15) == 0) {
      ulonglong2 *q = (ulonglong2 *)(depth + p0);
      const ulonglong2 inf2 = make_ulonglong2(0x7ff0000000000000ull, 0x7ff0000000000000ull);
#pragma unroll
      for (int i = 0; i < 16; ++i) q[i] = inf2;
    } else {
      for (int64_t i = 0; i < n; ++i) depth[p0 + i] = 0x7ff0000000000000ull;
    }
    if (ids) {
      if (n == 32 && ((uintptr_t)(ids + p0) & 15) == 0) {
        int4 *q = (int4 *)(ids + p0);
#pragma unroll
        for (int i = 0; i < 8; ++i) q[i] = make_int4(-1, -1, -1, -1);
      } else {
        for (int64_t i = 0; i < n; ++i) ids[p0 + i] = -1;
      }
    }
    dirty[f] = 0;
  }
}

// D-1 preparation in one launch: the first nb_fill blocks bring the depth
// planes back to the +inf background (a full fill, or with a dirty map only
// the tiles the last raster wrote; HBM-bound), the others project the
// vertices (FP64-bound), so the two overlap instead of running back to back.
__global__ void raster_prep_kernel(const __grid_constant__ RasterCams C,
                                   const double *__restrict__ V, int64_t nv,
                                   const int64_t *nv_dev, double4 *__restrict__ proj,
                                   float2 *__restrict__ q, unsigned long long *depth, int32_t *ids,
                                   uint8_t *dirty, int64_t npx, int nb_fill) {
  pdl_wait();
  if ((int)blockIdx.x < nb_fill) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)nb_fill * blockDim.x;
    if (dirty)
      reset_dirty(depth, ids, dirty, npx, tid, stride);
    else
      fill_u64(depth, npx, 0x7ff0000000000000ull, tid, stride);
    return;
  }
  if (nv > 0)
    project_vertices(C, V, nv, device_count(nv_dev, nv),
                     (blockIdx.x - nb_fill) * (int64_t)blockDim.x + threadIdx.x,
                     (int64_t)(gridDim.x - nb_fill) * blockDim.x, proj, q);
}

__global__ void fill_u64_kernel(unsigned long long *p, int64_t n, unsigned long long v) {
  pdl_wait();
  // 16-byte stores for the aligned bulk, scalar head/tail
  fill_u64(p, n, v, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
           (int64_t)gridDim.x * blockDim.x);
}

// ---- D-2: visibility.py:106-129 ------------------------------------------------
struct ClassifyArgs {
  const double *V;
  const int32_t *T;
  int64_t nt;
  const int64_t *nt_dev;
  const double *depth;
  double t_v;
  uint32_t *vis;       // [ncam][stride] bits
  int64_t vis_stride;  // words per camera
  // optional (render.py:35-43 triangle_sources, fused): the first ranked
  // camera seeing each triangle, by rig position rank_pos[r] / id rank_id[r]
  int32_t *src;
  int nrank;
  int32_t rank_pos[FVV_MAX_CAMS], rank_id[FVV_MAX_CAMS];
};

__global__ void classify_kernel(const __grid_constant__ RasterCams C,
                                const __grid_constant__ ClassifyArgs A) {
  pdl_wait();
  // one thread per triangle, 32 consecutive triangles (one visibility word)
  // per warp: the centroid (three divisions) is computed once and projected
  // into every camera, instead of once per (camera, triangle); the pixel
  // rounding is certified in FP32 (project_rint32)
  __shared__ CamF32 cf[FVV_MAX_CAMS];
  for (int c = threadIdx.x; c < C.ncam; c += blockDim.x) cf[c] = cam_f32(C.cams[c]);
  __syncthreads();
  const int64_t nt = device_count(A.nt_dev, A.nt);
  const bool gemv = nt == 1;
  const int lane = threadIdx.x & 31;
  const int64_t words = (nt + 31) / 32;
  for (int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; w0 < words * 32;
       w0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t wi = w0 >> 5;
    const int64_t t = w0 + lane;
    double mx = 0.0, my = 0.0, mz = 0.0;
    if (t < nt) {
      const double *a = A.V + 3 * (int64_t)A.T[3 * t], *b = A.V + 3 * (int64_t)A.T[3 * t + 1],
                   *cc = A.V + 3 * (int64_t)A.T[3 * t + 2];
      mx = ((a[0] + b[0]) + cc[0]) / 3.0;  // mesh.py:84-85 mean
      my = ((a[1] + b[1]) + cc[1]) / 3.0;
      mz = ((a[2] + b[2]) + cc[2]) / 3.0;
    }
    unsigned long long seen = 0;  // rig positions that see triangle t
    for (int c = 0; c < C.ncam; ++c) {
      bool vis = false;
      if (t < nt) {
        const CamF32 &f = cf[c];
        int ix, iy;
        double z;
        if (project_rint32(C.cams[c], f, mx, my, mz, gemv, ix, iy, z)) {
          const int64_t p = (int64_t)iy * f.width + ix;
          vis = (z - __ldg(A.depth + C.depth_off[c] + p)) <= A.t_v;
        }
      }
      seen |= (unsigned long long)vis << c;
      const uint32_t bits = __ballot_sync(0xffffffffu, vis);
      if (lane == 0) A.vis[(int64_t)c * A.vis_stride + wi] = bits;
    }
    if (A.src != nullptr && t < nt) {
      int32_t s = -1;
      for (int r = 0; r < A.nrank; ++r)
        if ((seen >> A.rank_pos[r]) & 1ull) {
          s = A.rank_id[r];
          break;
        }
      A.src[t] = s;
    }
  }
}

// ---- E: render.py:35-43 triangle_sources ------------------------------------
struct SourceArgs {
  int nrank;
  int32_t rank_pos[FVV_MAX_CAMS];  // rig position of the r-th ranked camera
  int32_t rank_id[FVV_MAX_CAMS];
  const uint32_t *vis;
  int64_t vis_stride;
  int64_t nt;
  const int64_t *nt_dev;
  int32_t *src;
};

__global__ void sources_kernel(const __grid_constant__ SourceArgs A) {
  pdl_wait();
  const int64_t nt = device_count(A.nt_dev, A.nt);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = -1;
    for (int r = 0; r < A.nrank; ++r) {
      const uint32_t w = A.vis[(int64_t)A.rank_pos[r] * A.vis_stride + (t >> 5)];
      if ((w >> (t & 31)) & 1u) {
        s = A.rank_id[r];
        break;
      }
    }
    A.src[t] = s;
  }
}

// camera.py:204-220 back_project (zero distortion) of one pixel at depth d.
// `(pc - t) @ R`: OpenBLAS gemm (>= 2 rows) fuses fma(q2,R2c, fma(q1,R1c, q0*R0c));
// one row goes through gemv, whose Haswell kernel sums unfused.
__device__ __forceinline__ void back_project1(const fvv_camera &c, double px, double py, double d,
                                              bool gemv, double &X, double &Y, double &Z) {
  const double yn = (py - c.cy) / c.fy;
  const double xn = (px - c.cx) / c.fx - c.skew * yn;
  const double q0 = xn * d - c.t[0], q1 = yn * d - c.t[1], q2 = d - c.t[2];
  double out[3];
#pragma unroll
  for (int col = 0; col < 3; ++col) {
    const double r0 = c.R[col], r1 = c.R[3 + col], r2 = c.R[6 + col];
    out[col] = gemv ? (q0 * r0 + q1 * r1) + q2 * r2 : fma(q2, r2, fma(q1, r1, q0 * r0));
  }
  X = out[0];
  Y = out[1];
  Z = out[2];
}

struct RenderArgs {
  fvv_camera virt;
  int ncam;
  int32_t cam_id[FVV_MAX_CAMS];
  int64_t frame_off[FVV_MAX_CAMS];
  fvv_camera cams[FVV_MAX_CAMS];
  const uint8_t *frames;
  const double *depth;
  const int32_t *ids;
  const int32_t *tri_src;
  uint8_t fallback[4];
  uint8_t *color;
  int32_t *source;
  uint8_t *covered;
  int8_t *code;     // optional: -2 uncovered, -1 fallback colour, else source rig position
  int64_t *counts;  // [0] covered pixels, [1 + pos] pixels sourced from camera pos
  const FrameInputs *in;  // when set: frames / frame_off from here (device)
};

__device__ __forceinline__ int cam_pos(const RenderArgs &A, int32_t id) {
  for (int c = 0; c < A.ncam; ++c)
    if (A.cam_id[c] == id) return c;
  return -1;
}

// covered pixels and pixels per source camera (numpy's one-row gemv rule
// applies when a count is 1); warp-aggregated atomics.
__global__ void render_count_kernel(const __grid_constant__ RenderArgs A) {
  pdl_wait();
  const int64_t np = (int64_t)A.virt.width * A.virt.height;
  const int lane = threadIdx.x & 31;
  for (int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; p0 < np;
       p0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = p0 + lane;
    const int32_t t = p < np ? A.ids[p] : -1;
    int c = -1;
    if (t >= 0) {
      const int32_t s = A.tri_src[t];
      if (s >= 0) c = cam_pos(A, s);
    }
    const unsigned cov = __ballot_sync(0xffffffffu, t >= 0);
    if (lane == 0 && cov) atomicAdd((unsigned long long *)A.counts, (unsigned long long)__popc(cov));
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    if (c >= 0 && lane == __ffs(grp) - 1)
      atomicAdd((unsigned long long *)(A.counts + 1 + c), (unsigned long long)__popc(grp));
  }
}

// render.py:46-61 sample_bilinear, render.py:104-113 rint/clip.
__global__ void render_color_kernel(const __grid_constant__ RenderArgs A) {
  pdl_wait();
  const int W = A.virt.width;
  const int64_t np = (int64_t)W * A.virt.height;
  const bool bp_gemv = A.counts[0] == 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = A.ids[p];
    uint8_t rgb[3] = {0, 0, 0};
    int32_t src = -1;
    int cpos = -1;
    if (t >= 0) {
      src = A.tri_src[t];
      const int c = src >= 0 ? cam_pos(A, src) : -1;
      cpos = c;
      if (c < 0) {
        rgb[0] = A.fallback[0];
        rgb[1] = A.fallback[1];
        rgb[2] = A.fallback[2];
      } else {
        double X, Y, Z;
        back_project1(A.virt, (double)(p % W), (double)(p / W), A.depth[p], bp_gemv, X, Y, Z);
        const fvv_camera &cam = A.cams[c];
        double u, v, zc;
        project_exact(cam, X, Y, Z, true, A.counts[1 + c] == 1, u, v, zc);
        const int w = cam.width, h = cam.height;
        u = fmin(fmax(u, 0.0), (double)w - 1.0);
        v = fmin(fmax(v, 0.0), (double)h - 1.0);
        const int x0 = (int)floor(u), y0 = (int)floor(v);
        const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
        const double fx = u - (double)x0, fy = v - (double)y0;
        const uint8_t *img = A.in ? A.in->frames + A.in->frame_off[c] : A.frames + A.frame_off[c];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const double a = img[((int64_t)y0 * w + x0) * 3 + ch];
          const double b = img[((int64_t)y0 * w + x1) * 3 + ch];
          const double cc = img[((int64_t)y1 * w + x0) * 3 + ch];
          const double d = img[((int64_t)y1 * w + x1) * 3 + ch];
          const double top = a * (1.0 - fx) + b * fx;
          const double bot = cc * (1.0 - fx) + d * fx;
          double q = rint(top * (1.0 - fy) + bot * fy);
          q = q < 0.0 ? 0.0 : (q > 255.0 ? 255.0 : q);
          rgb[ch] = (uint8_t)q;
        }
      }
    }
    A.color[3 * p] = rgb[0];
    A.color[3 * p + 1] = rgb[1];
    A.color[3 * p + 2] = rgb[2];
    A.source[p] = src;
    if (A.covered) A.covered[p] = t >= 0;
    if (A.code) A.code[p] = t < 0 ? (int8_t)-2 : (int8_t)cpos;
  }
}

__global__ void back_project_kernel(fvv_camera cam, const double *__restrict__ px,
                                    const double *__restrict__ d, int64_t n, double *out) {
  pdl_wait();
  const bool gemv = n == 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    back_project1(cam, px[2 * i], px[2 * i + 1], d[i], gemv, out[3 * i], out[3 * i + 1],
                  out[3 * i + 2]);
}

constexpr int kRasterGrid = 148 * 16;

static int fill_cams(RasterCams &C, const fvv_camera *cams, int ncam, const int64_t *off) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("raster: %d cameras (1..%d)", ncam, FVV_MAX_CAMS);
    return FVV_E_LIMIT;
  }
  memset(&C, 0, sizeof(C));
  C.ncam = ncam;
  for (int c = 0; c < ncam; ++c) {
    C.cams[c] = cams[c];
    C.depth_off[c] = off[c];
  }
  return FVV_OK;
}

}  // namespace fvv

using namespace fvv;

extern "C" {

static int64_t raster_queue_cap(int64_t num_triangles, int ncam) {
  int64_t cap = num_triangles * (int64_t)ncam;
  if (cap > (4ll << 20)) cap = 4ll << 20;
  return cap > 0 ? cap : 1;
}

static size_t align256(size_t n) { return (n + 255) & ~(size_t)255; }

// The FP32 filter's launch shape and its per-warp list sizes.
struct FilterShape {
  int64_t bx, nwl, wl_items, wl_pairs;
};

static FilterShape filter_shape(int64_t num_triangles, int ncam) {
  const int64_t nt = num_triangles > 0 ? num_triangles : 1;
  FilterShape f;
  f.bx = (nt + 255) / 256;
  if (f.bx > 148 * 8) f.bx = 148 * 8;
  f.nwl = f.bx * 8;  // 256-thread blocks
  // a filter warp visits ceil(nt / stride) chunks of 32 triangles x ncam cameras
  f.wl_items = (int64_t)ncam * 32 * ((nt + 256 * f.bx - 1) / (256 * f.bx));
  f.wl_pairs = 2 * f.wl_items;
  return f;
}

struct RasterLayout {
  size_t counts, queue, proj, q, slow, pairs, hits, total;
  int64_t hit_cap;
};

// hit-list entries of a one-camera raster (the virtual view's id pass)
static int64_t raster_hit_cap(int64_t num_triangles, int ncam) {
  if (ncam != 1) return 0;
  int64_t cap = 2 * num_triangles;
  cap = cap < (1 << 16) ? (1 << 16) : cap;
  return cap > ((int64_t)8 << 20) ? ((int64_t)8 << 20) : cap;
}

// [counters][per-warp list counts][big queue][projected vertices f64]
// [projected vertices f32][sweep items][candidate pixel pairs]
static RasterLayout raster_layout(int64_t num_vertices, int64_t num_triangles, int ncam) {
  const size_t nvc = (size_t)(num_vertices > 0 ? num_vertices : 1) * (size_t)ncam;
  const FilterShape f = filter_shape(num_triangles, ncam);
  RasterLayout L;
  L.counts = 256;
  L.queue = align256(L.counts + 2 * 4 * (size_t)f.nwl);
  L.proj = align256(L.queue + 8 * (size_t)raster_queue_cap(num_triangles, ncam));
  L.q = align256(L.proj + sizeof(double4) * nvc);
  L.slow = align256(L.q + sizeof(float2) * nvc);
  L.pairs = align256(L.slow + 4 * (size_t)(f.nwl * f.wl_items));
  L.hits = align256(L.pairs + sizeof(uint2) * (size_t)(f.nwl * f.wl_pairs));
  L.hit_cap = raster_hit_cap(num_triangles, ncam);
  L.total = L.hits + sizeof(uint4) * (size_t)L.hit_cap;
  return L;
}

size_t fvv_raster_workspace_bytes(int64_t num_vertices, int64_t num_triangles, int ncam) {
  return raster_layout(num_vertices, num_triangles, ncam).total;
}

// dirty == nullptr: the planes are filled with the background here.
// dirty != nullptr (contiguous planes only): the planes already hold the
// background except the 32-pixel tiles flagged in dirty[], which are reset;
// full_reset fills everything and clears the flags instead (first use).
static int rasterize_impl(const fvv_camera *cams, int ncam, const double *verts_dev, int64_t nv,
                          const int64_t *nv_dev, const int32_t *tris_dev, int64_t nt,
                          const int64_t *nt_dev,
                          double *depth_dev, const int64_t *plane_off, int32_t *tri_id_dev,
                          void *ws_dev, size_t ws_bytes, uint8_t *dirty, bool full_reset,
                          cudaStream_t st) {
  static thread_local RasterCams C;
  int rc = fill_cams(C, cams, ncam, plane_off);
  if (rc) return rc;
  for (int c = 0; c < ncam; ++c) {
    if (cams[c].width > 65535 || cams[c].height > 65535) {  // packed pixel pairs
      set_error("fvv_rasterize: camera %d image %dx%d exceeds 65535", cams[c].id, cams[c].width,
                cams[c].height);
      return FVV_E_LIMIT;
    }
  }
  if (nt > 0 && (nt * (int64_t)ncam >= 0xffffffffll || nt > (int64_t)kPairTriMask)) {
    // 32-bit item indices; pair entries hold 26-bit triangle indices
    set_error("fvv_rasterize: %lld triangles x %d cameras exceeds 2^32 - 1 (or 2^26 triangles)",
              (long long)nt, ncam);
    return FVV_E_LIMIT;
  }
  // background: depth +inf, id -1 (visibility.py:44-45); one fill when the
  // planes are contiguous (the executor's layout), else one per camera
  bool contiguous = true;
  int64_t total_px = 0;
  for (int c = 0; c < ncam; ++c) {
    contiguous = contiguous && plane_off[c] == plane_off[0] + total_px;
    total_px += (int64_t)cams[c].width * cams[c].height;
  }
  if (dirty && !contiguous) {
    set_error("fvv_rasterize_tracked: planes must be contiguous");
    return FVV_E_ARG;
  }
  if (dirty && full_reset) fill_async(dirty, 0, (size_t)((total_px + 31) >> 5), st);
  const bool tracked = dirty && !full_reset;
  // contiguous planes: the fill (or tracked reset) rides in the
  // vertex-projection launch (raster_prep_kernel); otherwise fill here
  const bool fused_fill = contiguous;
  for (int c = 0; c < (contiguous ? 1 : ncam); ++c) {
    const int64_t n = contiguous ? total_px : (int64_t)cams[c].width * cams[c].height;
    if (!fused_fill) {
      launch_k(fill_u64_kernel, 148 * 8, 256, 0, st, (unsigned long long *)(depth_dev + plane_off[c]),
                                               n, 0x7ff0000000000000ull);
      note_launches(1);
    }
    if (tri_id_dev && !tracked) fill_async(tri_id_dev + plane_off[c], 0xff, 4 * n, st);
  }
  const bool work = nt > 0 && nv > 0;
  const RasterLayout L = raster_layout(nv, nt, ncam);
  if (work && ws_bytes < L.total) {
    set_error("fvv_rasterize: workspace %zu < %zu bytes", ws_bytes, L.total);
    return FVV_E_ARG;
  }
  char *ws = (char *)ws_dev;
  if (fused_fill) {
    double4 *proj = work ? (double4 *)(ws + L.proj) : nullptr;
    float2 *q = work ? (float2 *)(ws + L.q) : nullptr;
    int64_t blocks = work ? (nv * ncam + 255) / 256 : 0;
    if (blocks > kRasterGrid) blocks = kRasterGrid;
    // fill blocks in proportion to the bytes they write (~0.3 us of work per
    // block); a tracked reset reads one flag per 32 pixels
    int64_t nb_fill = tracked ? total_px / (256 * 32 * 8) + 1 : total_px / (256 * 64) + 1;
    if (nb_fill > 148 * 8) nb_fill = 148 * 8;
    launch_k(raster_prep_kernel, (int)(blocks + nb_fill), 256, 0, st, C, verts_dev, work ? nv : 0, nv_dev, proj, q,
        (unsigned long long *)(depth_dev + plane_off[0]),
        tracked ? tri_id_dev + plane_off[0] : nullptr, tracked ? dirty : nullptr, total_px,
        (int)nb_fill);
    note_launches(1);
  } else if (work) {
    int64_t blocks = (nv * ncam + 255) / 256;
    if (blocks > kRasterGrid) blocks = kRasterGrid;
    launch_k(raster_vertex_kernel, (int)blocks, 256, 0, st, C, verts_dev, nv, nv_dev,
                                                     (double4 *)(ws + L.proj), (float2 *)(ws + L.q));
    note_launches(1);
  }
  if (!work) return cuda_check("fvv_rasterize");
  RasterArgs A;
  A.T = tris_dev;
  A.nt = nt;
  A.nt_dev = nt_dev;
  A.nv = nv;
  A.depth = depth_dev + (dirty ? plane_off[0] : 0);
  A.ids = tri_id_dev ? tri_id_dev + (dirty ? plane_off[0] : 0) : nullptr;
  A.dirty = dirty;
  A.qcount = (int64_t *)ws;
  const FilterShape fs = filter_shape(nt, ncam);
  A.overflow = (int *)(ws + 8);
  A.wcount = (int *)(ws + L.counts);
  A.nwl = fs.nwl;
  A.wl_items = fs.wl_items;
  A.wl_pairs = fs.wl_pairs;
  A.queue = (int64_t *)(ws + L.queue);
  A.qcap = raster_queue_cap(nt, ncam);
  A.P = (const double4 *)(ws + L.proj);
  A.Q = (const float2 *)(ws + L.q);
  A.slow = (uint32_t *)(ws + L.slow);
  A.pairs = (uint2 *)(ws + L.pairs);
  if (dirty)  // planes addressed relative to plane 0 (the dirty map's origin)
    for (int c = 0; c < ncam; ++c) C.depth_off[c] = plane_off[c] - plane_off[0];
  const bool hits = tri_id_dev && L.hit_cap > 0;
  A.hits = hits ? (uint4 *)(ws + L.hits) : nullptr;
  A.hit_count = (unsigned long long *)(ws + 16);
  A.hit_cap = L.hit_cap;
  fill_async(ws, 0, 32, st);  // big-queue counter, overflow flag, hit count
  launch_k(raster_filter_kernel, (unsigned)fs.bx, 256, 0, st, C, A);
  note_launches(1);
  // pass 0: depth (RED.MIN of the depth bits); ids wanted: the lowest
  // triangle id reaching the final depth, from the hit list pass 0 recorded
  // (one camera), else (or when the list overflowed) a pass 1 over the same
  // work lists
  for (int pass = 0; pass < (tri_id_dev ? 2 : 1); ++pass) {
    A.pass = pass;
    if (pass == 1 && hits) {
      launch_k(raster_hits_kernel, 148 * 8, 256, 0, st, A);
      note_launches(1);
    }
    if (hits && pass == 0)
      launch_k(raster_pair_kernel<true>, 148 * 16, 256, 0, st, C, A);
    else
      launch_k(raster_pair_kernel<false>, 148 * 16, 256, 0, st, C, A);
    launch_k(raster_small_kernel, 148 * 16, kRasterThreads, 0, st, C, A);
    launch_k(raster_big_kernel, 148 * 4, kBigThreads, 0, st, C, A);
    note_launches(3);
  }
  return cuda_check("fvv_rasterize");
}

int fvv_rasterize(const fvv_camera *cams, int ncam, const double *verts_dev, int64_t nv,
                  const int32_t *tris_dev, int64_t nt, const int64_t *nt_dev, double *depth_dev,
                  const int64_t *plane_off, int32_t *tri_id_dev, void *ws_dev, size_t ws_bytes,
                  void *stream) {
  return rasterize_impl(cams, ncam, verts_dev, nv, nullptr, tris_dev, nt, nt_dev, depth_dev,
                        plane_off, tri_id_dev, ws_dev, ws_bytes, nullptr, false,
                        (cudaStream_t)stream);
}

int fvv_rasterize_tracked(const fvv_camera *cams, int ncam, const double *verts_dev, int64_t nv,
                          const int64_t *nv_dev, const int32_t *tris_dev, int64_t nt,
                          const int64_t *nt_dev,
                          double *depth_dev, const int64_t *plane_off, int32_t *tri_id_dev,
                          void *ws_dev, size_t ws_bytes, uint8_t *dirty_dev, int full_reset,
                          void *stream) {
  if (!dirty_dev) {
    set_error("fvv_rasterize_tracked: dirty map required");
    return FVV_E_ARG;
  }
  return rasterize_impl(cams, ncam, verts_dev, nv, nv_dev, tris_dev, nt, nt_dev, depth_dev,
                        plane_off, tri_id_dev, ws_dev, ws_bytes, dirty_dev, full_reset != 0,
                        (cudaStream_t)stream);
}

int fvv_classify(const fvv_camera *cams, int ncam, const double *verts_dev,
                 const int32_t *tris_dev, int64_t nt, const int64_t *nt_dev,
                 const double *depth_dev, const int64_t *plane_off, double t_v,
                 uint32_t *vis_dev, int64_t vis_stride_words, void *stream) {
  return classify_sources(cams, ncam, verts_dev, tris_dev, nt, nt_dev, depth_dev, plane_off, t_v,
                          vis_dev, vis_stride_words, 0, nullptr, nullptr, nullptr,
                          (cudaStream_t)stream);
}

int fvv_triangle_sources(const int32_t *rank_pos, const int32_t *rank_id, int nrank,
                         const uint32_t *vis_dev, int64_t vis_stride_words, int64_t nt,
                         const int64_t *nt_dev, int32_t *src_dev, void *stream) {
  if (nrank < 0 || nrank > FVV_MAX_CAMS) {
    set_error("fvv_triangle_sources: %d cameras", nrank);
    return FVV_E_LIMIT;
  }
  static thread_local SourceArgs A;
  memset(&A, 0, sizeof(A));
  A.nrank = nrank;
  for (int r = 0; r < nrank; ++r) {
    A.rank_pos[r] = rank_pos[r];
    A.rank_id[r] = rank_id[r];
  }
  A.vis = vis_dev;
  A.vis_stride = vis_stride_words;
  A.nt = nt;
  A.nt_dev = nt_dev;
  A.src = src_dev;
  launch_k(sources_kernel, kRasterGrid, 256, 0, (cudaStream_t)stream, A);
  note_launches(1);
  return cuda_check("fvv_triangle_sources");
}

static int fill_render(RenderArgs &A, const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                       const int64_t *frame_off, const fvv_camera *virt, const double *depth_dev,
                       const int32_t *tri_id_dev, const int32_t *tri_src_dev,
                       const uint8_t *fallback, uint8_t *color_dev, int32_t *source_dev,
                       uint8_t *covered_dev, int64_t *counts_dev) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("render: %d cameras", ncam);
    return FVV_E_LIMIT;
  }
  memset(&A, 0, sizeof(A));
  A.virt = *virt;
  A.ncam = ncam;
  for (int c = 0; c < ncam; ++c) {
    A.cams[c] = rig[c];
    A.cam_id[c] = rig[c].id;
    A.frame_off[c] = frame_off ? frame_off[c] : 0;
  }
  A.frames = frames_dev;
  A.depth = depth_dev;
  A.ids = tri_id_dev;
  A.tri_src = tri_src_dev;
  for (int ch = 0; ch < 3; ++ch) A.fallback[ch] = fallback ? fallback[ch] : 0;
  A.color = color_dev;
  A.source = source_dev;
  A.covered = covered_dev;
  A.counts = counts_dev;
  return FVV_OK;
}

}  // extern "C"

int fvv::classify_sources(const fvv_camera *cams, int ncam, const double *verts_dev,
                          const int32_t *tris_dev, int64_t nt, const int64_t *nt_dev,
                          const double *depth_dev, const int64_t *plane_off, double t_v,
                          uint32_t *vis_dev, int64_t vis_stride_words, int nrank,
                          const int32_t *rank_pos, const int32_t *rank_id, int32_t *src_dev,
                          cudaStream_t st) {
  static thread_local RasterCams C;
  int rc = fill_cams(C, cams, ncam, plane_off);
  if (rc) return rc;
  if (nrank < 0 || nrank > FVV_MAX_CAMS) {
    set_error("fvv_classify: %d ranked cameras", nrank);
    return FVV_E_LIMIT;
  }
  static thread_local ClassifyArgs A;
  memset(&A, 0, sizeof(A));
  A.V = verts_dev;
  A.T = tris_dev;
  A.nt = nt;
  A.nt_dev = nt_dev;
  A.depth = depth_dev;
  A.t_v = t_v;
  A.vis = vis_dev;
  A.vis_stride = vis_stride_words;
  A.src = src_dev;
  A.nrank = src_dev ? nrank : 0;
  for (int r = 0; r < A.nrank; ++r) {
    A.rank_pos[r] = rank_pos[r];
    A.rank_id[r] = rank_id[r];
  }
  launch_k(classify_kernel, kRasterGrid, 256, 0, st, C, A);
  note_launches(1);
  return cuda_check("fvv_classify");
}

int fvv::render_view_coded_bound(const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                                 const int64_t *frame_off, const FrameInputs *in,
                                 const fvv_camera *virt, const double *depth_dev,
                                 const int32_t *tri_id_dev, const int32_t *tri_src_dev,
                                 const uint8_t *fallback, uint8_t *color_dev,
                                 int32_t *source_dev, uint8_t *covered_dev, int8_t *code_dev,
                                 const int64_t *counts_dev, cudaStream_t st) {
  static thread_local RenderArgs A;
  int rc = fill_render(A, rig, ncam, frames_dev, frame_off, virt, depth_dev, tri_id_dev,
                       tri_src_dev, fallback, color_dev, source_dev, covered_dev,
                       const_cast<int64_t *>(counts_dev));
  if (rc) return rc;
  A.code = code_dev;
  A.in = in;
  launch_k(render_color_kernel, kRasterGrid, 256, 0, st, A);
  note_launches(1);
  return cuda_check("fvv_render_view");
}

extern "C" {

int fvv_render_count(const fvv_camera *rig, int ncam, const fvv_camera *virt,
                     const int32_t *tri_id_dev, const int32_t *tri_src_dev, int64_t *counts_dev,
                     void *stream) {
  static thread_local RenderArgs A;
  int rc = fill_render(A, rig, ncam, nullptr, nullptr, virt, nullptr, tri_id_dev, tri_src_dev,
                       nullptr, nullptr, nullptr, nullptr, counts_dev);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  fill_async(counts_dev, 0, sizeof(int64_t) * (1 + ncam), st);
  launch_k(render_count_kernel, kRasterGrid, 256, 0, st, A);
  note_launches(1);
  return cuda_check("fvv_render_count");
}

int fvv_render_view_coded(const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                          const int64_t *frame_off, const fvv_camera *virt,
                          const double *depth_dev, const int32_t *tri_id_dev,
                          const int32_t *tri_src_dev, const uint8_t *fallback,
                          uint8_t *color_dev, int32_t *source_dev, uint8_t *covered_dev,
                          int8_t *code_dev, const int64_t *counts_dev, void *stream) {
  return render_view_coded_bound(rig, ncam, frames_dev, frame_off, nullptr, virt, depth_dev,
                                 tri_id_dev, tri_src_dev, fallback, color_dev, source_dev,
                                 covered_dev, code_dev, counts_dev, (cudaStream_t)stream);
}

int fvv_render_view(const fvv_camera *rig, int ncam, const uint8_t *frames_dev,
                    const int64_t *frame_off, const fvv_camera *virt, const double *depth_dev,
                    const int32_t *tri_id_dev, const int32_t *tri_src_dev, const uint8_t *fallback,
                    uint8_t *color_dev, int32_t *source_dev, uint8_t *covered_dev,
                    const int64_t *counts_dev, void *stream) {
  return fvv_render_view_coded(rig, ncam, frames_dev, frame_off, virt, depth_dev, tri_id_dev,
                               tri_src_dev, fallback, color_dev, source_dev, covered_dev,
                               nullptr, counts_dev, stream);
}

int fvv_back_project(const fvv_camera *cam, const double *pixel_dev, const double *depth_dev,
                     int64_t n, double *out_dev, void *stream) {
  if (n <= 0) return FVV_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > kRasterGrid) blocks = kRasterGrid;
  launch_k(back_project_kernel, (int)blocks, 256, 0, (cudaStream_t)stream, *cam, pixel_dev, depth_dev,
                                                                      n, out_dev);
  note_launches(1);
  return cuda_check("fvv_back_project");
}

}  // extern "C"
