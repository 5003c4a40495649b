// The reference's synthetic scene renderer on the GPU (synthetic.py:21-243,
// SURVEY.md 8f4): per pixel, the camera ray (camera.py:223-235
// pixel_rays), the nearest sphere/box hit (cast_rays, Sphere/Box.ray_hits),
// the analytic silhouette and the Lambertian frame (shade_frame), plus the
// eroded foreground proposal (proposal_from_silhouette, scipy
// binary_erosion with the 3x3 cross and border 0). Float64 in numpy's
// order, with OpenBLAS's FMA chains where numpy calls BLAS (verified on
// the reference, scripts/make_golden.py): d_cam @ R as gemm
// fma(z, R2k, fma(y, R1k, x R0k)); dirs @ v (gemv, N x 3) as
// fma(a2, v2, fma(a0, v0, a1 v1)); 3-vector norms as sqrt((a0^2 + a1^2) + a2^2).
#include <cmath>

#include "fvv_common.cuh"

namespace fvv {

// object record, float64: sphere {0, center[3], radius^2, color[3]},
// box {1, lo[3], hi[3], color[3]} (radius^2 as Python's radius**2); the
// camera-dependent terms are formed in the kernel in numpy's order
constexpr int kSynthRec = 10;

struct SynthArgs {
  fvv_camera cam;
  double light[3];
  double ambient, one_minus_ambient, bg[3];
  const double *objs;
  int nobj;
  const double *noise;  // (H, W, 3) added before rounding, or null
  uint8_t *sil, *rgb;
};

__device__ __forceinline__ double sphere_hit(const double *r, const double o[3],
                                             const double d[3]) {
  const double oc[3] = {o[0] - r[1], o[1] - r[2], o[2] - r[3]};  // origin - center
  const double b = fma(d[2], oc[2], fma(d[0], oc[0], d[1] * oc[1]));  // dirs @ oc (gemv)
  const double c = ((oc[0] * oc[0] + oc[1] * oc[1]) + oc[2] * oc[2]) - r[4];  // ddot - r**2
  const double disc = b * b - c;
  const bool hit = disc >= 0.0;
  const double sq = sqrt(hit ? disc : 0.0);
  const double t0 = -b - sq, t1 = -b + sq;
  const double t = t0 > 1e-9 ? t0 : t1;
  return (hit && t > 1e-9) ? t : INFINITY;
}

__device__ __forceinline__ double nanmax3(double a, double b, double c) {
  double m = NAN;
  if (!isnan(a)) m = a;
  if (!isnan(b) && (isnan(m) || b > m)) m = b;
  if (!isnan(c) && (isnan(m) || c > m)) m = c;
  return m;
}
__device__ __forceinline__ double nanmin3(double a, double b, double c) {
  double m = NAN;
  if (!isnan(a)) m = a;
  if (!isnan(b) && (isnan(m) || b < m)) m = b;
  if (!isnan(c) && (isnan(m) || c < m)) m = c;
  return m;
}
// np.minimum / np.maximum propagate NaN
__device__ __forceinline__ double npmin(double a, double b) {
  return (isnan(a) || isnan(b)) ? NAN : (a < b ? a : b);
}
__device__ __forceinline__ double npmax(double a, double b) {
  return (isnan(a) || isnan(b)) ? NAN : (a > b ? a : b);
}

__device__ __forceinline__ double box_hit(const double *r, const double o[3], const double d[3]) {
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    const double inv = 1.0 / d[k];
    const double tl = (r[1 + k] - o[k]) * inv, th = (r[4 + k] - o[k]) * inv;
    lo[k] = npmin(tl, th);
    hi[k] = npmax(tl, th);
  }
  const double tmin = nanmax3(lo[0], lo[1], lo[2]);
  const double tmax = nanmin3(hi[0], hi[1], hi[2]);
  const bool hit = (tmax >= npmax(tmin, 1e-9)) && (tmax > 1e-9);
  const double t = tmin > 1e-9 ? tmin : tmax;
  return hit ? t : INFINITY;
}

__global__ void synth_kernel(const __grid_constant__ SynthArgs A) {
  pdl_wait();
  const int W = A.cam.width, H = A.cam.height;
  const int64_t np_ = (int64_t)W * H;
  const fvv_camera &c = A.cam;
  // camera centre -R^T t (gemv order), as camera.py:62-64
  double org[3];
  for (int k = 0; k < 3; ++k)
    org[k] = -fma(c.R[6 + k], c.t[2], fma(c.R[k], c.t[0], c.R[3 + k] * c.t[1]));
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np_;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(p % W), v = (double)(p / W);
    const double yn = (v - c.cy) / c.fy;
    const double xn = (u - c.cx) / c.fx - c.skew * yn;
    double d[3];
    for (int k = 0; k < 3; ++k)  // (xn, yn, 1) @ R (gemm chain)
      d[k] = fma(1.0, c.R[6 + k], fma(yn, c.R[3 + k], xn * c.R[k]));
    const double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    for (int k = 0; k < 3; ++k) d[k] = d[k] / nrm;
    double best = INFINITY;
    int bo = -1;
    for (int o = 0; o < A.nobj; ++o) {  // cast_rays: strict <, object order
      const double *r = A.objs + (int64_t)kSynthRec * o;
      const double t = r[0] == 0.0 ? sphere_hit(r, org, d) : box_hit(r, org, d);
      if (t < best) {
        best = t;
        bo = o;
      }
    }
    if (A.sil) A.sil[p] = isfinite(best);
    if (!A.rgb) continue;
    double img[3] = {A.bg[0], A.bg[1], A.bg[2]};
    if (bo >= 0) {
      const double *r = A.objs + (int64_t)kSynthRec * bo;
      double pt[3], n[3];
      for (int k = 0; k < 3; ++k) pt[k] = org[k] + best * d[k];
      if (r[0] == 0.0) {  // Sphere.normal_at
        for (int k = 0; k < 3; ++k) n[k] = pt[k] - r[1 + k];
        const double nn = sqrt((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2]);
        for (int k = 0; k < 3; ++k) n[k] = n[k] / nn;
      } else {  // Box.normal_at: sign of the dominant relative coordinate
        double rel[3];
        for (int k = 0; k < 3; ++k) {
          const double mid = 0.5 * (r[1 + k] + r[4 + k]), half = 0.5 * (r[4 + k] - r[1 + k]);
          rel[k] = (pt[k] - mid) / half;
        }
        int ax = 0;
        double best_abs = fabs(rel[0]);
        for (int k = 1; k < 3; ++k)
          if (fabs(rel[k]) > best_abs || isnan(fabs(rel[k])) && !isnan(best_abs)) {
            best_abs = fabs(rel[k]);
            ax = k;
          }
        for (int k = 0; k < 3; ++k) n[k] = 0.0;
        n[ax] = rel[ax] > 0.0 ? 1.0 : (rel[ax] < 0.0 ? -1.0 : rel[ax]);
      }
      const double dot = fma(n[2], A.light[2], fma(n[0], A.light[0], n[1] * A.light[1]));
      const double neg = -dot;
      const double diffuse = isnan(neg) ? neg : (neg > 0.0 ? neg : 0.0);  // np.maximum(0, .)
      const double shade = A.ambient + A.one_minus_ambient * diffuse;
      const double *col = r + (r[0] == 0.0 ? 5 : 7);
      for (int k = 0; k < 3; ++k) img[k] = col[k] * shade;
    }
    for (int k = 0; k < 3; ++k) {
      double x = img[k];
      if (A.noise) x = x + A.noise[3 * p + k];
      x = rint(x);
      x = x < 0.0 ? 0.0 : (x > 255.0 ? 255.0 : x);  // np.clip
      A.rgb[3 * p + k] = (uint8_t)x;
    }
  }
}

// One erosion iteration with the 3x3 cross, outside pixels = 0.
__global__ void erode_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int W,
                             int H) {
  pdl_wait();
  const int64_t np_ = (int64_t)W * H;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np_;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(p % W), y = (int)(p / W);
    uint8_t v = in[p];
    v = v && x > 0 && in[p - 1];
    v = v && x < W - 1 && in[p + 1];
    v = v && y > 0 && in[p - W];
    v = v && y < H - 1 && in[p + W];
    out[p] = v;
  }
}

}  // namespace fvv

using namespace fvv;

extern "C" {

int fvv_synth_render(const fvv_camera *cam, const double *light,
                     const double *shading, const double *objs_dev, int nobj,
                     const double *noise_dev, uint8_t *sil_dev, uint8_t *rgb_dev, void *stream) {
  if (!cam || !light || !shading || nobj < 0 || (nobj > 0 && !objs_dev)) {
    set_error("fvv_synth_render: bad arguments");
    return FVV_E_ARG;
  }
  static thread_local SynthArgs A;
  A.cam = *cam;
  for (int k = 0; k < 3; ++k) {
    A.light[k] = light[k];
    A.bg[k] = shading[2 + k];
  }
  A.ambient = shading[0];
  A.one_minus_ambient = shading[1];
  A.objs = objs_dev;
  A.nobj = nobj;
  A.noise = noise_dev;
  A.sil = sil_dev;
  A.rgb = rgb_dev;
  const int64_t np_ = (int64_t)cam->width * cam->height;
  int64_t blocks = (np_ + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(synth_kernel, (int)(blocks > 0 ? blocks : 1), 256, 0, (cudaStream_t)stream, A);
  note_launches(1);
  return cuda_check("fvv_synth_render");
}

int fvv_erode_cross(const uint8_t *in_dev, uint8_t *tmp_dev, uint8_t *out_dev, int width,
                    int height, int iterations, void *stream) {
  if (width <= 0 || height <= 0 || iterations < 0) {
    set_error("fvv_erode_cross: bad arguments");
    return FVV_E_ARG;
  }
  const int64_t np_ = (int64_t)width * height;
  cudaStream_t st = (cudaStream_t)stream;
  if (iterations == 0) {
    cudaMemcpyAsync(out_dev, in_dev, (size_t)np_, cudaMemcpyDeviceToDevice, st);
    return cuda_check("fvv_erode_cross");
  }
  int64_t blocks = (np_ + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const uint8_t *src = in_dev;
  for (int i = 0; i < iterations; ++i) {
    // ping-pong so the last iteration lands in out_dev
    uint8_t *dst = ((iterations - 1 - i) % 2 == 0) ? out_dev : tmp_dev;
    launch_k(erode_kernel, (int)blocks, 256, 0, st, src, dst, width, height);
    src = dst;
  }
  note_launches(iterations);
  return cuda_check("fvv_erode_cross");
}

}  // extern "C"
