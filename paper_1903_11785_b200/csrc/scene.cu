// Benchmark/test harness, not hot path: exact per-pixel ray
// casts of ellipsoid scenes into silhouettes and Lambertian-shaded frames,
// the GPU twin of paper_1903_11785_b200/synthetic.py render_camera (which
// follows the reference's synthetic.py:165-218). Generates the inputs of
// the volleyball-scale workloads fast enough to feed multi-frame runs.
#include "fvv_common.cuh"

namespace fvv {

constexpr int kPartDoubles = 18;  // centre[3] orient[9] (row-major) semi[3] rgb[3]

__global__ void render_parts_kernel(fvv_camera cam, const double *__restrict__ parts, int nparts,
                                    uint8_t *sil, uint8_t *rgb, double ambient, double lx,
                                    double ly, double lz, double bg_r, double bg_g, double bg_b) {
  pdl_wait();
  extern __shared__ double sp[];
  for (int i = threadIdx.x; i < nparts * kPartDoubles; i += blockDim.x) sp[i] = parts[i];
  __syncthreads();
  const int W = cam.width, H = cam.height;
  // optical centre C = -R^T t
  const double ox = -(cam.R[0] * cam.t[0] + cam.R[3] * cam.t[1] + cam.R[6] * cam.t[2]);
  const double oy = -(cam.R[1] * cam.t[0] + cam.R[4] * cam.t[1] + cam.R[7] * cam.t[2]);
  const double oz = -(cam.R[2] * cam.t[0] + cam.R[5] * cam.t[1] + cam.R[8] * cam.t[2]);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < (int64_t)W * H;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(p % W), v = (double)(p / W);
    const double yn = (v - cam.cy) / cam.fy;
    const double xn = (u - cam.cx) / cam.fx - cam.skew * yn;
    // d = (xn, yn, 1) @ R, normalised (camera.py:223-235 pixel_rays)
    double dx = xn * cam.R[0] + yn * cam.R[3] + cam.R[6];
    double dy = xn * cam.R[1] + yn * cam.R[4] + cam.R[7];
    double dz = xn * cam.R[2] + yn * cam.R[5] + cam.R[8];
    const double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    dx *= inv;
    dy *= inv;
    dz *= inv;
    double best = INFINITY;
    int owner = -1;
    for (int k = 0; k < nparts; ++k) {
      const double *q = sp + k * kPartDoubles;
      const double rx = ox - q[0], ry = oy - q[1], rz = oz - q[2];
      double oo[3], dd[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {  // local = (x @ Q) / semi
        const double s = q[12 + a];
        oo[a] = (rx * q[3 + a] + ry * q[6 + a] + rz * q[9 + a]) / s;
        dd[a] = (dx * q[3 + a] + dy * q[6 + a] + dz * q[9 + a]) / s;
      }
      const double A = dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2];
      const double B = dd[0] * oo[0] + dd[1] * oo[1] + dd[2] * oo[2];
      const double C = oo[0] * oo[0] + oo[1] * oo[1] + oo[2] * oo[2] - 1.0;
      const double disc = B * B - A * C;
      if (disc < 0.0) continue;
      const double sq = sqrt(disc);
      const double t0 = (-B - sq) / A, t1 = (-B + sq) / A;
      const double t = t0 > 1e-9 ? t0 : t1;
      if (t > 1e-9 && t < best) {
        best = t;
        owner = k;
      }
    }
    if (sil) sil[p] = owner >= 0;
    if (rgb) {
      double c0 = bg_r, c1 = bg_g, c2 = bg_b;
      if (owner >= 0) {
        const double *q = sp + owner * kPartDoubles;
        const double hx = ox + best * dx - q[0], hy = oy + best * dy - q[1],
                     hz = oz + best * dz - q[2];
        double n[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double s = q[12 + a];
          const double l = (hx * q[3 + a] + hy * q[6 + a] + hz * q[9 + a]) / (s * s);
          n[0] += l * q[3 + 3 * 0 + a];
          n[1] += l * q[3 + 3 * 1 + a];
          n[2] += l * q[3 + 3 * 2 + a];
        }
        const double nn = 1.0 / sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        const double diff = fmax(0.0, -(n[0] * lx + n[1] * ly + n[2] * lz) * nn);
        const double lum = ambient + (1.0 - ambient) * diff;
        c0 = q[15] * lum;
        c1 = q[16] * lum;
        c2 = q[17] * lum;
      }
      rgb[3 * p] = (uint8_t)fmin(fmax(rint(c0), 0.0), 255.0);
      rgb[3 * p + 1] = (uint8_t)fmin(fmax(rint(c1), 0.0), 255.0);
      rgb[3 * p + 2] = (uint8_t)fmin(fmax(rint(c2), 0.0), 255.0);
    }
  }
}

}  // namespace fvv

using namespace fvv;

extern "C" int fvv_render_ellipsoids(const fvv_camera *cam, const double *parts_dev, int nparts,
                                     uint8_t *sil_dev, uint8_t *rgb_dev, const double *shading,
                                     void *stream) {
  if (nparts < 0 || nparts * kPartDoubles * 8 > 160 * 1024) {
    set_error("fvv_render_ellipsoids: %d parts", nparts);
    return FVV_E_LIMIT;
  }
  const size_t smem = (size_t)(nparts > 0 ? nparts : 1) * kPartDoubles * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(render_parts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  // shading = {ambient, light x, y, z, background r, g, b}
  launch_k(render_parts_kernel, 148 * 4, 256, smem, (cudaStream_t)stream, *cam, parts_dev, nparts, sil_dev, rgb_dev, shading[0], shading[1], shading[2], shading[3],
      shading[4], shading[5], shading[6]);
  note_launches(1);
  return cuda_check("fvv_render_ellipsoids");
}
