// Silhouette extraction upstream of the carve (silhouette.py:59-109,
// SURVEY.md 8f2): exact Euclidean distance map of the proposal mask,
// per-pixel background statistics, distance-adaptive thresholding.
//
// EDT: squared distances are exact integers: per column the squared
// distance to the nearest proposal pixel above/below (two sweeps), then per
// row the lower envelope of parabolas (Felzenszwalb-Huttenlocher) with every
// breakpoint comparison done on int64 cross products, so sqrt of the result
// equals scipy's distance_transform_edt bit for bit. Background statistics
// accumulate over frames in numpy's order (axis 0, sequential); thresholds
// use the reference's float64 expressions (-fmad=false).
#include <climits>

#include "fvv_common.cuh"

namespace fvv {

constexpr int32_t kNoFeature = INT32_MAX;

__global__ void edt_columns_kernel(const uint8_t *__restrict__ prop, int H, int W,
                                   int32_t *__restrict__ g) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
    int last = -1;
    for (int y = 0; y < H; ++y) {
      if (prop[(int64_t)y * W + x]) last = y;
      g[(int64_t)y * W + x] = last < 0 ? kNoFeature : (y - last) * (y - last);
    }
    last = -1;
    for (int y = H - 1; y >= 0; --y) {
      if (prop[(int64_t)y * W + x]) last = y;
      if (last >= 0) {
        const int32_t d = (last - y) * (last - y);
        int32_t *p = g + (int64_t)y * W + x;
        if (d < *p) *p = d;
      }
    }
  }
}

// breakpoint of parabolas rooted at p < q: s = ((f_q + q^2) - (f_p + p^2)) / (2 (q - p))
__device__ __forceinline__ void breakpoint(int p, int64_t fp, int q, int64_t fq, int64_t &num,
                                           int64_t &den) {
  num = (fq + (int64_t)q * q) - (fp + (int64_t)p * p);
  den = 2 * (int64_t)(q - p);
}

// One lane per row; the envelope's parabola roots live in this lane's slice
// of shared memory.
__global__ void edt_rows_kernel(const int32_t *__restrict__ g, int H, int W, int rows_per_block,
                                int32_t *__restrict__ sq) {
  pdl_wait();
  extern __shared__ uint16_t roots[];
  const int lane = threadIdx.x;
  const int y = blockIdx.x * rows_per_block + lane;
  if (lane >= rows_per_block || y >= H) return;
  uint16_t *v = roots + (int64_t)lane * W;
  const int32_t *gr = g + (int64_t)y * W;
  int k = -1;
  for (int q = 0; q < W; ++q) {
    const int32_t fq = gr[q];
    if (fq == kNoFeature) continue;
    while (k >= 1) {
      int64_t n1, d1, n2, d2;
      breakpoint(v[k], gr[v[k]], q, fq, n1, d1);             // s(v[k], q)
      breakpoint(v[k - 1], gr[v[k - 1]], v[k], gr[v[k]], n2, d2);  // z[k]
      if (n1 * d2 <= n2 * d1) --k; else break;
    }
    v[++k] = (uint16_t)q;
  }
  int32_t *out = sq + (int64_t)y * W;
  if (k < 0) {  // no proposal pixel anywhere (rows are all-or-nothing)
    for (int x = 0; x < W; ++x) out[x] = kNoFeature;
    return;
  }
  int j = 0;
  for (int x = 0; x < W; ++x) {
    while (j < k) {
      int64_t n, d;
      breakpoint(v[j], gr[v[j]], v[j + 1], gr[v[j + 1]], n, d);
      if (n < (int64_t)x * d) ++j; else break;
    }
    const int64_t dx = x - (int)v[j];
    out[x] = (int32_t)(dx * dx + gr[v[j]]);
  }
}

__global__ void sq_to_dm_kernel(const int32_t *__restrict__ sq, int64_t n, double *__restrict__ dm) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dm[i] = sq[i] == kNoFeature ? INFINITY : sqrt((double)sq[i]);
}

// silhouette.py:72-87: numpy reduces axis 0 of the (K, ...) stack in order.
__global__ void background_kernel(const uint8_t *__restrict__ frames, int64_t K, int64_t n,
                                  double *__restrict__ mean, double *__restrict__ sd) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = (double)frames[i];
    for (int64_t k = 1; k < K; ++k) s = s + (double)frames[k * n + i];
    const double m = s / (double)K;
    double v = 0.0;
    for (int64_t k = 0; k < K; ++k) {
      const double d = (double)frames[k * n + i] - m;
      v = (k == 0) ? d * d : v + d * d;
    }
    const double st = sqrt(v / (double)K);
    mean[i] = m;
    sd[i] = st > 2.0 ? st : 2.0;  // np.maximum(std, STD_FLOOR)
  }
}

// silhouette.py:90-109 + AdaptiveParams.threshold (silhouette.py:44-47).
__global__ void extract_kernel(const uint8_t *__restrict__ frame, const double *__restrict__ mean,
                               const double *__restrict__ sd, int64_t npx, int C,
                               const int32_t *__restrict__ sq, const double *__restrict__ dm,
                               double theta_near, double theta_far, double d_max,
                               uint8_t *__restrict__ out) {
  pdl_wait();
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx;
       p += (int64_t)gridDim.x * blockDim.x) {
    double dev = -INFINITY;
    for (int c = 0; c < C; ++c) {
      const double x = (double)frame[p * C + c];
      const double d = fabs(x - mean[p * C + c]) / sd[p * C + c];
      if (d > dev || isnan(d)) dev = d;
    }
    const double dist = dm ? dm[p] : (sq[p] == kNoFeature ? INFINITY : sqrt((double)sq[p]));
    double t = dist / d_max;
    t = t < 1.0 ? t : 1.0;
    const double thr = theta_near + (theta_far - theta_near) * t;
    out[p] = dev > thr;
  }
}

static int blocks_for(int64_t n, int threads, int cap) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  return (int)(b > 0 ? b : 1);
}

}  // namespace fvv

using namespace fvv;

extern "C" {

int fvv_distance_map(const uint8_t *prop_dev, int64_t H, int64_t W, int32_t *sqdist_dev,
                     double *dm_dev, int32_t *ws_dev, void *stream) {
  if (H <= 0 || W <= 0 || W > 65535 || H > 65535) {
    set_error("fvv_distance_map: image %lld x %lld", (long long)H, (long long)W);
    return FVV_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  launch_k(edt_columns_kernel, blocks_for(W, 128, 148 * 8), 128, 0, st, prop_dev, (int)H, (int)W,
                                                                  ws_dev);
  int rows = (int)((160 * 1024) / (2 * W));
  if (rows > 32) rows = 32;
  if (rows < 1) rows = 1;
  const size_t smem = (size_t)rows * W * sizeof(uint16_t);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(edt_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  launch_k(edt_rows_kernel, (int)((H + rows - 1) / rows), 32, smem, st, ws_dev, (int)H, (int)W, rows,
                                                                  sqdist_dev);
  note_launches(2);
  if (dm_dev) {
    launch_k(sq_to_dm_kernel, blocks_for(H * W, 256, 148 * 8), 256, 0, st, sqdist_dev, H * W, dm_dev);
    note_launches(1);
  }
  return cuda_check("fvv_distance_map");
}

int fvv_background(const uint8_t *frames_dev, int64_t K, int64_t n, double *mean_dev,
                   double *std_dev, void *stream) {
  if (K < 2) {
    set_error("need at least 2 background frames");
    return FVV_E_ARG;
  }
  launch_k(background_kernel, blocks_for(n, 256, 148 * 8), 256, 0, (cudaStream_t)stream, frames_dev, K, n, mean_dev, std_dev);
  note_launches(1);
  return cuda_check("fvv_background");
}

int fvv_extract_silhouette(const uint8_t *frame_dev, const double *mean_dev,
                           const double *std_dev, int64_t npx, int C, const int32_t *sqdist_dev,
                           const double *dm_dev, double theta_near, double theta_far,
                           double d_max, uint8_t *mask_dev, void *stream) {
  launch_k(extract_kernel, blocks_for(npx, 256, 148 * 8), 256, 0, (cudaStream_t)stream, frame_dev, mean_dev, std_dev, npx, C, sqdist_dev, dm_dev, theta_near, theta_far, d_max,
      mask_dev);
  note_launches(1);
  return cuda_check("fvv_extract_silhouette");
}

}  // extern "C"
