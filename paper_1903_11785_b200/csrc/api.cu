// C-ABI plumbing (errors, version) plus the small camera kernels:
// fvv_project (camera.py:164-201) and fvv_pack_silhouettes (hull.py:63-75).
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstring>

#include "fvv_common.cuh"

namespace fvv {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

static thread_local long long t_launches = 0;  // this thread's (graph capture counts its own)
void note_launches(long long n) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  t_launches += n;
}
long long thread_launch_count() { return t_launches; }

// cudaMemsetAsync as a kernel launched with programmatic serialisation:
// inside a frame graph a memset node would break the chain of early-launched
// kernels (each following launch then starts cold). 16-byte stores for the
// aligned body, bytes for the head and tail.
__global__ void fill_bytes_kernel(uint8_t *p, size_t n, uint32_t v4) {
  pdl_wait();
  size_t head = (16 - ((uintptr_t)p & 15)) & 15;
  if (head > n) head = n;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  if (tid < head) p[tid] = (uint8_t)v4;
  const size_t body = (n - head) / 16;
  uint4 *q = reinterpret_cast<uint4 *>(p + head);
  const uint4 vv = make_uint4(v4, v4, v4, v4);
  for (size_t i = tid; i < body; i += stride) q[i] = vv;
  const size_t tail = head + body * 16;
  if (tid < n - tail) p[tail + tid] = (uint8_t)v4;
}

void fill_async(void *p, int value, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  const uint32_t v4 = (uint32_t)(uint8_t)value * 0x01010101u;
  size_t blocks = (bytes / 16 + 255) / 256 + 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_k(fill_bytes_kernel, (unsigned)blocks, 256, 0, st, (uint8_t *)p, bytes, v4);
  note_launches(1);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("FVV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FVV_E_CUDA;
  }
  return FVV_OK;
}

__global__ void project_kernel(fvv_camera cam, const double *__restrict__ pts, int64_t n,
                               bool use_dist, bool gemv, double *__restrict__ pix,
                               double *__restrict__ zo, uint8_t *__restrict__ ino) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double u, v, z;
    bool in = project_exact(cam, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], use_dist, gemv, u,
                            v, z);
    pix[2 * i] = u;
    pix[2 * i + 1] = v;
    zo[i] = z;
    ino[i] = in;
  }
}

struct PackParams {
  int ncam;
  const uint8_t *masks;
  const FrameInputs *in;  // when set: masks from in->masks
  uint32_t *sil;
  int64_t mask_off[FVV_MAX_CAMS];
  int64_t sil_off[FVV_MAX_CAMS];
  int32_t width[FVV_MAX_CAMS];
  int32_t height[FVV_MAX_CAMS];
  int64_t word_start[FVV_MAX_CAMS + 1];  // cumulative words over cameras
};

// Rows whose width is a multiple of 32 (1080p, 4K): each thread turns 32
// mask bytes (two 16-byte loads) into one word, so a warp streams 1 KB.
__device__ __forceinline__ const uint8_t *pack_masks(const PackParams &p) {
  const uint8_t *m = p.masks;
  if (p.in != nullptr) m = p.in->masks;
  return m;
}

__global__ void pack_wide_kernel(const __grid_constant__ PackParams p) {
  pdl_wait();
  const int64_t total = p.word_start[p.ncam];
  const uint8_t *masks = pack_masks(p);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    while (w >= p.word_start[c + 1]) ++c;
    const int64_t local = w - p.word_start[c];
    const uint4 *src = reinterpret_cast<const uint4 *>(masks + p.mask_off[c] + local * 32);
    const uint4 a = __ldcs(src), b = __ldcs(src + 1);
    const uint32_t q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // byte j of q[k] nonzero -> bit 4k + j: 0xff per nonzero byte, its top
      // bits gathered into bits 28..31 by one multiply (the four partial
      // products land on distinct bits, so nothing carries)
      const uint32_t ne = __vcmpne4(q[k], 0u) & 0x80808080u;
      bits |= ((ne * 0x00204081u) >> 28) << (4 * k);
    }
    p.sil[p.sil_off[c] + local] = bits;
  }
}

// One warp builds one 32-pixel word from 32 coalesced mask bytes (ballot).
__global__ void pack_kernel(const __grid_constant__ PackParams p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t total = p.word_start[p.ncam];
  const uint8_t *masks = pack_masks(p);
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < total; w += warps) {
    int c = 0;
    while (w >= p.word_start[c + 1]) ++c;
    int64_t local = w - p.word_start[c];
    int stride = (p.width[c] + 31) >> 5;
    int64_t row = local / stride;
    int x = (int)(local - row * stride) * 32 + lane;
    bool fg = false;
    if (x < p.width[c]) fg = masks[p.mask_off[c] + row * p.width[c] + x] != 0;
    uint32_t bits = __ballot_sync(0xffffffffu, fg);
    if (lane == 0) p.sil[p.sil_off[c] + local] = bits;
  }
}

int pack_silhouettes_bound(const fvv_camera *cams, int ncam, const uint8_t *masks_dev,
                           const FrameInputs *in, const int64_t *mask_off, uint32_t *sil_dev,
                           const int64_t *sil_word_off, cudaStream_t st) {
  if (ncam < 1 || ncam > FVV_MAX_CAMS) {
    set_error("fvv_pack_silhouettes: %d cameras (limit %d)", ncam, FVV_MAX_CAMS);
    return ncam < 1 ? FVV_E_ARG : FVV_E_LIMIT;
  }
  PackParams p;
  memset(&p, 0, sizeof(p));
  p.ncam = ncam;
  p.masks = masks_dev;
  p.in = in;
  p.sil = sil_dev;
  p.word_start[0] = 0;
  for (int c = 0; c < ncam; ++c) {
    p.mask_off[c] = mask_off[c];
    p.sil_off[c] = sil_word_off[c];
    p.width[c] = cams[c].width;
    p.height[c] = cams[c].height;
    p.word_start[c + 1] = p.word_start[c] + (int64_t)sil_stride_words(cams[c].width) * cams[c].height;
  }
  bool wide = ((uintptr_t)masks_dev & 15) == 0;
  for (int c = 0; c < ncam; ++c)
    wide = wide && (cams[c].width % 32 == 0) && (mask_off[c] % 16 == 0);
  int64_t words = p.word_start[ncam];
  if (wide) {
    int64_t blocks = (words + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_k(pack_wide_kernel, (int)blocks, 256, 0, st, p);
  } else {
    int64_t blocks = (words * 32 + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    launch_k(pack_kernel, (int)blocks, 256, 0, st, p);
  }
  note_launches(1);
  return cuda_check("fvv_pack_silhouettes");
}

}  // namespace fvv

using namespace fvv;

extern "C" {

const char *fvv_last_error(void) { return g_err; }

int fvv_version(void) { return 1; }

long long fvv_launch_count(void) { return g_launches.load(); }

int fvv_host_mapped(const void *p) {
  cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

int fvv_copy_gather(const void *const *src, const int64_t *bytes, int64_t n, void *dst,
                    void *stream) {
  if (n < 0 || (n > 0 && (!src || !bytes || !dst))) {
    set_error("fvv_copy_gather: bad arguments");
    return FVV_E_ARG;
  }
  char *d = static_cast<char *>(dst);
  for (int64_t i = 0; i < n; ++i) {
    if (bytes[i] < 0 || (bytes[i] > 0 && !src[i])) {
      set_error("fvv_copy_gather: piece %lld has no data", (long long)i);
      return FVV_E_ARG;
    }
    if (bytes[i] &&
        cudaMemcpyAsync(d, src[i], (size_t)bytes[i], cudaMemcpyDefault,
                        (cudaStream_t)stream) != cudaSuccess)
      return cuda_check("fvv_copy_gather");
    d += bytes[i];
  }
  return FVV_OK;
}

int fvv_project(const fvv_camera *cam, const double *pts_dev, int64_t n, int use_distortion,
                int single_point, double *pixel_dev, double *z_dev, uint8_t *in_dev,
                void *stream) {
  if (!cam || n < 0) {
    set_error("fvv_project: bad arguments");
    return FVV_E_ARG;
  }
  if (n == 0) return FVV_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  launch_k(project_kernel, blocks, 256, 0, (cudaStream_t)stream, *cam, pts_dev, n, use_distortion != 0,
                                                           single_point != 0, pixel_dev, z_dev,
                                                           in_dev);
  note_launches(1);
  return cuda_check("fvv_project");
}

int fvv_pack_silhouettes(const fvv_camera *cams, int ncam, const uint8_t *masks_dev,
                         const int64_t *mask_off, uint32_t *sil_dev, const int64_t *sil_word_off,
                         void *stream) {
  return pack_silhouettes_bound(cams, ncam, masks_dev, nullptr, mask_off, sil_dev, sil_word_off,
                                (cudaStream_t)stream);
}

}  // extern "C"
