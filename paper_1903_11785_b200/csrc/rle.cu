// Run-length dump of an occupancy grid (voxels.py:100-162 save_grid /
// _rle_encode, pkg/docs/formats.md): the run boundaries are the bit
// transitions of the occupancy field, found per 32-bit word (bit b differs
// from the bit before it, bit -1 counting as OFF) and compacted in order
// with the single-pass scan. The host turns positions into run lengths.
#include "scan.cuh"

namespace fvv {

struct RleTransitions {
  const uint32_t *occ;
  int64_t words, nvox;
  int64_t *pos;
  __device__ uint32_t word(int64_t w) const {
    uint32_t v = __ldg(occ + w);
    if (w == words - 1 && (nvox & 31)) v &= (1u << (nvox & 31)) - 1u;
    return v;
  }
  __device__ uint32_t tmask(int64_t w) const {
    const uint32_t v = word(w);
    const uint32_t carry = w > 0 ? (word(w - 1) >> 31) : 0u;
    uint32_t t = v ^ ((v << 1) | carry);
    if (w == words - 1 && (nvox & 31)) t &= (1u << (nvox & 31)) - 1u;  // positions < nvox
    return t;
  }
  typedef uint32_t Item;
  __device__ uint32_t load(int64_t w) const { return tmask(w); }
  __device__ int64_t value(uint32_t t) const { return __popc(t); }
  __device__ void emit(int64_t w, int64_t prefix, uint32_t t) const {
    while (t) {
      const int b = __ffs(t) - 1;
      t &= t - 1;
      pos[prefix++] = w * 32 + b;
    }
  }
};

}  // namespace fvv

using namespace fvv;

extern "C" {

size_t fvv_rle_workspace_bytes(int64_t nvox) {
  return onepass_bytes<int64_t>((nvox + 31) / 32 + 1);
}

int fvv_rle_transitions(const uint32_t *occ_dev, int64_t nvox, int64_t *pos_dev,
                        int64_t *count_dev, void *ws_dev, size_t ws_bytes, void *stream) {
  if (nvox < 0 || (nvox > 0 && (!occ_dev || !pos_dev || !count_dev))) {
    set_error("fvv_rle_transitions: bad arguments");
    return FVV_E_ARG;
  }
  if (ws_bytes < fvv_rle_workspace_bytes(nvox)) {
    set_error("fvv_rle_transitions: workspace %zu < %zu bytes", ws_bytes,
              fvv_rle_workspace_bytes(nvox));
    return FVV_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t words = (nvox + 31) / 32;
  if (words == 0) {
    fill_async(count_dev, 0, sizeof(int64_t), st);
    return cuda_check("fvv_rle_transitions");
  }
  RleTransitions f{occ_dev, words, nvox, pos_dev};
  onepass_scan(f, nullptr, words, words, ws_dev, count_dev, st);
  return cuda_check("fvv_rle_transitions");
}

}  // extern "C"
