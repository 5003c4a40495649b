// Native frame-sequence runner: the engine under pipeline.run_sequence
// (video form of pipeline.py:115-220 run_frame + render.py:64-113
// render_view, pipelined over host threads as PAPER.md:561 describes).
//
// `lanes` C++ threads each own a CUDA stream pair (compute, readback) and two
// frame executors used alternately, so one frame's device->host copies
// overlap the lane's next frame. Frame n goes to lane n mod lanes; results
// come back in submission order. No Python runs per frame on the lanes, so
// the caller's interpreter lock never serialises them. Per frame a lane:
//   1. copies the silhouette masks host/device -> its slot's mask buffer
//      (the caller's pointers; pinned sources copy asynchronously) and,
//      when the colour frames are not device-accessible (pageable host
//      memory), uploads them; device or mapped pinned frames are sampled in
//      place by the colour pass (zero-copy);
//   2. runs fvv_frame_run (B-1 .. D-2 + the colour pass);
//   3. optionally packs the mesh + visibility bits into a device payload
//      (export mode: a frame-sharded rank ships those to rank 0 over NCCL);
//   4. queues one fvv_frame_readback into a pinned block from a pool and
//      records the result's completion event.
// Result records own their stats, ROI tables, pinned block and payload until
// fvv_seq_result_free, so the caller may keep bundles built on them.
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fvv_common.cuh"

namespace {

struct Block {
  void *p = nullptr;
  size_t cap = 0;
  bool busy = false;
  bool device = false;
};

// Pinned host (or device) blocks reused across frames; a block is busy from
// the lane's acquire until the caller frees the result that owns it.
class Pool {
 public:
  static constexpr size_t kMaxBlocks = 96;
  explicit Pool(bool device) : device_(device) {}
  ~Pool() {
    for (Block *b : blocks_) {
      if (b->p) device_ ? cudaFree(b->p) : cudaFreeHost(b->p);
      delete b;
    }
  }
  Block *acquire(size_t bytes) {
    std::lock_guard<std::mutex> g(m_);
    Block *best = nullptr;
    for (Block *b : blocks_)
      if (!b->busy && b->cap >= bytes && (!best || b->cap < best->cap)) best = b;
    if (!best) {
      // add a block while the pool is small: re-sizing a free one frees it
      // first, and cudaFree / cudaFreeHost wait for the whole device (every
      // lane stalls); past kMaxBlocks a free block is re-sized
      if (blocks_.size() >= kMaxBlocks)
        for (Block *b : blocks_)
          if (!b->busy) {
            best = b;
            break;
          }
      if (!best) {
        best = new Block();
        best->device = device_;
        blocks_.push_back(best);
      }
      if (best->p) device_ ? cudaFree(best->p) : cudaFreeHost(best->p);
      best->p = nullptr;
      best->cap = 0;
      // generous headroom: a block re-pinned later (frames vary in size)
      // costs a device-wide synchronisation in cudaFreeHost and ms of pinning
      const size_t want = bytes + bytes / 2 + 4096;
      const cudaError_t e = device_ ? cudaMalloc(&best->p, want) : cudaHostAlloc(&best->p, want, 0);
      if (e != cudaSuccess) {
        cudaGetLastError();
        best->p = nullptr;
        return nullptr;
      }
      best->cap = want;
    }
    best->busy = true;
    return best;
  }
  void release(Block *b) {
    if (!b) return;
    std::lock_guard<std::mutex> g(m_);
    b->busy = false;
  }

 private:
  bool device_;
  std::mutex m_;
  std::vector<Block *> blocks_;
};

struct Input {
  int64_t id = 0;
  std::vector<const void *> mask_src;
  std::vector<int64_t> mask_bytes;
  std::vector<const void *> frame_src;  // per camera (colour pass), may be empty
  bool stop = false;
};

}  // namespace

struct fvv_seq_result {
  int64_t id = 0;
  int status = 0, stage = 0;
  std::string err;
  fvv_frame_stats stats{};
  int64_t nv = 0, nt = 0, vis_stride = 0, n_rois = 0;
  std::vector<int64_t> comp, info;
  std::vector<double> boxes;
  std::vector<fvv_grid> grids;
  int64_t layout[16] = {};
  Block *block = nullptr, *payload = nullptr;
  int64_t payload_bytes = 0;
  cudaEvent_t done = nullptr;
  struct fvv_seq *owner = nullptr;
};

struct Lane {
  std::thread th;
  cudaStream_t compute = nullptr, readback = nullptr, copy = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr};  // masks of the slot's next frame uploaded
  int64_t staged_id[2] = {-1, -1};             // frame whose masks the slot buffer holds
  fvv_frame *ex[2] = {nullptr, nullptr};
  cudaEvent_t slot_free[2] = {nullptr, nullptr};
  bool slot_used[2] = {false, false};
  void *masks[2] = {nullptr, nullptr};
  size_t masks_cap[2] = {0, 0};
  void *frames[2] = {nullptr, nullptr};
  size_t frames_cap[2] = {0, 0};
  std::deque<Input> in;
  std::deque<fvv_seq_result *> out;
  std::mutex m;
  std::condition_variable cv_in, cv_out;
  int64_t n_run = 0;
  // a frame begun on ex[pend_slot] (its graph replay running) whose results
  // are read back after the lane has launched its next frame
  fvv_seq_result *pend = nullptr;
  int pend_slot = 0;
};

struct fvv_seq {
  int device = 0, ncam = 0, lanes = 0;
  fvv_seq_config cfg{};
  std::vector<fvv_camera> cams;
  std::vector<int64_t> frame_bytes;  // H*W*3 per camera
  int64_t mask_total = 0;
  Lane *lane = nullptr;
  Pool host_pool{false}, dev_pool{true};
  std::mutex ev_m;
  std::vector<cudaEvent_t> free_events;
  int64_t n_in = 0, n_out = 0;
};

namespace {

// FVV_SEQ_ASYNC=0: every frame completes before the lane takes the next
bool async_enabled() {
  static const bool on = [] {
    const char *e = getenv("FVV_SEQ_ASYNC");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaEvent_t take_event(fvv_seq *s) {
  std::lock_guard<std::mutex> g(s->ev_m);
  if (!s->free_events.empty()) {
    cudaEvent_t e = s->free_events.back();
    s->free_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

void give_event(fvv_seq *s, cudaEvent_t e) {
  if (!e) return;
  std::lock_guard<std::mutex> g(s->ev_m);
  s->free_events.push_back(e);
}

int ensure_dev(void *&p, size_t &cap, size_t bytes) {
  if (bytes <= cap && p) return FVV_OK;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  const size_t want = bytes + bytes / 8 + 256;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    fvv::set_error("fvv_seq: cudaMalloc(%zu) failed", want);
    return FVV_E_CUDA;
  }
  cap = want;
  return FVV_OK;
}

// device-accessible at the same address: device memory or mapped pinned host
bool accessible(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return true;
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

// device memory proper (masks are read many times by the packing kernel:
// host memory, even mapped, is uploaded instead of read in place)
bool on_device(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// sharding.py payload_layout: verts, tris, visibility bits, 256-aligned
int64_t payload_layout(int64_t nv, int64_t nt, int64_t ncam, int64_t stride, int64_t off[3],
                       int64_t sz[3]) {
  sz[0] = 24 * nv;
  sz[1] = 12 * nt;
  sz[2] = 4 * ncam * stride;
  int64_t o = 0;
  for (int i = 0; i < 3; ++i) {
    off[i] = o;
    o += (sz[i] + 255) & ~255ll;
  }
  return o;
}

// Queue the upload of a frame's silhouette masks into a slot's buffer on the
// lane's copy stream (the lane uploads its next frame while this one runs).
// Returns the masks' device pointer, or nullptr with R's error set.
const uint8_t *stage_masks(fvv_seq *s, Lane &L, int slot, const Input &in, fvv_seq_result *R) {
  if (in.mask_src.size() == 1 && in.mask_bytes[0] == s->mask_total && on_device(in.mask_src[0]))
    return (const uint8_t *)in.mask_src[0];  // device masks in rig order: used in place
  int64_t tot = 0;
  for (int64_t b : in.mask_bytes) tot += b;
  if (tot != s->mask_total) {
    if (R) {
      R->status = FVV_E_ARG;
      R->stage = 1;
      R->err = "silhouettes do not match the rig's image sizes";
    }
    return nullptr;
  }
  if (L.staged_id[slot] == in.id) return (const uint8_t *)L.masks[slot];
  if (ensure_dev(L.masks[slot], L.masks_cap[slot], (size_t)s->mask_total)) {
    if (R) {
      R->status = FVV_E_CUDA;
      R->stage = 1;
      R->err = fvv_last_error();
    }
    return nullptr;
  }
  char *d = (char *)L.masks[slot];
  for (size_t i = 0; i < in.mask_src.size(); ++i) {
    if (in.mask_bytes[i])
      cudaMemcpyAsync(d, in.mask_src[i], (size_t)in.mask_bytes[i], cudaMemcpyDefault, L.copy);
    d += in.mask_bytes[i];
  }
  cudaEventRecord(L.copied[slot], L.copy);
  L.staged_id[slot] = in.id;
  return (const uint8_t *)L.masks[slot];
}

// After a lane's frame has completed on ex[slot]: ROI tables, the export
// payload, and its readback queued on the readback stream behind `ran`.
void finish_one(fvv_seq *s, Lane &L, int slot, fvv_seq_result *R, cudaEvent_t ran) {
  fvv_frame *ex = L.ex[slot];
  fvv_frame_outputs o;
  fvv_frame_get_outputs(ex, &o);
  R->nv = o.nv;
  R->nt = o.nt;
  R->vis_stride = o.vis_stride;
  R->n_rois = o.n_rois;
  const size_t nr = (size_t)o.n_rois;
  R->comp.resize(nr);
  R->boxes.resize(6 * nr);
  R->grids.resize(nr);
  R->info.resize(8 * nr);
  fvv_frame_get_rois(ex, R->comp.data(), R->boxes.data(), R->grids.data(), R->info.data());
  // 3. export payload (device) for a frame-sharded rank, behind the frame
  if (s->cfg.export_payload) {
    int64_t off[3], sz[3];
    const int64_t tot = payload_layout(o.nv, o.nt, s->ncam, o.vis_stride, off, sz);
    R->payload = s->dev_pool.acquire((size_t)(tot > 0 ? tot : 1));
    if (!R->payload) {
      R->status = FVV_E_CUDA;
      R->stage = 8;
      R->err = "fvv_seq: payload allocation failed";
      return;
    }
    cudaStreamWaitEvent(L.readback, ran, 0);
    const void *src[3] = {o.verts, o.tris, o.vis};
    for (int i = 0; i < 3; ++i)
      if (sz[i]) cudaMemcpyAsync((char *)R->payload->p + off[i], src[i], (size_t)sz[i],
                                 cudaMemcpyDeviceToDevice, L.readback);
    R->payload_bytes = tot;
  }
  // 4. readback into a pinned block
  const int flags = s->cfg.readback_flags | (s->cfg.export_payload ? 4 : 0);
  const int64_t total = fvv_frame_readback_layout(ex, flags, R->layout);
  R->block = s->host_pool.acquire((size_t)(total > 0 ? total : 1));
  if (!R->block) {
    R->status = FVV_E_CUDA;
    R->stage = 8;
    R->err = "fvv_seq: pinned block allocation failed";
    return;
  }
  cudaStreamWaitEvent(L.readback, ran, 0);
  fvv_frame_readback(ex, R->block->p, flags, L.readback);
  R->done = take_event(s);
  cudaEventRecord(R->done, L.readback);
  cudaEventRecord(L.slot_free[slot], L.readback);
  L.slot_used[slot] = true;
  const int e = fvv::cuda_check("fvv_seq lane");
  if (e != FVV_OK) {
    R->status = e;
    R->stage = 8;
    R->err = fvv_last_error();
  }
}

void push_result(Lane &L, fvv_seq_result *R) {
  {
    std::lock_guard<std::mutex> g(L.m);
    L.out.push_back(R);
  }
  L.cv_out.notify_all();
}

// The lane's begun frame: wait for it (not for the frame launched after
// it), read it back, hand the result out.
void end_pending(fvv_seq *s, Lane &L) {
  fvv_seq_result *R = L.pend;
  if (!R) return;
  L.pend = nullptr;
  const int slot = L.pend_slot;
  int stage = 0;
  const int rc = fvv::frame_end(L.ex[slot], &R->stats, &stage);
  if (rc != FVV_OK) {
    R->status = rc;
    R->stage = stage;
    R->err = fvv_last_error();
    cudaGetLastError();
  } else {
    // (a frame redone host-planned ran after the lane's next frame on the
    // compute stream: read it back behind everything queued there so far)
    cudaEvent_t ran = fvv_frame_last_mode(L.ex[slot]) == 0
                          ? nullptr
                          : fvv::frame_launched_event(L.ex[slot]);
    cudaEvent_t own = nullptr;
    if (!ran) {
      own = take_event(s);
      cudaEventRecord(own, L.compute);
      ran = own;
    }
    finish_one(s, L, slot, R, ran);
    if (own) give_event(s, own);
  }
  push_result(L, R);
}

void run_one(fvv_seq *s, Lane &L, Input &in, fvv_seq_result *R, const Input *next_in) {
  const int slot = (int)(L.n_run++ & 1);
  fvv_frame *ex = L.ex[slot];
  cudaStream_t st = L.compute;
  if (L.slot_used[slot]) cudaStreamWaitEvent(st, L.slot_free[slot], 0);  // readback drained
  // 1. inputs (normally uploaded while the lane's previous frame ran)
  const uint8_t *masks = stage_masks(s, L, slot, in, R);
  if (!masks) {
    end_pending(s, L);
    push_result(L, R);
    return;
  }
  if (L.staged_id[slot] == in.id) cudaStreamWaitEvent(st, L.copied[slot], 0);
  L.staged_id[slot] = -1;  // consumed: the buffer is this frame's until it has run
  const bool colour = s->cfg.has_virtual && !in.frame_src.empty();
  const uint8_t *fbase = nullptr;
  int64_t foff[FVV_MAX_CAMS] = {};
  if (colour) {
    bool direct = true;
    for (const void *p : in.frame_src) direct = direct && p && accessible(p);
    if (direct) {  // zero-copy: the colour pass samples them in place
      const char *lo = (const char *)in.frame_src[0];
      for (const void *p : in.frame_src) lo = (const char *)p < lo ? (const char *)p : lo;
      fbase = (const uint8_t *)lo;
      for (int c = 0; c < s->ncam; ++c) foff[c] = (const char *)in.frame_src[c] - lo;
    } else {
      int64_t tot = 0;
      for (int c = 0; c < s->ncam; ++c) tot += s->frame_bytes[c];
      if (ensure_dev(L.frames[slot], L.frames_cap[slot], (size_t)tot)) {
        R->status = FVV_E_CUDA;
        R->stage = 7;
        R->err = fvv_last_error();
        end_pending(s, L);
        push_result(L, R);
        return;
      }
      int64_t o = 0;
      for (int c = 0; c < s->ncam; ++c) {
        cudaMemcpyAsync((char *)L.frames[slot] + o, in.frame_src[c], (size_t)s->frame_bytes[c],
                        cudaMemcpyDefault, st);
        foff[c] = o;
        o += s->frame_bytes[c];
      }
      fbase = (const uint8_t *)L.frames[slot];
    }
  }
  // 2. the frame: a graph replay is launched and left running while the
  // lane finishes its previous frame; any other frame completes here
  int stage = 0;
  bool async = false;
  const int rc = fvv::frame_begin(ex, masks, colour ? &s->cfg.virt : nullptr, s->cfg.rank_pos,
                                  fbase, foff, s->cfg.fallback, st, &R->stats, &stage, &async);
  end_pending(s, L);  // (in order: the previous frame's result first)
  if (next_in && !next_in->stop) {
    // the other slot's previous frame has completed (end_pending / a
    // synchronous run), so its mask buffer can take the next frame's upload
    stage_masks(s, L, slot ^ 1, *next_in, nullptr);
  }
  if (rc != FVV_OK) {
    R->status = rc;
    R->stage = stage;
    R->err = fvv_last_error();
    cudaStreamSynchronize(st);
    cudaGetLastError();
    push_result(L, R);
    return;
  }
  if (async && async_enabled()) {
    L.pend = R;
    L.pend_slot = slot;
    return;
  }
  if (async) {  // (FVV_SEQ_ASYNC=0: complete it now)
    L.pend = R;
    L.pend_slot = slot;
    end_pending(s, L);
    return;
  }
  cudaEvent_t ran = take_event(s);
  cudaEventRecord(ran, st);
  finish_one(s, L, slot, R, ran);
  give_event(s, ran);  // (an event may be re-recorded once its waits are queued)
  push_result(L, R);
}

void lane_main(fvv_seq *s, int k) {
  Lane &L = s->lane[k];
  cudaSetDevice(s->device);
  while (true) {
    Input in;
    {
      std::unique_lock<std::mutex> g(L.m);
      if (L.in.empty() && L.pend) {  // nothing queued: finish the running frame first
        g.unlock();
        end_pending(s, L);
        g.lock();
      }
      L.cv_in.wait(g, [&] { return !L.in.empty(); });
      in = std::move(L.in.front());
      L.in.pop_front();
    }
    L.cv_in.notify_all();  // room for the next submit
    if (in.stop) {
      end_pending(s, L);
      return;
    }
    fvv_seq_result *R = new fvv_seq_result();
    R->id = in.id;
    R->owner = s;
    Input next_copy;
    bool have_next = false;
    {
      std::lock_guard<std::mutex> g(L.m);
      if (!L.in.empty()) {
        next_copy = L.in.front();  // (pointer lists only: the caller owns the data)
        have_next = true;
      }
    }
    run_one(s, L, in, R, have_next ? &next_copy : nullptr);  // (it hands results out)
  }
}

}  // namespace

extern "C" {

fvv_seq *fvv_seq_create(const fvv_camera *cams, int ncam, const fvv_frame_config *fcfg,
                        const fvv_seq_config *cfg) {
  if (!cams || !fcfg || !cfg || ncam < 1 || ncam > FVV_MAX_CAMS || cfg->lanes < 1 ||
      cfg->lanes > 64) {
    fvv::set_error("fvv_seq_create: bad arguments");
    return nullptr;
  }
  fvv_seq *s = new fvv_seq();
  cudaGetDevice(&s->device);
  s->ncam = ncam;
  s->lanes = cfg->lanes;
  s->cfg = *cfg;
  s->cams.assign(cams, cams + ncam);
  for (int c = 0; c < ncam; ++c) {
    s->mask_total += (int64_t)cams[c].width * cams[c].height;
    s->frame_bytes.push_back(3 * (int64_t)cams[c].width * cams[c].height);
  }
  s->lane = new Lane[s->lanes];
  for (int k = 0; k < s->lanes; ++k) {
    Lane &L = s->lane[k];
    cudaStreamCreateWithFlags(&L.compute, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&L.readback, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&L.copy, cudaStreamNonBlocking);
    for (int j = 0; j < 2; ++j) {
      cudaEventCreateWithFlags(&L.copied[j], cudaEventDisableTiming);
      L.ex[j] = fvv_frame_create(cams, ncam, fcfg);
      cudaEventCreateWithFlags(&L.slot_free[j], cudaEventDisableTiming);
      if (!L.ex[j]) {
        const std::string msg = fvv_last_error();
        fvv_seq_destroy(s);
        fvv::set_error("%s", msg.c_str());
        return nullptr;
      }
    }
  }
  for (int k = 0; k < s->lanes; ++k) s->lane[k].th = std::thread(lane_main, s, k);
  return s;
}

// Queue frame `id`: ncam_masks pointers (one contiguous rig-order buffer, or
// one per camera) with their byte sizes; per-camera colour frames (or NULL).
// The caller keeps every input alive until the frame's result is returned.
// Blocks while the lane already holds two queued frames.
int fvv_seq_submit(fvv_seq *s, int64_t id, const void *const *mask_src, const int64_t *mask_bytes,
                   int nmask, const void *const *frame_src) {
  if (!s || !mask_src || !mask_bytes || nmask < 1) {
    fvv::set_error("fvv_seq_submit: bad arguments");
    return FVV_E_ARG;
  }
  Input in;
  in.id = id;
  in.mask_src.assign(mask_src, mask_src + nmask);
  in.mask_bytes.assign(mask_bytes, mask_bytes + nmask);
  if (frame_src) in.frame_src.assign(frame_src, frame_src + s->ncam);
  Lane &L = s->lane[s->n_in % s->lanes];
  {
    std::unique_lock<std::mutex> g(L.m);
    L.cv_in.wait(g, [&] { return L.in.size() < 2; });
    L.in.push_back(std::move(in));
  }
  L.cv_in.notify_all();
  ++s->n_in;
  return FVV_OK;
}

// Next result in submission order: 1 = *out set, 0 = nothing ready (wait = 0)
// or nothing pending. The result's readback has completed when returned.
int fvv_seq_next(fvv_seq *s, int wait, fvv_seq_result **out) {
  *out = nullptr;
  if (s->n_out >= s->n_in) return 0;
  Lane &L = s->lane[s->n_out % s->lanes];
  fvv_seq_result *R = nullptr;
  {
    std::unique_lock<std::mutex> g(L.m);
    if (!wait && L.out.empty()) return 0;
    L.cv_out.wait(g, [&] { return !L.out.empty(); });
    R = L.out.front();
    if (!wait && R->done && cudaEventQuery(R->done) == cudaErrorNotReady) {
      cudaGetLastError();
      return 0;
    }
    L.out.pop_front();
  }
  if (R->done) cudaEventSynchronize(R->done);
  ++s->n_out;
  *out = R;
  return 1;
}

int fvv_seq_result_get(const fvv_seq_result *R, fvv_seq_result_info *info) {
  memset(info, 0, sizeof(*info));
  info->id = R->id;
  info->status = R->status;
  info->stage = R->stage;
  info->err = R->err.c_str();
  info->stats = R->stats;
  info->nv = R->nv;
  info->nt = R->nt;
  info->vis_stride = R->vis_stride;
  info->n_rois = R->n_rois;
  info->component_ids = R->comp.data();
  info->boxes = R->boxes.data();
  info->grids = R->grids.data();
  info->roi_info = R->info.data();
  memcpy(info->layout, R->layout, sizeof(R->layout));
  info->host = R->block ? R->block->p : nullptr;
  info->payload_dev = R->payload ? R->payload->p : nullptr;
  info->payload_bytes = R->payload_bytes;
  return FVV_OK;
}

void fvv_seq_result_free(fvv_seq_result *R) {
  if (!R) return;
  fvv_seq *s = R->owner;
  s->host_pool.release(R->block);
  s->dev_pool.release(R->payload);
  give_event(s, R->done);
  delete R;
}

void fvv_seq_destroy(fvv_seq *s) {
  if (!s) return;
  for (int k = 0; k < s->lanes; ++k) {
    Lane &L = s->lane[k];
    if (L.th.joinable()) {
      Input stop;
      stop.stop = true;
      {
        std::lock_guard<std::mutex> g(L.m);
        L.in.push_back(std::move(stop));
      }
      L.cv_in.notify_all();
      L.th.join();
    }
  }
  for (int k = 0; k < s->lanes; ++k) {
    Lane &L = s->lane[k];
    if (L.compute) cudaStreamSynchronize(L.compute);
    if (L.readback) cudaStreamSynchronize(L.readback);
    if (L.copy) cudaStreamSynchronize(L.copy);
    for (fvv_seq_result *R : L.out) fvv_seq_result_free(R);
    for (int j = 0; j < 2; ++j) {
      fvv_frame_destroy(L.ex[j]);
      if (L.slot_free[j]) cudaEventDestroy(L.slot_free[j]);
      if (L.copied[j]) cudaEventDestroy(L.copied[j]);
      if (L.masks[j]) cudaFree(L.masks[j]);
      if (L.frames[j]) cudaFree(L.frames[j]);
    }
    if (L.compute) cudaStreamDestroy(L.compute);
    if (L.readback) cudaStreamDestroy(L.readback);
    if (L.copy) cudaStreamDestroy(L.copy);
  }
  for (cudaEvent_t e : s->free_events) cudaEventDestroy(e);
  delete[] s->lane;
  delete s;
}

}  // extern "C"

extern "C" int fvv_abi_sizes(int64_t *out, int n) {
  const int64_t s[8] = {(int64_t)sizeof(fvv_camera),        (int64_t)sizeof(fvv_grid),
                        (int64_t)sizeof(fvv_component),     (int64_t)sizeof(fvv_frame_config),
                        (int64_t)sizeof(fvv_frame_stats),   (int64_t)sizeof(fvv_frame_outputs),
                        (int64_t)sizeof(fvv_seq_config),    (int64_t)sizeof(fvv_seq_result_info)};
  for (int i = 0; i < n && i < 8; ++i) out[i] = s[i];
  return 8;
}
