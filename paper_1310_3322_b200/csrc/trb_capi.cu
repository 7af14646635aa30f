// trb_capi.cu — the extern "C" boundary (include/trb.h).  Converts
// trb::Error exceptions into status codes + thread-local messages, owns the
// per-handle device buffers and CUDA streams.  No computation happens on
// the host: every result comes from the sm_100a kernels.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "trb_engine.cuh"
#include "trb_exact.cuh"
#include "trb_track.cuh"

using trb::DevBuf;
using trb::Error;
using trb::PinnedBuf;

namespace {
thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return TRB_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return TRB_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TRB_INVALID_ARGUMENT;
  }
}

void need(bool cond, const char* msg, trb_status code = TRB_INVALID_ARGUMENT) {
  if (!cond) throw Error(code, msg);
}

// Binds the calling thread to `device`, failing loudly when no sm_100
// device exists (there is no CPU fallback).
void use_device(int device) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw Error(TRB_CUDA_ERROR, std::string("no CUDA device available: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) throw Error(TRB_INVALID_ARGUMENT, "device index out of range");
  TRB_CUDA(cudaSetDevice(device));
}

trb_motion_config default_motion() { return trb_motion_config{TRB_BG_MEAN, 91, 25, 32, 0, TRB_MORPH_NONE}; }
}  // namespace

// ---------------------------------------------------------------- handles
struct trb_motion {
  int device;
  int w, h;
  std::unique_ptr<trb::MotionState> m;
  DevBuf frame, mask, tmp, ptrs;
  cudaStream_t st = nullptr;
  ~trb_motion() {
    if (st) cudaStreamDestroy(st);
  }
};

struct trb_tracker {
  int device;
  trb_tracker_config cfg;
  std::unique_ptr<trb::TrackerState> t;
  DevBuf frame, ptrs, blobs, nblobs;
  size_t frame_bytes = 0;
  int64_t blob_cap = 0;
  cudaStream_t st = nullptr;
  ~trb_tracker() {
    if (st) cudaStreamDestroy(st);
  }
};

struct trb_streams {
  int device;
  std::unique_ptr<trb::Streams> s;
};

extern "C" {

const char* trb_last_error(void) { return g_last_error.c_str(); }
const char* trb_version(void) { return "trb 0.1 (sm_100a)"; }

int trb_device_count(int* n) {
  return guard([&] {
    need(n != nullptr, "null output");
    *n = 0;
    const cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) *n = 0;
  });
}

void trb_default_motion_config(trb_motion_config* c) { *c = default_motion(); }
void trb_default_seg_config(trb_seg_config* c) { *c = trb_seg_config{4, TRB_CONN_EIGHT, 4}; }
void trb_default_tracker_config(trb_tracker_config* c) { *c = trb_tracker_config{16, 20, 0.5, 20, 0, 0}; }

int trb_motion_config_validate(const trb_motion_config* c) {
  return guard([&] { trb::validate_motion(*c); });
}
int trb_seg_config_validate(const trb_seg_config* c) {
  return guard([&] { trb::validate_seg(*c, 0, 0); });
}
int trb_tracker_config_validate(const trb_tracker_config* c) {
  return guard([&] { trb::validate_tracker(*c); });
}

// ------------------------------------------------------------- motion
int trb_motion_create(const trb_motion_config* cfg, int width, int height, int device, trb_motion** out) {
  return guard([&] {
    need(cfg && out, "null argument");
    *out = nullptr;
    trb::validate_motion(*cfg);
    if (width < 1 || height < 1) throw Error(TRB_INVALID_ARGUMENT, "motion detector needs positive frame dimensions");
    use_device(device);
    auto m = std::make_unique<trb_motion>();
    m->device = device;
    m->w = width;
    m->h = height;
    m->m = std::make_unique<trb::MotionState>(*cfg, 1, width, height, 1);
    const size_t px = static_cast<size_t>(width) * height;
    m->frame.alloc(px, false);
    m->mask.alloc(px);
    if (cfg->morph != TRB_MORPH_NONE) m->tmp.alloc(2 * px);  // raw mask + 2-pass scratch
    m->ptrs.alloc(sizeof(void*), false);
    const void* fp = m->frame.p;
    TRB_CUDA(cudaMemcpy(m->ptrs.p, &fp, sizeof(void*), cudaMemcpyHostToDevice));
    TRB_CUDA(cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking));
    *out = m.release();
  });
}

int trb_motion_destroy(trb_motion* m) {
  return guard([&] {
    if (m) {
      cudaSetDevice(m->device);
      delete m;
    }
  });
}

int trb_motion_push(trb_motion* m, const uint8_t* gray, int width, int height, int channels, int64_t frame_index,
                    uint8_t* mask_out, int* has_mask) {
  return guard([&] {
    need(m && gray && has_mask, "null argument");
    // MotionDetector::push checks, motion.hpp:165-167
    if (channels != 1) throw Error(TRB_INVALID_ARGUMENT, "motion detector expects grayscale frames");
    if (width != m->w || height != m->h)
      throw Error(TRB_INVALID_ARGUMENT,
                  "frame " + std::to_string(frame_index) + " dimensions do not match detector");
    TRB_CUDA(cudaSetDevice(m->device));
    const size_t px = static_cast<size_t>(width) * height;
    TRB_CUDA(cudaMemcpyAsync(m->frame.p, gray, px, cudaMemcpyHostToDevice, m->st));
    int launches = 0;
    const bool emitted = m->m->push(m->ptrs.as<const uint8_t* const>(), m->mask.as<uint8_t>(), m->tmp.as<uint8_t>(),
                                    m->st, &launches);
    *has_mask = emitted ? 1 : 0;
    if (emitted && mask_out) TRB_CUDA(cudaMemcpyAsync(mask_out, m->mask.p, px, cudaMemcpyDeviceToHost, m->st));
    TRB_CUDA(cudaStreamSynchronize(m->st));
  });
}

int trb_motion_background(trb_motion* m, uint8_t* out) {
  return guard([&] {
    need(m && out, "null argument");
    TRB_CUDA(cudaSetDevice(m->device));
    const size_t px = static_cast<size_t>(m->w) * m->h;
    DevBuf bg;
    bg.alloc(px, false);
    m->m->background(bg.as<uint8_t>(), m->st);
    TRB_CUDA(cudaMemcpyAsync(out, bg.p, px, cudaMemcpyDeviceToHost, m->st));
    TRB_CUDA(cudaStreamSynchronize(m->st));
  });
}

int trb_motion_frames_seen(const trb_motion* m, int* n) {
  return guard([&] {
    need(m && n, "null argument");
    *n = m->m->frames_seen();
  });
}

// ------------------------------------------------------------ labelling
namespace {
struct LabelWs {
  std::unique_ptr<trb::CclState> ccl;
  DevBuf mask;
  cudaStream_t st = nullptr;
  ~LabelWs() {
    if (st) cudaStreamDestroy(st);
  }
};

LabelWs& label_ws(int device, int w, int h, const trb_seg_config& cfg) {
  thread_local std::map<std::tuple<int, int, int, int, int>, std::unique_ptr<LabelWs>> cache;
  auto key = std::make_tuple(device, w, h, cfg.connectivity, cfg.min_area);
  auto& slot = cache[key];
  if (!slot) {
    if (cache.size() > 8) {  // keep the cache small
      for (auto it = cache.begin(); it != cache.end();)
        if (it->first != key) it = cache.erase(it);
        else ++it;
    }
    auto ws = std::make_unique<LabelWs>();
    trb_seg_config c = cfg;
    c.n_blocks = 1;
    ws->ccl = std::make_unique<trb::CclState>(1, w, h, c);
    ws->mask.alloc(static_cast<size_t>(w) * h, false);
    TRB_CUDA(cudaStreamCreateWithFlags(&ws->st, cudaStreamNonBlocking));
    slot = std::move(ws);
  }
  return *cache[key];
}

__global__ void mask_normalize_kernel(uint8_t* m, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) m[i] = m[i] != 0;
}

__global__ void iota_kernel(int64_t* v, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

struct NonZero {
  __host__ __device__ bool operator()(const int32_t& x) const { return x != 0; }
};

// Blob::pixels: stable sort of the foreground pixel indices (already in
// raster order) by label, on the device.
void pixel_lists(const int32_t* labels, int64_t px, int64_t n_fg, int64_t* out_host, cudaStream_t st) {
  DevBuf idx, keys, sel_idx, sel_keys, sorted_idx, sorted_keys, nsel, tmp;
  idx.alloc(sizeof(int64_t) * px, false);
  sel_idx.alloc(sizeof(int64_t) * (n_fg + 1), false);
  sel_keys.alloc(sizeof(int32_t) * (n_fg + 1), false);
  sorted_idx.alloc(sizeof(int64_t) * (n_fg + 1), false);
  sorted_keys.alloc(sizeof(int32_t) * (n_fg + 1), false);
  nsel.alloc(sizeof(int64_t), false);
  iota_kernel<<<static_cast<unsigned>(trb::ceil_div64(px, 256)), 256, 0, st>>>(idx.as<int64_t>(), px);
  size_t tb1 = 0, tb2 = 0, tb3 = 0;
  cub::DeviceSelect::Flagged(nullptr, tb1, idx.as<int64_t>(), labels, sel_idx.as<int64_t>(), nsel.as<int64_t>(), px,
                             st);
  cub::DeviceSelect::If(nullptr, tb2, labels, sel_keys.as<int32_t>(), nsel.as<int64_t>(), px, NonZero(), st);
  cub::DeviceRadixSort::SortPairs(nullptr, tb3, sel_keys.as<int32_t>(), sorted_keys.as<int32_t>(),
                                  sel_idx.as<int64_t>(), sorted_idx.as<int64_t>(), n_fg, 0, 32, st);
  tmp.alloc(std::max(tb1, std::max(tb2, tb3)), false);
  size_t t1 = tmp.n;
  cub::DeviceSelect::Flagged(tmp.p, t1, idx.as<int64_t>(), labels, sel_idx.as<int64_t>(), nsel.as<int64_t>(), px, st);
  size_t t2 = tmp.n;
  cub::DeviceSelect::If(tmp.p, t2, labels, sel_keys.as<int32_t>(), nsel.as<int64_t>(), px, NonZero(), st);
  size_t t3 = tmp.n;
  cub::DeviceRadixSort::SortPairs(tmp.p, t3, sel_keys.as<int32_t>(), sorted_keys.as<int32_t>(), sel_idx.as<int64_t>(),
                                  sorted_idx.as<int64_t>(), n_fg, 0, 32, st);
  TRB_LAUNCH_CHECK("pixel_lists");
  TRB_CUDA(cudaMemcpyAsync(out_host, sorted_idx.p, sizeof(int64_t) * n_fg, cudaMemcpyDeviceToHost, st));
}
}  // namespace

int trb_label(const uint8_t* mask, int width, int height, const trb_seg_config* cfg, int device, int32_t* labels_out,
              trb_blob* blobs_out, int blob_cap, int* n_blobs, int64_t* pixels_out, int64_t pixels_cap) {
  return guard([&] {
    need(mask && cfg && n_blobs, "null argument");
    need(width >= 1 && height >= 1, "mask dimensions must be >= 1");
    trb::validate_seg(*cfg, width, height);
    use_device(device);
    LabelWs& ws = label_ws(device, width, height, *cfg);
    const int64_t px = static_cast<int64_t>(width) * height;
    TRB_CUDA(cudaMemcpyAsync(ws.mask.p, mask, px, cudaMemcpyHostToDevice, ws.st));
    mask_normalize_kernel<<<static_cast<unsigned>(trb::ceil_div64(px, 256)), 256, 0, ws.st>>>(ws.mask.as<uint8_t>(),
                                                                                              px);
    int launches = 0;
    ws.ccl->run(ws.mask.as<uint8_t>(), ws.st, &launches);
    int32_t nb = 0;
    TRB_CUDA(cudaMemcpyAsync(&nb, ws.ccl->nblobs(), sizeof(int32_t), cudaMemcpyDeviceToHost, ws.st));
    if (labels_out)
      TRB_CUDA(cudaMemcpyAsync(labels_out, ws.ccl->labels(), sizeof(int32_t) * px, cudaMemcpyDeviceToHost, ws.st));
    TRB_CUDA(cudaStreamSynchronize(ws.st));
    *n_blobs = nb;
    if (blobs_out && nb > 0)
      TRB_CUDA(cudaMemcpyAsync(blobs_out, ws.ccl->blobs(), sizeof(trb_blob) * std::min(nb, blob_cap),
                               cudaMemcpyDeviceToHost, ws.st));
    if (pixels_out) {
      // foreground pixels that survived min_area = sum of blob areas
      std::vector<trb_blob> bl(nb);
      if (nb > 0)
        TRB_CUDA(cudaMemcpyAsync(bl.data(), ws.ccl->blobs(), sizeof(trb_blob) * nb, cudaMemcpyDeviceToHost, ws.st));
      TRB_CUDA(cudaStreamSynchronize(ws.st));
      int64_t n_fg = 0;
      for (const auto& b : bl) n_fg += b.area;
      if (n_fg > pixels_cap) throw Error(TRB_CAPACITY, "pixel list buffer too small");
      if (n_fg > 0) pixel_lists(ws.ccl->labels(), px, n_fg, pixels_out, ws.st);
    }
    TRB_CUDA(cudaStreamSynchronize(ws.st));
    if (blobs_out && nb > blob_cap) throw Error(TRB_CAPACITY, "blob buffer too small");
  });
}

// ------------------------------------------------- blob appearance features
namespace {
// extract_blob_features (segmentation.hpp:268-291).  The reference's double
// sums of byte values are exact (< 2^53), so per-label integer sums with
// atomics give the same doubles.  One thread = 16 consecutive pixels; runs
// of one label are flushed with one atomic.
__global__ void blob_feature_sum_kernel(const int32_t* labels, int64_t px, const uint8_t* frame, int ch, int n_blobs,
                                        unsigned long long* sums) {
  const int64_t p0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16;
  if (p0 >= px) return;
  const int64_t p1 = min(px, p0 + 16);
  int cur = 0;
  unsigned long long acc = 0;
  for (int64_t p = p0; p < p1; ++p) {
    const int l = labels[p];
    if (l != cur) {
      if (cur > 0 && cur <= n_blobs) atomicAdd(&sums[cur - 1], acc);
      cur = l, acc = 0;
    }
    if (l == 0) continue;
    unsigned v;
    if (ch == 1) {
      v = frame[p];
    } else {
      const uint8_t* q = frame + 3 * p;
      v = (77u * q[0] + 150u * q[1] + 29u * q[2] + 128u) >> 8;  // luma, frame.hpp:91-93
    }
    acc += v;
  }
  if (cur > 0 && cur <= n_blobs) atomicAdd(&sums[cur - 1], acc);
}

__global__ void blob_feature_final_kernel(const trb_blob* blobs, int n, const unsigned long long* sums, double* mean,
                                          double* aspect) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const trb_blob b = blobs[i];
  mean[i] = __ddiv_rn(static_cast<double>(sums[i]), static_cast<double>(b.area));
  aspect[i] = __ddiv_rn(static_cast<double>(b.x_max - b.x_min + 1), static_cast<double>(b.y_max - b.y_min + 1));
}

// device pointers in, device pointers out
void device_blob_features(const int32_t* labels, int64_t px, const uint8_t* frame, int ch, const trb_blob* blobs,
                          int n, double* mean, double* aspect, cudaStream_t st) {
  if (n <= 0) return;
  trb::DevBuf sums;
  sums.alloc(sizeof(unsigned long long) * n, false);
  TRB_CUDA(cudaMemsetAsync(sums.p, 0, sizeof(unsigned long long) * n, st));  // ordered before the atomics
  blob_feature_sum_kernel<<<static_cast<unsigned>(trb::ceil_div64(trb::ceil_div64(px, 16), 256)), 256, 0, st>>>(
      labels, px, frame, ch, n, sums.as<unsigned long long>());
  TRB_LAUNCH_CHECK("blob_feature_sum_kernel");
  blob_feature_final_kernel<<<static_cast<unsigned>(trb::ceil_div64(n, 256)), 256, 0, st>>>(
      blobs, n, sums.as<unsigned long long>(), mean, aspect);
  TRB_LAUNCH_CHECK("blob_feature_final_kernel");
  TRB_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

int trb_extract_blob_features(const int32_t* labels, int width, int height, const uint8_t* frame, int frame_width,
                              int frame_height, int channels, const trb_blob* blobs, int n_blobs, int device,
                              double* mean_intensity, double* aspect) {
  return guard([&] {
    need(labels && frame && (blobs || n_blobs == 0) && (mean_intensity || n_blobs == 0) &&
             (aspect || n_blobs == 0),
         "null argument");
    if (width != frame_width || height != frame_height)
      throw Error(TRB_INVALID_ARGUMENT, "label image dimensions do not match frame");
    need(channels == 1 || channels == 3, "frame channels must be 1 or 3");
    need(width >= 1 && height >= 1 && n_blobs >= 0, "dimensions must be >= 1");
    use_device(device);
    if (n_blobs == 0) return;
    const int64_t px = static_cast<int64_t>(width) * height;
    trb::DevBuf dl, df, db, dm, da;
    dl.alloc(sizeof(int32_t) * px, false);
    df.alloc(static_cast<size_t>(px) * channels, false);
    db.alloc(sizeof(trb_blob) * n_blobs, false);
    dm.alloc(sizeof(double) * n_blobs, false);
    da.alloc(sizeof(double) * n_blobs, false);
    TRB_CUDA(cudaMemcpy(dl.p, labels, sizeof(int32_t) * px, cudaMemcpyHostToDevice));
    TRB_CUDA(cudaMemcpy(df.p, frame, static_cast<size_t>(px) * channels, cudaMemcpyHostToDevice));
    TRB_CUDA(cudaMemcpy(db.p, blobs, sizeof(trb_blob) * n_blobs, cudaMemcpyHostToDevice));
    device_blob_features(dl.as<int32_t>(), px, df.as<uint8_t>(), channels, db.as<trb_blob>(), n_blobs,
                         dm.as<double>(), da.as<double>(), 0);
    TRB_CUDA(cudaMemcpy(mean_intensity, dm.p, sizeof(double) * n_blobs, cudaMemcpyDeviceToHost));
    TRB_CUDA(cudaMemcpy(aspect, da.p, sizeof(double) * n_blobs, cudaMemcpyDeviceToHost));
  });
}

// ------------------------------------------------------------- tracker
int trb_tracker_create(const trb_tracker_config* cfg, int device, trb_tracker** out) {
  return guard([&] {
    need(cfg && out, "null argument");
    *out = nullptr;
    trb::validate_tracker(*cfg);
    use_device(device);
    auto t = std::make_unique<trb_tracker>();
    t->device = device;
    t->cfg = *cfg;
    t->t = std::make_unique<trb::TrackerState>(*cfg, 1, 4096, 1 << 20);
    t->ptrs.alloc(sizeof(void*), false);
    t->nblobs.alloc(sizeof(int32_t));
    TRB_CUDA(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
    *out = t.release();
  });
}

int trb_tracker_destroy(trb_tracker* t) {
  return guard([&] {
    if (t) {
      cudaSetDevice(t->device);
      delete t;
    }
  });
}

int trb_tracker_process(trb_tracker* t, const uint8_t* frame, int width, int height, int channels,
                        const trb_blob* blobs, int n_blobs) {
  return guard([&] {
    need(t && frame, "null argument");
    need(width >= 1 && height >= 1, "frame dimensions must be >= 1");
    need(channels == 1 || channels == 3, "frame channels must be 1 or 3");
    need(n_blobs >= 0 && (n_blobs == 0 || blobs), "bad blob list");
    TRB_CUDA(cudaSetDevice(t->device));
    const size_t fb = static_cast<size_t>(width) * height * channels;
    if (fb > t->frame_bytes) {
      t->frame.alloc(fb, false);
      t->frame_bytes = fb;
      const void* fp = t->frame.p;
      TRB_CUDA(cudaMemcpy(t->ptrs.p, &fp, sizeof(void*), cudaMemcpyHostToDevice));
    }
    if (n_blobs > t->blob_cap) {
      t->blob_cap = std::max<int64_t>(n_blobs, 2 * t->blob_cap);
      t->blobs.alloc(sizeof(trb_blob) * t->blob_cap, false);
    }
    if (t->blob_cap == 0) {
      t->blob_cap = 16;
      t->blobs.alloc(sizeof(trb_blob) * 16, false);
    }
    TRB_CUDA(cudaMemcpyAsync(t->frame.p, frame, fb, cudaMemcpyHostToDevice, t->st));
    if (n_blobs > 0)
      TRB_CUDA(cudaMemcpyAsync(t->blobs.p, blobs, sizeof(trb_blob) * n_blobs, cudaMemcpyHostToDevice, t->st));
    const int32_t nb = n_blobs;
    TRB_CUDA(cudaMemcpyAsync(t->nblobs.p, &nb, sizeof(int32_t), cudaMemcpyHostToDevice, t->st));
    int launches = 0;
    t->t->process(t->ptrs.as<const uint8_t* const>(), width, height, channels, t->blobs.as<trb_blob>(), t->blob_cap,
                  t->nblobs.as<int32_t>(), t->st, &launches);
    t->t->check_errors(t->st);
  });
}

int trb_tracker_num_tracks(const trb_tracker* t, int* n) {
  return guard([&] {
    need(t && n, "null argument");
    TRB_CUDA(cudaSetDevice(t->device));
    *n = t->t->num_tracks(0, t->st);
  });
}

int trb_tracker_tracks(const trb_tracker* t, trb_track* out, int cap) {
  return guard([&] {
    need(t && out, "null argument");
    TRB_CUDA(cudaSetDevice(t->device));
    t->t->tracks(0, out, cap, t->st);
  });
}

int trb_tracker_track_model(const trb_tracker* t, int i, double* centers, double* target_hist) {
  return guard([&] {
    need(t != nullptr, "null argument");
    TRB_CUDA(cudaSetDevice(t->device));
    need(i >= 0 && i < t->t->num_tracks(0, t->st), "track index out of range");
    t->t->track_model(0, i, centers, target_hist, t->st);
  });
}

int trb_tracker_log_size(const trb_tracker* t, int64_t* n) {
  return guard([&] {
    need(t && n, "null argument");
    TRB_CUDA(cudaSetDevice(t->device));
    *n = t->t->log_size(0, t->st);
  });
}

int trb_tracker_log(const trb_tracker* t, trb_track_log_entry* out, int64_t cap) {
  return guard([&] {
    need(t && out, "null argument");
    TRB_CUDA(cudaSetDevice(t->device));
    t->t->log(0, out, cap, t->st);
  });
}

int trb_tracker_frames_processed(const trb_tracker* t, int* n) {
  return guard([&] {
    need(t && n, "null argument");
    TRB_CUDA(cudaSetDevice(t->device));
    *n = t->t->frames_processed(0, t->st);
  });
}

// ------------------------------------------------------------- streams
void trb_default_streams_options(trb_streams_options* o) {
  if (o) *o = trb_streams_options{256, 0, 1 << 16};
}

int trb_streams_create(int n_streams, int width, int height, int channels, const trb_motion_config* mc,
                       const trb_seg_config* sc, const trb_tracker_config* tc, int device, trb_streams** out) {
  return trb_streams_create_ex(n_streams, width, height, channels, mc, sc, tc, nullptr, device, out);
}

int trb_streams_create_ex(int n_streams, int width, int height, int channels, const trb_motion_config* mc,
                          const trb_seg_config* sc, const trb_tracker_config* tc, const trb_streams_options* opt,
                          int device, trb_streams** out) {
  return guard([&] {
    need(out != nullptr, "null argument");
    *out = nullptr;
    use_device(device);
    const trb_motion_config m = mc ? *mc : default_motion();
    const trb_seg_config s = sc ? *sc : trb_seg_config{4, TRB_CONN_EIGHT, 4};
    trb_tracker_config t{16, 20, 0.5, 20, 0, 0};
    if (tc) t = *tc;
    auto h = std::make_unique<trb_streams>();
    h->device = device;
    trb_streams_options o{256, 0, 1 << 16};
    if (opt) o = *opt;
    need(o.track_cap >= 1 && o.track_cap <= (1 << 20), "track_cap must be in [1, 2^20]");
    need(o.log_cap >= 1, "log_cap must be >= 1");
    h->s = std::make_unique<trb::Streams>(n_streams, width, height, channels, m, s, t, tc != nullptr, o.track_cap,
                                          o.log_cap);
    *out = h.release();
  });
}

int trb_streams_destroy(trb_streams* s) {
  return guard([&] {
    if (s) {
      cudaSetDevice(s->device);
      delete s;
    }
  });
}

int trb_streams_step_device(trb_streams* s, const uint8_t* const* frames, void* cuda_stream) {
  return guard([&] {
    need(s && frames, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    s->s->step_device(frames, static_cast<cudaStream_t>(cuda_stream));
  });
}

int trb_streams_join(trb_streams* s, void* cuda_stream) {
  return guard([&] {
    need(s != nullptr, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    s->s->join(static_cast<cudaStream_t>(cuda_stream));
  });
}

int trb_streams_step_host(trb_streams* s, const uint8_t* const* frames, int32_t* result_host, void* cuda_stream) {
  return guard([&] {
    need(s && frames, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    s->s->step_host(frames, result_host, static_cast<cudaStream_t>(cuda_stream));
  });
}

int trb_streams_step_device_warp(trb_streams* s, const uint8_t* const* frames, const double* homographies,
                                 void* cuda_stream) {
  return guard([&] {
    need(s && frames, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    s->s->step_device_warp(frames, homographies, static_cast<cudaStream_t>(cuda_stream));
  });
}

int trb_morph_device(const uint8_t* in, uint8_t* out, int width, int height, int n_planes, int op,
                     void* cuda_stream) {
  return guard([&] {
    need(in && out, "null argument");
    need(width >= 1 && height >= 1 && n_planes >= 1, "morphology needs positive dimensions");
    need(op >= TRB_MORPH_ERODE && op <= TRB_MORPH_CLOSE, "unknown morphology op");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    thread_local trb::DevBuf scratch;  // two-pass path only (width not a multiple of 16)
    if (width % 16 != 0 && (op == TRB_MORPH_OPEN || op == TRB_MORPH_CLOSE))
      scratch.alloc(static_cast<size_t>(width) * height * n_planes, false);
    trb::launch_morph(in, out, scratch.as<uint8_t>(), width, height, n_planes, op, st);
  });
}

int trb_warp_frame(const uint8_t* frame, int width, int height, int channels, const double* homography, int device,
                   uint8_t* out) {
  return guard([&] {
    need(frame && homography && out, "null argument");
    need(width >= 1 && height >= 1, "frame dimensions must be >= 1");
    need(channels == 1 || channels == 3, "frame channels must be 1 or 3");
    double inv[9];
    trb::homography_inverse(homography, inv);  // validation first, like warp_frame
    use_device(device);
    const size_t fb = static_cast<size_t>(width) * height * channels;
    trb::DevBuf din, dout, dinv, dptr;
    din.alloc(fb, false);
    dout.alloc(fb, false);
    dinv.alloc(sizeof(inv), false);
    dptr.alloc(sizeof(void*), false);
    const uint8_t* p = din.as<uint8_t>();
    TRB_CUDA(cudaMemcpy(din.p, frame, fb, cudaMemcpyHostToDevice));
    TRB_CUDA(cudaMemcpy(dinv.p, inv, sizeof(inv), cudaMemcpyHostToDevice));
    TRB_CUDA(cudaMemcpy(dptr.p, &p, sizeof(void*), cudaMemcpyHostToDevice));
    trb::launch_warp_frames(dptr.as<const uint8_t*>(), dout.as<uint8_t>(), static_cast<int64_t>(fb),
                            dinv.as<double>(), width, height, channels, 1, 0);
    TRB_CUDA(cudaMemcpy(out, dout.p, fb, cudaMemcpyDeviceToHost));
  });
}

int trb_streams_step_host_async(trb_streams* s, const uint8_t* const* frames, int32_t* result_host,
                                void* cuda_stream) {
  return guard([&] {
    need(s && frames, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    s->s->step_host_async(frames, result_host, static_cast<cudaStream_t>(cuda_stream));
  });
}

int trb_streams_step_host_async_out(trb_streams* s, const uint8_t* const* frames, const trb_step_output* out,
                                    void* cuda_stream) {
  return guard([&] {
    need(s && frames && out, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    s->s->step_host_async(frames, nullptr, static_cast<cudaStream_t>(cuda_stream), out);
  });
}

int trb_streams_drain_log(trb_streams* s, int stream, trb_track_log_entry* out, int64_t cap, int64_t* n) {
  return guard([&] {
    need(s && out && n, "null argument");
    need(s->s->tracker() != nullptr, "streams were created without a tracker");
    need(stream >= 0 && stream < s->s->S(), "stream index out of range");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    *n = s->s->tracker()->drain_log(stream, out, cap, s->s->stream());
  });
}

int trb_streams_synchronize(trb_streams* s) {
  return guard([&] {
    need(s != nullptr, "null argument");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    if (s->s->tracker()) s->s->tracker()->check_errors(s->s->stream());
  });
}

int trb_streams_frames_seen(const trb_streams* s, int* n) {
  return guard([&] {
    need(s && n, "null argument");
    *n = s->s->frames_seen();
  });
}

int trb_streams_has_output(const trb_streams* s, int* has) {
  return guard([&] {
    need(s && has, "null argument");
    *has = s->s->has_output() ? 1 : 0;
  });
}

int trb_streams_download_mask(trb_streams* s, int stream, uint8_t* out) {
  return guard([&] {
    need(s && out, "null argument");
    need(stream >= 0 && stream < s->s->S(), "stream index out of range");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    TRB_CUDA(cudaMemcpy(out, s->s->mask(stream), s->s->px(), cudaMemcpyDeviceToHost));
  });
}

int trb_streams_download_labels(trb_streams* s, int stream, int32_t* out) {
  return guard([&] {
    need(s && out, "null argument");
    need(stream >= 0 && stream < s->s->S(), "stream index out of range");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    TRB_CUDA(cudaMemcpy(out, s->s->ccl().labels() + s->s->px() * stream, sizeof(int32_t) * s->s->px(),
                        cudaMemcpyDeviceToHost));
  });
}

int trb_streams_download_blobs(trb_streams* s, int stream, trb_blob* out, int cap, int* n) {
  return guard([&] {
    need(s && n, "null argument");
    need(stream >= 0 && stream < s->s->S(), "stream index out of range");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    int32_t nb = 0;
    TRB_CUDA(cudaMemcpy(&nb, s->s->ccl().nblobs() + stream, sizeof(int32_t), cudaMemcpyDeviceToHost));
    *n = nb;
    if (out && nb > 0)
      TRB_CUDA(cudaMemcpy(out, s->s->ccl().blobs() + s->s->ccl().blob_cap() * stream,
                          sizeof(trb_blob) * std::min(nb, cap), cudaMemcpyDeviceToHost));
    if (out && nb > cap) throw Error(TRB_CAPACITY, "blob buffer too small");
  });
}

int trb_streams_log_size(trb_streams* s, int stream, int64_t* n) {
  return guard([&] {
    need(s && n, "null argument");
    need(s->s->tracker() != nullptr, "streams were created without a tracker");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    *n = s->s->tracker()->log_size(stream, s->s->stream());
  });
}

int trb_streams_download_log(trb_streams* s, int stream, trb_track_log_entry* out, int64_t cap) {
  return guard([&] {
    need(s && out, "null argument");
    need(s->s->tracker() != nullptr, "streams were created without a tracker");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    s->s->tracker()->check_errors(s->s->stream(), false);  // the entries held are valid after a log overflow
    s->s->tracker()->log(stream, out, cap, s->s->stream());
  });
}

int trb_streams_num_tracks(trb_streams* s, int stream, int* n) {
  return guard([&] {
    need(s && n, "null argument");
    need(s->s->tracker() != nullptr, "streams were created without a tracker");
    TRB_CUDA(cudaSetDevice(s->device));
    TRB_CUDA(cudaDeviceSynchronize());
    *n = s->s->tracker()->num_tracks(stream, s->s->stream());
  });
}

int trb_streams_last_step_launches(const trb_streams* s, int* n) {
  return guard([&] {
    need(s && n, "null argument");
    *n = s->s->last_launches();
  });
}

int trb_streams_profile(trb_streams* s, int enable) {
  return guard([&] {
    need(s != nullptr, "null argument");
    s->s->set_profiling(enable != 0);
  });
}

int trb_streams_profile_read(const trb_streams* s, double* ms_out, int* steps) {
  return guard([&] {
    need(s && ms_out && steps, "null argument");
    for (int i = 0; i < trb::Streams::kStages; ++i) ms_out[i] = s->s->profile_ms()[i];
    *steps = s->s->profile_steps();
  });
}

int trb_streams_blob_features(trb_streams* s, int stream, const uint8_t* frame_dev, double* mean_intensity,
                              double* aspect, int cap, int* n) {
  return guard([&] {
    need(s && frame_dev && n, "null argument");
    need(stream >= 0 && stream < s->s->S(), "stream index out of range");
    TRB_CUDA(cudaSetDevice(s->device));
    trb::Streams& st = *s->s;
    TRB_CUDA(cudaDeviceSynchronize());
    int32_t nb = 0;
    if (st.has_output())
      TRB_CUDA(cudaMemcpy(&nb, st.ccl().nblobs() + stream, sizeof(int32_t), cudaMemcpyDeviceToHost));
    *n = nb;
    if (nb == 0) return;
    if (nb > cap) throw Error(TRB_CAPACITY, "feature buffer too small");
    need(mean_intensity && aspect, "null argument");
    trb::DevBuf dm, da;
    dm.alloc(sizeof(double) * nb, false);
    da.alloc(sizeof(double) * nb, false);
    device_blob_features(st.ccl().labels() + st.px() * stream, st.px(), frame_dev, st.ch(),
                         st.ccl().blobs() + st.ccl().blob_cap() * stream, nb, dm.as<double>(), da.as<double>(),
                         st.stream());
    TRB_CUDA(cudaMemcpy(mean_intensity, dm.p, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    TRB_CUDA(cudaMemcpy(aspect, da.p, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  });
}

int trb_streams_device_planes(trb_streams* s, int stream, uint8_t** mask, int32_t** labels) {
  return guard([&] {
    need(s != nullptr, "null argument");
    need(stream >= 0 && stream < s->s->S(), "stream index out of range");
    if (mask) *mask = s->s->mask(stream);
    if (labels) *labels = s->s->ccl().labels() + s->s->px() * stream;
  });
}

int trb_synth_raster(uint8_t* out_device, int width, int height, int channels, uint8_t background,
                     const int32_t* rects, const uint8_t* colors, int n_shapes, void* cuda_stream) {
  return guard([&] {
    need(out_device != nullptr, "null argument");
    need(channels == 1 || channels == 3, "clip channels must be 1 or 3");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    thread_local DevBuf d;  // reused: the call synchronises before returning
    d.alloc(sizeof(int32_t) * 4 * n_shapes + 3 * n_shapes + 16, false);
    int32_t* dr = d.as<int32_t>();
    uint8_t* dc = reinterpret_cast<uint8_t*>(dr + 4 * n_shapes);
    if (n_shapes > 0) {
      TRB_CUDA(cudaMemcpyAsync(dr, rects, sizeof(int32_t) * 4 * n_shapes, cudaMemcpyHostToDevice, st));
      TRB_CUDA(cudaMemcpyAsync(dc, colors, 3 * n_shapes, cudaMemcpyHostToDevice, st));
    }
    trb::launch_synth_raster(out_device, width, height, channels, background, dr, dc, n_shapes, st);
    TRB_CUDA(cudaStreamSynchronize(st));
  });
}

int trb_synth_raster_frames(uint8_t* out_device, int64_t frame_stride, int n_frames, int width, int height,
                            int channels, uint8_t background, const int32_t* rects, const uint8_t* colors,
                            int n_shapes, void* cuda_stream) {
  return guard([&] {
    need(out_device != nullptr && n_frames >= 1, "bad argument");
    need(channels == 1 || channels == 3, "clip channels must be 1 or 3");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    DevBuf d;
    const size_t nr = static_cast<size_t>(4) * n_shapes * n_frames;
    d.alloc(sizeof(int32_t) * nr + 3 * n_shapes + 16, false);
    int32_t* dr = d.as<int32_t>();
    uint8_t* dc = reinterpret_cast<uint8_t*>(dr + nr);
    if (n_shapes > 0) {
      TRB_CUDA(cudaMemcpyAsync(dr, rects, sizeof(int32_t) * nr, cudaMemcpyHostToDevice, st));
      TRB_CUDA(cudaMemcpyAsync(dc, colors, 3 * n_shapes, cudaMemcpyHostToDevice, st));
    }
    trb::launch_synth_raster(out_device, width, height, channels, background, dr, dc, n_shapes, st, n_frames,
                             frame_stride);
    TRB_CUDA(cudaStreamSynchronize(st));
  });
}

// ----------------------------------------------------- standalone ops
int trb_meanshift_step(const uint8_t* frame, int width, int height, int channels, double* cx, double* cy, int w,
                       int h, const double* centers, const double* target_hist, int k, int max_iters, double eps,
                       int* status, int device) {
  return guard([&] {
    need(frame && cx && cy && centers && target_hist && status, "null argument");
    need(channels == 1 || channels == 3, "frame channels must be 1 or 3");
    need(k >= 1, "quantizer needs at least one centre");
    if (*status != TRB_TRACK_ACTIVE) return;  // meanshift_step, tracking.hpp:126
    use_device(device);
    const size_t fb = static_cast<size_t>(width) * height * channels;
    DevBuf f;
    f.alloc(fb, false);
    TRB_CUDA(cudaMemcpy(f.p, frame, fb, cudaMemcpyHostToDevice));
    trb::device_meanshift_step(f.as<uint8_t>(), width, height, channels, cx, cy, w, h, centers, target_hist, k,
                               max_iters, eps, status, nullptr);
  });
}

int trb_histogram(const uint8_t* frame, int width, int height, int channels, double cx, double cy, int w, int h,
                  const double* centers, int k, int epanechnikov, double* hist_out, int device) {
  return guard([&] {
    need(frame && centers && hist_out, "null argument");
    // histogram(), tracking.hpp:108-110
    if (w < 3 || h < 3) throw Error(TRB_INVALID_ARGUMENT, "histogram window must be >= 3x3");
    use_device(device);
    const size_t fb = static_cast<size_t>(width) * height * channels;
    DevBuf f;
    f.alloc(fb, false);
    TRB_CUDA(cudaMemcpy(f.p, frame, fb, cudaMemcpyHostToDevice));
    if (!trb::device_histogram(f.as<uint8_t>(), width, height, channels, cx, cy, w, h, centers, k, epanechnikov,
                               hist_out, nullptr))
      throw Error(TRB_INVALID_ARGUMENT, "histogram window does not intersect the frame");
  });
}

int trb_quantize_colors(const double* pixels, int64_t n, int k, int iters, uint64_t seed, double* centers_out,
                        int device) {
  return guard([&] {
    need(pixels && centers_out, "null argument");
    use_device(device);
    trb::device_quantize_colors(pixels, n, k, iters, seed, centers_out, nullptr);
  });
}

}  // extern "C"

extern "C" int trb_debug_stats(uint64_t* out16, int reset) {  // 32 entries
  return guard([&] {
    need(out16 != nullptr, "null argument");
    use_device(0);
    trb::read_debug_stats(reinterpret_cast<unsigned long long*>(out16), reset != 0);
  });
}

// ------------------------------------------------------------ self tests
namespace {
__global__ void hypot_kernel(const double* x, const double* y, int64_t n, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = trb::glibc_hypot(x[i], y[i]);
}
}  // namespace

extern "C" int trb_selftest_hypot(const double* x, const double* y, int64_t n, double* out, int on_device) {
  return guard([&] {
    need(x && y && out, "null argument");
    if (!on_device) {
      for (int64_t i = 0; i < n; ++i) out[i] = trb::glibc_hypot(x[i], y[i]);
      return;
    }
    use_device(0);
    DevBuf dx, dy, dout;
    dx.alloc(sizeof(double) * n, false);
    dy.alloc(sizeof(double) * n, false);
    dout.alloc(sizeof(double) * n, false);
    TRB_CUDA(cudaMemcpy(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    TRB_CUDA(cudaMemcpy(dy.p, y, sizeof(double) * n, cudaMemcpyHostToDevice));
    hypot_kernel<<<static_cast<unsigned>(trb::ceil_div64(n, 256)), 256>>>(dx.as<double>(), dy.as<double>(), n,
                                                                         dout.as<double>());
    TRB_LAUNCH_CHECK("hypot_kernel");
    TRB_CUDA(cudaMemcpy(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  });
}

extern "C" int trb_debug_progress(int n_ctas, int** host_out) {
  return guard([&] {
    need(host_out != nullptr, "null argument");
    use_device(0);
    *host_out = trb::enable_progress(n_ctas);
  });
}

extern "C" int trb_debug_itlog(int enable, int64_t* out_pairs, int64_t cap, int64_t* n) {
  return guard([&] {
    use_device(0);
    if (out_pairs && n) *n = trb::read_itlog(reinterpret_cast<long long*>(out_pairs), cap);
    if (enable >= 0) trb::enable_itlog(enable != 0);
  });
}

extern "C" int trb_debug_cta_times(uint64_t* out2048, int reset) {
  return guard([&] {
    need(out2048 != nullptr, "null argument");
    use_device(0);
    trb::read_cta_times(reinterpret_cast<unsigned long long*>(out2048), reset != 0);
  });
}

extern "C" int trb_debug_warp_walks(uint64_t* out128, int reset) {
  return guard([&] {
    need(out128 != nullptr, "null argument");
    use_device(0);
    trb::read_warpwalk(reinterpret_cast<unsigned long long*>(out128), reset != 0);
  });
}

extern "C" int trb_debug_phases(uint64_t* out128) {
  return guard([&] {
    need(out128 != nullptr, "null argument");
    use_device(0);
    trb::read_phases(reinterpret_cast<unsigned long long*>(out128));
  });
}

// ===================================================================== I/O
// SURVEY §8(f) row 3, host side: PNM ingest (frame.hpp:119-225) and the
// track-log interchange (tracking.hpp:244-285), restated in C++ with the
// reference's parsing rules and IoError messages (same standard library, so
// std::stoi / istream / std::sort behave identically).
namespace {
namespace fs = std::filesystem;

std::string pnm_token(const uint8_t* b, size_t n, size_t& pos, const std::string& src) {  // frame.hpp:120-134
  for (;;) {
    while (pos < n && std::isspace(b[pos])) ++pos;
    if (pos < n && b[pos] == '#') {
      while (pos < n && b[pos] != '\n') ++pos;
      continue;
    }
    break;
  }
  if (pos >= n) throw Error(TRB_IO_ERROR, "truncated pnm header in " + src);
  std::string tok;
  while (pos < n && !std::isspace(b[pos])) tok.push_back(static_cast<char>(b[pos++]));
  return tok;
}

int pnm_int(const uint8_t* b, size_t n, size_t& pos, const std::string& src) {  // frame.hpp:136-148
  const std::string tok = pnm_token(b, n, pos, src);
  try {
    size_t used = 0;
    const int v = std::stoi(tok, &used);
    if (used != tok.size()) throw std::invalid_argument(tok);
    return v;
  } catch (const std::exception&) {
    throw Error(TRB_IO_ERROR, "bad pnm header value '" + tok + "' in " + src);
  }
}

struct Pnm {
  int w, h, ch;
  size_t off;  // first pixel byte
};

Pnm decode_pnm_header(const uint8_t* b, size_t n, const std::string& src) {  // decode_pnm, frame.hpp:152-175
  size_t pos = 0;
  const std::string magic = pnm_token(b, n, pos, src);
  int ch = 0;
  if (magic == "P5") ch = 1;
  else if (magic == "P6") ch = 3;
  else throw Error(TRB_IO_ERROR, "unsupported pnm magic '" + magic + "' in " + src + " (want P5 or P6)");
  const int w = pnm_int(b, n, pos, src);
  const int h = pnm_int(b, n, pos, src);
  const int maxval = pnm_int(b, n, pos, src);
  if (w < 1 || h < 1) throw Error(TRB_IO_ERROR, "bad pnm dimensions in " + src);
  if (maxval != 255) throw Error(TRB_IO_ERROR, "unsupported pnm maxval " + std::to_string(maxval) + " in " + src);
  ++pos;  // single whitespace after maxval
  const size_t need = static_cast<size_t>(w) * h * ch;
  if (n < pos || n - pos < need) throw Error(TRB_IO_ERROR, "truncated pnm pixel data in " + src);
  return Pnm{w, h, ch, pos};
}

std::vector<uint8_t> slurp_bytes(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(TRB_IO_ERROR, "cannot open " + path);
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

std::string fmt_g17(double v) {  // textio.hpp:16-20
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

std::string format_track_log(const trb_track_log_entry* log, int64_t n) {  // tracking.hpp:247-256
  std::string out = "# frame track_id x y w h status\n";
  for (int64_t i = 0; i < n; ++i) {
    const auto& e = log[i];
    out += std::to_string(e.frame) + " " + std::to_string(e.track_id) + " " + fmt_g17(e.x) + " " + fmt_g17(e.y) +
           " " + std::to_string(e.w) + " " + std::to_string(e.h) + " " +
           (e.status == TRB_TRACK_ACTIVE ? "active" : "lost") + "\n";
  }
  return out;
}

std::vector<trb_track_log_entry> parse_track_log(const std::string& text, const std::string& source) {  // :258-277
  std::vector<trb_track_log_entry> out;
  std::istringstream in(text);
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const auto first = line.find_first_not_of(" \t\r");
    if (first == std::string::npos || line[first] == '#') continue;
    std::istringstream ls(line);
    trb_track_log_entry e{};
    int frame = 0, id = 0, w = 0, h = 0;
    double x = 0, y = 0;
    std::string status;
    if (!(ls >> frame >> id >> x >> y >> w >> h >> status))
      throw Error(TRB_IO_ERROR, "bad track log record at " + source + ":" + std::to_string(lineno));
    e.frame = frame, e.track_id = id, e.x = x, e.y = y, e.w = w, e.h = h;
    if (status == "active") e.status = TRB_TRACK_ACTIVE;
    else if (status == "lost") e.status = TRB_TRACK_LOST;
    else throw Error(TRB_IO_ERROR, "unknown track status '" + status + "' at " + source + ":" + std::to_string(lineno));
    out.push_back(e);
  }
  return out;
}
}  // namespace

extern "C" {

int trb_decode_pnm(const uint8_t* bytes, int64_t n, const char* source_name, int* width, int* height, int* channels,
                   uint8_t* out, int64_t out_cap) {
  return guard([&] {
    need(bytes && width && height && channels, "null argument");
    const Pnm p = decode_pnm_header(bytes, static_cast<size_t>(n), source_name ? source_name : "<memory>");
    *width = p.w, *height = p.h, *channels = p.ch;
    if (!out) return;
    const size_t need_b = static_cast<size_t>(p.w) * p.h * p.ch;
    if (static_cast<int64_t>(need_b) > out_cap) throw Error(TRB_CAPACITY, "pixel buffer too small");
    std::memcpy(out, bytes + p.off, need_b);
  });
}

int trb_load_pnm(const char* path, int* width, int* height, int* channels, uint8_t* out, int64_t out_cap) {
  return guard([&] {
    need(path && width && height && channels, "null argument");
    const auto b = slurp_bytes(path);
    const Pnm p = decode_pnm_header(b.data(), b.size(), path);
    *width = p.w, *height = p.h, *channels = p.ch;
    if (!out) return;
    const size_t need_b = static_cast<size_t>(p.w) * p.h * p.ch;
    if (static_cast<int64_t>(need_b) > out_cap) throw Error(TRB_CAPACITY, "pixel buffer too small");
    std::memcpy(out, b.data() + p.off, need_b);
  });
}

int trb_load_frame_sequence(const char* dir, int* n_frames, int* width, int* height, int* channels,
                            int64_t* indices, uint8_t* out, int64_t out_cap) {
  return guard([&] {  // load_frame_sequence, frame.hpp:198-225
    need(dir && n_frames && width && height && channels, "null argument");
    const fs::path d(dir);
    if (!fs::is_directory(d)) throw Error(TRB_IO_ERROR, "not a directory: " + d.string());
    std::vector<fs::path> files;
    for (const auto& e : fs::directory_iterator(d)) {
      if (!e.is_regular_file()) continue;
      const auto ext = e.path().extension().string();
      if (ext == ".pgm" || ext == ".ppm") files.push_back(e.path());
    }
    std::sort(files.begin(), files.end());
    struct F {
      std::vector<uint8_t> bytes;
      Pnm p;
      int64_t index;
    };
    std::vector<F> frames;
    for (const auto& path : files) {
      F f;
      f.bytes = slurp_bytes(path.string());
      f.p = decode_pnm_header(f.bytes.data(), f.bytes.size(), path.string());
      const std::string stem = path.stem().string();
      size_t k = stem.size();
      while (k > 0 && std::isdigit(static_cast<unsigned char>(stem[k - 1]))) --k;
      f.index = k < stem.size() ? std::stoll(stem.substr(k)) : static_cast<int64_t>(frames.size());
      if (!frames.empty()) {
        const Pnm& a = frames.front().p;
        if (a.w != f.p.w || a.h != f.p.h || a.ch != f.p.ch)
          throw Error(TRB_IO_ERROR, "dimension mismatch in " + path.string() + ": expected " + std::to_string(a.w) +
                                        "x" + std::to_string(a.h) + "x" + std::to_string(a.ch) + ", got " +
                                        std::to_string(f.p.w) + "x" + std::to_string(f.p.h) + "x" +
                                        std::to_string(f.p.ch));
      }
      frames.push_back(std::move(f));
    }
    std::sort(frames.begin(), frames.end(), [](const F& a, const F& b) { return a.index < b.index; });
    *n_frames = static_cast<int>(frames.size());
    *width = frames.empty() ? 0 : frames[0].p.w;
    *height = frames.empty() ? 0 : frames[0].p.h;
    *channels = frames.empty() ? 0 : frames[0].p.ch;
    if (!out) return;
    const size_t fb = frames.empty() ? 0 : static_cast<size_t>(*width) * *height * *channels;
    if (static_cast<int64_t>(fb * frames.size()) > out_cap) throw Error(TRB_CAPACITY, "frame buffer too small");
    for (size_t i = 0; i < frames.size(); ++i) {
      std::memcpy(out + fb * i, frames[i].bytes.data() + frames[i].p.off, fb);
      if (indices) indices[i] = frames[i].index;
    }
  });
}

int trb_format_track_log(const trb_track_log_entry* log, int64_t n, char* out, int64_t cap, int64_t* len) {
  return guard([&] {
    need((log || n == 0) && len, "null argument");
    const std::string s = format_track_log(log, n);
    *len = static_cast<int64_t>(s.size());
    if (!out) return;
    if (static_cast<int64_t>(s.size()) + 1 > cap) throw Error(TRB_CAPACITY, "text buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

int trb_parse_track_log(const char* text, int64_t len, const char* source, trb_track_log_entry* out, int64_t cap,
                        int64_t* n) {
  return guard([&] {
    need(text && n, "null argument");
    const auto v = parse_track_log(std::string(text, static_cast<size_t>(len)), source ? source : "<memory>");
    *n = static_cast<int64_t>(v.size());
    if (!out) return;
    if (static_cast<int64_t>(v.size()) > cap) throw Error(TRB_CAPACITY, "log buffer too small");
    std::copy(v.begin(), v.end(), out);
  });
}

int trb_save_track_log(const char* path, const trb_track_log_entry* log, int64_t n) {
  return guard([&] {  // save_track_log -> detail::spit (textio.hpp:43-48)
    need(path && (log || n == 0), "null argument");
    std::ofstream o(path, std::ios::binary);
    if (!o) throw Error(TRB_IO_ERROR, std::string("cannot write ") + path);
    o << format_track_log(log, n);
    if (!o) throw Error(TRB_IO_ERROR, std::string("write failed for ") + path);
  });
}

int trb_load_track_log(const char* path, trb_track_log_entry* out, int64_t cap, int64_t* n) {
  return guard([&] {  // load_track_log -> slurp (textio.hpp:35-41) + parse
    need(path && n, "null argument");
    const auto b = slurp_bytes(path);
    const auto v = parse_track_log(std::string(b.begin(), b.end()), path);
    *n = static_cast<int64_t>(v.size());
    if (!out) return;
    if (static_cast<int64_t>(v.size()) > cap) throw Error(TRB_CAPACITY, "log buffer too small");
    std::copy(v.begin(), v.end(), out);
  });
}

}  // extern "C"
