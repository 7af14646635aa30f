// trb_engine.cu — host state machines (see trb_engine.cuh).
#include <algorithm>
#include <cstring>
#include <string>

#include "trb_engine.cuh"
#include "trb_track.cuh"

namespace trb {

// ---------------------------------------------------------------- validate
// MotionConfig::validate (motion.hpp:51-55); morph is this build's extension.
void validate_motion(const trb_motion_config& c) {
  if (c.window < 2) throw Error(TRB_CONFIG_ERROR, "motion window_w must be >= 2");
  if (c.threshold <= 0 || c.threshold >= 255) throw Error(TRB_CONFIG_ERROR, "motion threshold must be in (0,255)");
  if (c.bins < 2 || c.bins > 256) throw Error(TRB_CONFIG_ERROR, "motion histogram_bins must be in [2,256]");
  if (c.method != TRB_BG_MEAN && c.method != TRB_BG_MODE)
    throw Error(TRB_INVALID_ARGUMENT, "unknown background method (expected mean|mode)");
  if (c.morph < TRB_MORPH_NONE || c.morph > TRB_MORPH_CLOSE)
    throw Error(TRB_CONFIG_ERROR, "motion morph must be none|erode|dilate|open|close");
  if (c.warp != 0 && c.warp != 1)
    throw Error(TRB_CONFIG_ERROR, "unknown warp mode (expected identity|homography)");
}

// block_grid (segmentation.hpp:79-84): most-square factorisation.
static std::pair<int, int> block_grid(int n) {
  int rows = 1;
  for (int r = 1; r * r <= n; ++r)
    if (n % r == 0) rows = r;
  return {rows, n / rows};
}

// SegmentationConfig::validate (segmentation.hpp:30-33) + label_blocked's
// grid check (segmentation.hpp:201-205).
void validate_seg(const trb_seg_config& c, int w, int h) {
  if (c.n_blocks < 1) throw Error(TRB_CONFIG_ERROR, "n_blocks must be >= 1");
  if (c.min_area < 1) throw Error(TRB_CONFIG_ERROR, "min_area must be >= 1");
  if (c.connectivity != TRB_CONN_FOUR && c.connectivity != TRB_CONN_EIGHT)
    throw Error(TRB_INVALID_ARGUMENT, "unknown connectivity (expected four|eight)");
  if (w < 1 || h < 1) return;
  const auto [rows, cols] = block_grid(c.n_blocks);
  if (rows > h || cols > w)
    throw Error(TRB_CONFIG_ERROR, "n_blocks=" + std::to_string(c.n_blocks) + " does not tile a " + std::to_string(w) +
                                      "x" + std::to_string(h) + " image (grid " + std::to_string(rows) + "x" +
                                      std::to_string(cols) + ")");
}

// TrackerConfig::validate (tracking.hpp:28-33)
void validate_tracker(const trb_tracker_config& c) {
  if (c.k_clusters < 2) throw Error(TRB_CONFIG_ERROR, "tracker k_clusters must be >= 2");
  if (!(c.eps > 0.0)) throw Error(TRB_CONFIG_ERROR, "tracker eps must be > 0");
  if (c.max_iters < 1) throw Error(TRB_CONFIG_ERROR, "tracker max_iters must be >= 1");
  if (c.kmeans_iters < 1) throw Error(TRB_CONFIG_ERROR, "tracker kmeans_iters must be >= 1");
}

// ------------------------------------------------------------------ motion
MotionState::MotionState(const trb_motion_config& cfg, int S, int w, int h, int ch)
    : cfg_(cfg), S_(S), w_(w), h_(h), ch_(ch) {
  validate_motion(cfg);
  if (w < 1 || h < 1) throw Error(TRB_INVALID_ARGUMENT, "motion detector needs positive frame dimensions");
  px_ = static_cast<int64_t>(w) * h;
  wide_ = cfg.window > 257;  // 255*257 < 2^16
  ring_.alloc(static_cast<size_t>(px_) * cfg.window * S);
  sums_.alloc(static_cast<size_t>(px_) * S * (wide_ ? 4 : 2));
  // Mode: incremental per-bin counts / sums / mode bin when the counts fit
  // a byte (W <= 255); TRB_MODE_INC=0 keeps the ring re-read (A/B)
  const char* e = getenv("TRB_MODE_INC");
  mode_inc_ = cfg.method == TRB_BG_MODE && cfg.window <= 255 && !(e && atoi(e) == 0);
  if (mode_inc_) {
    cnt_.alloc(static_cast<size_t>(px_) * cfg.bins * S);
    bsum_.alloc(sizeof(uint16_t) * static_cast<size_t>(px_) * cfg.bins * S);
    mode_.alloc(static_cast<size_t>(px_) * S);
  }
}

bool MotionState::push(const uint8_t* const* frames_dev, uint8_t* mask, uint8_t* tmp, cudaStream_t st,
                       int* launches, bool frames_aligned) {
  const int W = cfg_.window;
  MotionArgs a{};
  a.frames = frames_dev;
  a.ring = ring_.as<uint8_t>();
  a.ring_stride = px_ * W;
  a.sums = sums_.p;
  // with morphology, motion writes its raw mask into tmp and the (fused)
  // morphology stage writes the final mask
  const bool morph = cfg_.morph != TRB_MORPH_NONE;
  uint8_t* raw = morph ? tmp : mask;
  a.mask = raw;
  a.px = px_;
  a.slot = frames_seen_ % W;
  a.full_before = frames_seen_ >= W;
  a.emit = frames_seen_ + 1 >= W;
  a.threshold = cfg_.threshold;
  a.W = static_cast<uint32_t>(W);
  a.div = FastDiv::make(2u * static_cast<uint32_t>(W));
  a.vec_ok = (px_ % 16 == 0) && frames_aligned;
  if (cfg_.method == TRB_BG_MEAN) {
    launch_motion_mean(a, ch_, wide_, S_, st);
    ++*launches;
  } else if (mode_inc_) {
    ModeIncArgs m{};
    m.frames = frames_dev;
    m.ring = ring_.as<uint8_t>();
    m.ring_stride = px_ * W;
    m.cnt = cnt_.as<uint8_t>();
    m.bsum = bsum_.as<uint16_t>();
    m.mode = mode_.as<uint8_t>();
    m.mask = raw;
    m.px = px_;
    m.slot = a.slot;
    m.full_before = a.full_before;
    m.emit = a.emit;
    m.threshold = cfg_.threshold;
    m.bins = cfg_.bins;
    launch_motion_mode_inc(m, ch_, S_, st);
    ++*launches;
  } else {
    launch_ring_update(a, ch_, wide_, S_, st);
    ++*launches;
    if (a.emit) {
      ModeArgs m{};
      m.ring = ring_.as<uint8_t>();
      m.ring_stride = px_ * W;
      m.px = px_;
      m.W = W;
      m.bins = cfg_.bins;
      m.threshold = cfg_.threshold;
      m.newest = a.slot;
      m.mask = raw;
      launch_motion_mode(m, S_, st);
      ++*launches;
    }
  }
  ++frames_seen_;
  if (!a.emit) return false;
  if (morph) *launches += launch_morph(raw, mask, tmp + static_cast<size_t>(px_) * S_, w_, h_, S_, cfg_.morph, st);
  return true;
}

void MotionState::background(uint8_t* out_dev, cudaStream_t st) {
  if (frames_seen_ < cfg_.window)
    throw Error(TRB_INVALID_ARGUMENT, "background not available before the window fills");
  if (cfg_.method == TRB_BG_MEAN) {
    launch_mean_background(sums_.p, px_, cfg_.window, wide_, out_dev, st);
  } else {
    ModeArgs m{};
    m.ring = ring_.as<uint8_t>();
    m.ring_stride = px_ * cfg_.window;
    m.px = px_;
    m.W = cfg_.window;
    m.bins = cfg_.bins;
    m.threshold = cfg_.threshold;
    m.bg_out = out_dev;
    launch_motion_mode(m, 1, st);
  }
}

// --------------------------------------------------------------------- CCL
CclState::CclState(int S, int w, int h, const trb_seg_config& cfg) : S_(S), w_(w), h_(h) {
  validate_seg(cfg, w, h);
  px_ = static_cast<int64_t>(w) * h;
  const int tx = ceil_div(w, kTileW), ty = ceil_div(h, kTileH);
  if (tx > 1024 || ty > 1024 || S > 2047)  // packed tile-list entries (trb_ccl.cu: tile_pack)
    throw Error(TRB_CONFIG_ERROR, "labelling supports frames up to 32768 x 32768 and 2047 streams per handle");
  slot_cap_ = static_cast<int64_t>(tx) * ty * kMaxTileComps;
  blob_cap_ = px_ / 2 + 1;
  const int wpr = ceil_div(w, 32);
  labg_.alloc(sizeof(int32_t) * px_ * S, false);
  labels_.alloc(sizeof(int32_t) * px_ * S);
  // 11 per-slot arrays: 9 x int32 + 2 x u64
  slots_.alloc(static_cast<size_t>(slot_cap_) * S * (9 * 4 + 2 * 8), false);
  nslots_.alloc(sizeof(int32_t) * S);
  rowcount_.alloc(sizeof(int32_t) * h * S);
  bitmap_.alloc(sizeof(uint32_t) * static_cast<size_t>(h) * wpr * S);
  for (int b = 0; b < 2; ++b) {
    blobs_[b].alloc(sizeof(trb_blob) * blob_cap_ * S, false);
    nblobs_[b].alloc(sizeof(int32_t) * S);
  }
  tiles_.alloc(sizeof(int32_t) * (static_cast<size_t>(tx) * ty * S + 1));  // zeroed: the tile-list counter starts at 0 (then ccl_final resets it)
  tile_state_.alloc(static_cast<size_t>(tx) * ty * S);  // zeroed: no tile labelled yet (labels_ is zeroed too)

  CclArgs& a = args_;
  a.labg = labg_.as<int32_t>();
  a.labels = labels_.as<int32_t>();
  a.w = w;
  a.h = h;
  a.px = px_;
  a.conn = cfg.connectivity;
  a.min_area = cfg.min_area;
  a.tiles_x = tx;
  a.tiles_y = ty;
  const size_t n = static_cast<size_t>(slot_cap_) * S;
  char* base = slots_.as<char>();
  // u64 arrays first for alignment
  a.slots.sx = reinterpret_cast<unsigned long long*>(base);
  a.slots.sy = a.slots.sx + n;
  int32_t* i32 = reinterpret_cast<int32_t*>(a.slots.sy + n);
  a.slots.parent = i32 + 0 * n;
  a.slots.root = i32 + 1 * n;
  a.slots.area = i32 + 2 * n;
  a.slots.x0 = i32 + 3 * n;
  a.slots.y0 = i32 + 4 * n;
  a.slots.x1 = i32 + 5 * n;
  a.slots.y1 = i32 + 6 * n;
  a.slots.minpix = i32 + 7 * n;
  a.slots.dense = i32 + 8 * n;
  a.slot_cap = slot_cap_;
  a.nslots = nslots_.as<int32_t>();
  a.rowcount = rowcount_.as<int32_t>();
  a.bitmap = bitmap_.as<uint32_t>();
  a.wpr = wpr;
  a.blob_cap = blob_cap_;
  a.tile_count = tiles_.as<int32_t>();
  a.tile_list = a.tile_count + 1;
  a.tile_state = tile_state_.as<uint8_t>();
}

void CclState::run(const uint8_t* mask, cudaStream_t st, int* launches) {
  const int b = cur_ ^ 1;
  args_.mask = mask;
  args_.blobs = blobs_[b].as<trb_blob>();
  args_.nblobs = nblobs_[b].as<int32_t>();
  *launches += launch_ccl(args_, S_, st);
  cur_ = b;
}

// ----------------------------------------------------------------- streams
Streams::Streams(int S, int w, int h, int ch, const trb_motion_config& mc, const trb_seg_config& sc,
                 const trb_tracker_config& tc, bool with_tracker, int track_cap, int64_t log_cap)
    : S_(S), w_(w), h_(h), ch_(ch), mc_(mc) {
  if (S < 1) throw Error(TRB_INVALID_ARGUMENT, "need at least one stream");
  if (ch != 1 && ch != 3) throw Error(TRB_INVALID_ARGUMENT, "frame channels must be 1 or 3");
  if (w < 1 || h < 1) throw Error(TRB_INVALID_ARGUMENT, "frame dimensions must be >= 1");
  if (with_tracker) validate_tracker(tc);
  px_ = static_cast<int64_t>(w) * h;
  motion_ = std::make_unique<MotionState>(mc, S, w, h, ch);
  ccl_ = std::make_unique<CclState>(S, w, h, sc);
  if (with_tracker) tracker_ = std::make_unique<TrackerState>(tc, S, track_cap, log_cap);
  mask_.alloc(static_cast<size_t>(px_) * S);
  if (mc.morph != TRB_MORPH_NONE) mask_tmp_.alloc(static_cast<size_t>(px_) * S * 2);  // raw mask + 2-pass scratch
  // ring of per-step frame-pointer tables: a table is rewritten only after
  // the event of its previous use completed, so steps never block the host
  frame_ptrs_.alloc(sizeof(void*) * S * kPtrSlots);
  ptrs_host_.alloc(sizeof(void*) * S * kPtrSlots);
  for (int i = 0; i < kPtrSlots; ++i) TRB_CUDA(cudaEventCreateWithFlags(&slot_ev_[i], cudaEventDisableTiming));
  for (int i = 0; i < kStages + 1; ++i) TRB_CUDA(cudaEventCreate(&prof_ev_[i]));
  TRB_CUDA(cudaStreamCreateWithFlags(&own_, cudaStreamNonBlocking));
  TRB_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
  {
    // The tracker's internal stream runs at the highest priority: with the
    // step overlap its persistent mean-shift CTAs are then dispatched ahead
    // of the next step's motion / CCL blocks, which fill the SMs around them
    // (C5MODE +15 %, C5 neutral; profiles/r02_ab_tracker_priority.txt).
    // TRB_TRK_PRIO (A/B): 1 highest (default), 0 default priority, -1 lowest.
    const char* e = getenv("TRB_TRK_PRIO");
    const int want = e ? atoi(e) : 1;
    int lo = 0, hi = 0;
    TRB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (want == 0) TRB_CUDA(cudaStreamCreateWithFlags(&trk_, cudaStreamNonBlocking));
    else TRB_CUDA(cudaStreamCreateWithPriority(&trk_, cudaStreamNonBlocking, want > 0 ? hi : lo));
  }
  if (const char* e = getenv("TRB_OVERLAP")) overlap_ = atoi(e) != 0;
  if (const char* e = getenv("TRB_EARLY_MS")) early_ms_ = atoi(e) != 0;
  if (const char* e = getenv("TRB_DIRECT_OUT")) direct_out_ = atoi(e) != 0;
  // host-path staging ring, allocated up front: a step never cudaMallocs
  // (that would serialise the device inside the first host steps)
  for (int i = 0; i < kStaging; ++i) staging_[i].alloc(static_cast<size_t>(px_) * ch_ * S_, false);
  {
    // the host path's frame-pointer tables never change (stream s of staging
    // buffer b is at a fixed offset): uploaded once instead of every step
    std::vector<const uint8_t*> tab(static_cast<size_t>(kStaging) * S_);
    const size_t fb = static_cast<size_t>(px_) * ch_;
    for (int i = 0; i < kStaging; ++i)
      for (int s = 0; s < S_; ++s) tab[static_cast<size_t>(i) * S_ + s] = staging_[i].as<uint8_t>() + fb * s;
    staging_ptrs_.alloc(sizeof(void*) * tab.size(), false);
    TRB_CUDA(cudaMemcpy(staging_ptrs_.p, tab.data(), sizeof(void*) * tab.size(), cudaMemcpyHostToDevice));
  }
  for (int i = 0; i < kStaging; ++i) {
    TRB_CUDA(cudaEventCreateWithFlags(&copied_[i], cudaEventDisableTiming));
    TRB_CUDA(cudaEventCreateWithFlags(&consumed_[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < 2; ++i) {
    TRB_CUDA(cudaEventCreateWithFlags(&ccl_ev_[i], cudaEventDisableTiming));
    TRB_CUDA(cudaEventCreateWithFlags(&mot_ev_[i], cudaEventDisableTiming));
    TRB_CUDA(cudaEventCreateWithFlags(&trk_ev_[i], cudaEventDisableTiming));
  }
}

Streams::~Streams() {
  for (auto& e : slot_ev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : prof_ev_)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < kStaging; ++i) {
    if (copied_[i]) cudaEventDestroy(copied_[i]);
    if (consumed_[i]) cudaEventDestroy(consumed_[i]);
  }
  for (int i = 0; i < 2; ++i) {
    if (ccl_ev_[i]) cudaEventDestroy(ccl_ev_[i]);
    if (mot_ev_[i]) cudaEventDestroy(mot_ev_[i]);
    if (trk_ev_[i]) cudaEventDestroy(trk_ev_[i]);
  }
  if (trk_) cudaStreamDestroy(trk_);
  if (copy_) cudaStreamDestroy(copy_);
  if (own_) cudaStreamDestroy(own_);
}

void Streams::set_profiling(bool on) {
  profiling_ = on;
  for (double& v : prof_ms_) v = 0.0;
  prof_steps_ = 0;
}

// Step overlap.  Motion and CCL of step t+1 do not depend on the tracker of
// step t (only step t+1's tracker does), so with `overlap` the tracker runs
// on the internal stream trk_ behind an event of this step's CCL, and the
// caller's stream goes on to the next step's motion + CCL while it runs.
// Hazards: CCL(t+1) writes the other blob table (double-buffered) and waits
// for the tracker that last read it (step t-1); at the end of step t the
// caller's stream also waits for the tracker of step t-1 (a lag-one join,
// which costs no overlap: that tracker ended before step t's began), so the
// caller's stream trails the issued work by at most one tracker — join()
// closes it.  `done` (frames released) is recorded after the tracker.
cudaStream_t Streams::run_(const uint8_t* const* frames_dev, cudaStream_t st, bool overlap, cudaEvent_t done) {
  int launches = 0;
  overlap = overlap && tracker_ && !profiling_;
  if (profiling_) TRB_CUDA(cudaEventRecord(prof_ev_[0], st));
  const bool emitted =
      motion_->push(frames_dev, mask_.as<uint8_t>(), mask_tmp_.as<uint8_t>(), st, &launches, frames_aligned_);
  has_output_ = emitted;
  if (profiling_) TRB_CUDA(cudaEventRecord(prof_ev_[1], st));
  const int b = ccl_->next_buffer();
  // the step's frames (and their pointer table) are ready for the tracker
  // once the motion kernel has run (it waited for any upload)
  if (emitted && tracker_ && overlap && early_ms_) TRB_CUDA(cudaEventRecord(mot_ev_[b], st));
  if (emitted) {
    if (trk_pending_[b]) TRB_CUDA(cudaStreamWaitEvent(st, trk_ev_[b], 0));  // its last reader
    ccl_->run(mask_.as<uint8_t>(), st, &launches);
  }
  if (profiling_) TRB_CUDA(cudaEventRecord(prof_ev_[2], st));
  if (emitted && tracker_ && overlap) {
    TRB_CUDA(cudaEventRecord(ccl_ev_[b], st));
    // mean-shift needs the frames and the track state only: it starts after
    // the step's motion kernel, beside the CCL; the gate (the blob table's
    // first reader) waits for the CCL
    TRB_CUDA(cudaStreamWaitEvent(trk_, early_ms_ ? mot_ev_[b] : ccl_ev_[b], 0));
    tracker_->process(frames_dev, w_, h_, ch_, ccl_->blobs(), ccl_->blob_cap(), ccl_->nblobs(), trk_, &launches,
                      nullptr, early_ms_ ? ccl_ev_[b] : nullptr);
    if (pending_out_) output_(pending_out_, trk_, &launches);  // before CCL(t+2) may reuse this blob table
    TRB_CUDA(cudaEventRecord(trk_ev_[b], trk_));
    trk_pending_[b] = true;
    last_trk_ = b;
    if (trk_pending_[b ^ 1]) TRB_CUDA(cudaStreamWaitEvent(st, trk_ev_[b ^ 1], 0));  // lag-one join
    if (done) TRB_CUDA(cudaEventRecord(done, trk_));
  } else {
    if (last_trk_ >= 0) join(st), last_trk_ = -1;  // back to in-stream tracking (profiling, warp mode)
    if (emitted && tracker_) {
      tracker_->process(frames_dev, w_, h_, ch_, ccl_->blobs(), ccl_->blob_cap(), ccl_->nblobs(), st, &launches,
                        profiling_ ? prof_ev_[3] : nullptr);
    }
    if (pending_out_) output_(pending_out_, st, &launches);
    if (!(emitted && tracker_) && profiling_)
      TRB_CUDA(cudaEventRecord(prof_ev_[3], st));
    if (done) TRB_CUDA(cudaEventRecord(done, st));
  }
  if (profiling_) {
    TRB_CUDA(cudaEventRecord(prof_ev_[4], st));
    TRB_CUDA(cudaEventSynchronize(prof_ev_[4]));
    for (int i = 0; i < kStages; ++i) {
      float ms = 0.f;
      TRB_CUDA(cudaEventElapsedTime(&ms, prof_ev_[i], prof_ev_[i + 1]));
      prof_ms_[i] += ms;
    }
    ++prof_steps_;
  }
  has_output_ = emitted;
  last_launches_ = launches;
  return (overlap && emitted) ? trk_ : st;
}

void Streams::join(cudaStream_t st) {
  if (!st) st = own_;
  if (last_trk_ >= 0) TRB_CUDA(cudaStreamWaitEvent(st, trk_ev_[last_trk_], 0));
}

const uint8_t* const* Streams::upload_ptrs_(const uint8_t* const* frames, cudaStream_t st) {
  const int slot = ptr_slot_;
  ptr_slot_ = (ptr_slot_ + 1) % kPtrSlots;
  TRB_CUDA(cudaEventSynchronize(slot_ev_[slot]));  // previous use of this table is done
  const uint8_t** hp = ptrs_host_.as<const uint8_t*>() + static_cast<size_t>(slot) * S_;
  std::memcpy(hp, frames, sizeof(void*) * S_);
  const uint8_t** dp = frame_ptrs_.as<const uint8_t*>() + static_cast<size_t>(slot) * S_;
  TRB_CUDA(cudaMemcpyAsync(dp, hp, sizeof(void*) * S_, cudaMemcpyHostToDevice, st));
  return dp;
}

void Streams::step_device_warp(const uint8_t* const* frames, const double* h9s, cudaStream_t st) {
  if (!st) st = own_;
  check_sticky_errors();
  if (!h9s) throw Error(TRB_INVALID_ARGUMENT, "warp mode homography requires per-frame homographies");
  const size_t fb = static_cast<size_t>(px_) * ch_;
  if (!warp_buf_.p) {
    warp_buf_.alloc(fb * S_);
    std::vector<const uint8_t*> wp(S_);
    for (int s = 0; s < S_; ++s) wp[s] = warp_buf_.as<uint8_t>() + fb * s;
    warp_ptrs_.alloc(sizeof(void*) * S_, false);
    TRB_CUDA(cudaMemcpy(warp_ptrs_.p, wp.data(), sizeof(void*) * S_, cudaMemcpyHostToDevice));
    invs_dev_.alloc(sizeof(double) * 9 * S_ * kPtrSlots, false);
    invs_host_.alloc(sizeof(double) * 9 * S_ * kPtrSlots);
  }
  frames_aligned_ = true;  // the motion kernel reads the warped planes (own buffers)
  const int slot = ptr_slot_;
  const uint8_t* const* dp = upload_ptrs_(frames, st);  // waits for the slot's previous use
  double* ih = static_cast<double*>(invs_host_.p) + static_cast<size_t>(slot) * 9 * S_;
  for (int s = 0; s < S_; ++s) homography_inverse(h9s + 9 * s, ih + 9 * s);
  double* id = invs_dev_.as<double>() + static_cast<size_t>(slot) * 9 * S_;
  TRB_CUDA(cudaMemcpyAsync(id, ih, sizeof(double) * 9 * S_, cudaMemcpyHostToDevice, st));
  // no overlap: the next step's warp rewrites the plane this tracker reads
  launch_warp_frames(dp, warp_buf_.as<uint8_t>(), static_cast<int64_t>(fb), id, w_, h_, ch_, S_, st);
  run_(warp_ptrs_.as<const uint8_t*>(), st, false, slot_ev_[slot]);
}

void Streams::step_device(const uint8_t* const* frames, cudaStream_t st) {
  if (!st) st = own_;
  check_sticky_errors();
  if (mc_.warp == 1) throw Error(TRB_INVALID_ARGUMENT, "warp mode homography requires per-frame homographies");
  frames_aligned_ = true;  // caller frames at any offset: misaligned ones take the scalar path
  for (int s = 0; s < S_; ++s) {
    if (!frames[s]) throw Error(TRB_INVALID_ARGUMENT, "null frame pointer for stream " + std::to_string(s));
    if (reinterpret_cast<uintptr_t>(frames[s]) & 15) frames_aligned_ = false;
  }
  const int slot = ptr_slot_;
  const uint8_t* const* dp = upload_ptrs_(frames, st);
  run_(dp, st, overlap_, slot_ev_[slot]);
}

namespace {
struct ResultCopy {
  const int32_t* src;
  int32_t* dst;
  size_t bytes;
};
void CUDART_CB copy_result(void* p) {
  auto* r = static_cast<ResultCopy*>(p);
  std::memcpy(r->dst, r->src, r->bytes);
  delete r;
}
}  // namespace

bool is_pinned_host(const void* p) { return pinned_device_alias(p) != nullptr || pinned_unmapped(p); }

// Pinned host memory's device-side address (UVA: normally the same pointer),
// or nullptr when `p` is not pinned host memory or not mapped for the device.
void* pinned_device_alias(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

bool pinned_unmapped(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && !a.devicePointer;
}

void Streams::check_sticky_errors() {
  const int32_t e = tracker_ ? tracker_->host_errors() : 0;  // the gate kernel's stores (mapped memory)
  if (e & 1) throw Error(TRB_CAPACITY, "tracker: track capacity exceeded (raise trb_streams_options.track_cap)");
  if (e & 2)
    throw Error(TRB_CAPACITY,
                "tracker: track-log ring full (drain it with trb_streams_drain_log or raise trb_streams_options.log_cap)");
}

// The step's results packed on the device (blob counts, the first blob_cap
// blobs, the frame's log entries) and copied to the caller's host buffers on
// the stream of the step's last reader.
void Streams::output_(const trb_step_output* out, cudaStream_t rs, int* launches) {
  const int bcap = out->blobs ? std::max(0, out->blob_cap) : 0;
  const int lcap = (out->log && tracker_) ? std::max(0, out->log_cap) : 0;
  const size_t hdr = sizeof(int32_t) * 2 * S_;
  const size_t bbytes = sizeof(trb_blob) * static_cast<size_t>(S_) * bcap;
  const size_t lbytes = sizeof(trb_track_log_entry) * static_cast<size_t>(S_) * lcap;
  if (bcap != out_bcap_ || lcap != out_lcap_) {
    TRB_CUDA(cudaStreamSynchronize(rs));
    out_dev_.alloc(hdr + bbytes + lbytes + 16, false);
    out_bcap_ = bcap, out_lcap_ = lcap;
  }
  char* base = out_dev_.as<char>();
  int32_t* nb = reinterpret_cast<int32_t*>(base);
  int32_t* nl = nb + S_;
  trb_blob* bl = reinterpret_cast<trb_blob*>(base + hdr);
  trb_track_log_entry* lg = reinterpret_cast<trb_track_log_entry*>(base + hdr + bbytes);
  if (has_output_ && tracker_ && direct_out_) {
    // the pack kernel stores straight into the caller's pinned buffers
    // (their device aliases): no copy launches on the step's chain
    void* d[4] = {nullptr, nullptr, nullptr, nullptr};
    const void* h[4] = {out->n_blobs, out->n_log, bcap ? out->blobs : nullptr, lcap ? out->log : nullptr};
    bool ok = true;
    for (int i = 0; i < 4 && ok; ++i)
      if (h[i]) ok = (d[i] = pinned_device_alias(h[i])) != nullptr;
    if (ok) {
      tracker_->pack_step(ccl_->blobs(), ccl_->blob_cap(), ccl_->nblobs(), d[0] ? static_cast<int32_t*>(d[0]) : nb,
                          d[2] ? static_cast<trb_blob*>(d[2]) : bl, bcap, d[1] ? static_cast<int32_t*>(d[1]) : nl,
                          d[3] ? static_cast<trb_track_log_entry*>(d[3]) : lg, lcap, rs);
      ++*launches;
      return;
    }
  }
  if (!has_output_) {
    TRB_CUDA(cudaMemsetAsync(base, 0, hdr, rs));
  } else if (tracker_) {
    tracker_->pack_step(ccl_->blobs(), ccl_->blob_cap(), ccl_->nblobs(), nb, bl, bcap, nl, lg, lcap, rs);
    ++*launches;
  } else {
    TRB_CUDA(cudaMemcpyAsync(nb, ccl_->nblobs(), sizeof(int32_t) * S_, cudaMemcpyDeviceToDevice, rs));
    TRB_CUDA(cudaMemsetAsync(nl, 0, sizeof(int32_t) * S_, rs));
    if (bcap > 0) launch_pack_blobs(ccl_->blobs(), ccl_->blob_cap(), ccl_->nblobs(), bl, bcap, S_, rs), ++*launches;
  }
  struct Region {
    void* dst;
    const void* src;
    size_t n;
  } regs[4] = {{out->n_blobs, nb, sizeof(int32_t) * S_}, {out->n_log, nl, sizeof(int32_t) * S_},
               {out->blobs, bl, bbytes}, {out->log, lg, lbytes}};
  for (const Region& r : regs) {
    if (!r.dst || r.n == 0) continue;
    if (is_pinned_host(r.dst)) {
      TRB_CUDA(cudaMemcpyAsync(r.dst, r.src, r.n, cudaMemcpyDeviceToHost, rs));
    } else {
      throw Error(TRB_INVALID_ARGUMENT, "trb_step_output buffers must be pinned host memory (cudaMallocHost)");
    }
  }
}

void Streams::step_host_async(const uint8_t* const* frames, int32_t* result_host, cudaStream_t st,
                              const trb_step_output* out) {
  if (!st) st = own_;
  check_sticky_errors();
  if (mc_.warp == 1) throw Error(TRB_INVALID_ARGUMENT, "warp mode homography requires per-frame homographies");
  const size_t fb = static_cast<size_t>(px_) * ch_;
  for (int s = 0; s < S_; ++s)
    if (!frames[s]) throw Error(TRB_INVALID_ARGUMENT, "null frame pointer for stream " + std::to_string(s));
  const int b = host_step_++ % kStaging;
  uint8_t* stage = staging_[b].as<uint8_t>();  // allocated with the handle (no cudaMalloc inside a step)
  frames_aligned_ = true;                       // staging planes sit at multiples of the frame size
  // the copy may start once the step kStaging back (same buffer) is done with it
  TRB_CUDA(cudaStreamWaitEvent(copy_, consumed_[b], 0));
  // one copy per run of frames that sit back to back in host memory (a
  // capture ring or a batched decoder hands them over that way): fewer,
  // larger DMA transfers
  for (int s = 0; s < S_;) {
    int e = s + 1;
    while (e < S_ && frames[e] == frames[e - 1] + fb) ++e;
    TRB_CUDA(cudaMemcpyAsync(stage + fb * s, frames[s], fb * (e - s), cudaMemcpyHostToDevice, copy_));
    s = e;
  }
  TRB_CUDA(cudaEventRecord(copied_[b], copy_));
  const uint8_t* const* dp = staging_ptrs_.as<const uint8_t*>() + static_cast<size_t>(b) * S_;
  TRB_CUDA(cudaStreamWaitEvent(st, copied_[b], 0));
  pending_out_ = out;
  cudaStream_t last_reader;
  try {
    last_reader = run_(dp, st, overlap_, nullptr);  // (staging reuse: consumed_[b] below)
  } catch (...) {
    pending_out_ = nullptr;
    throw;
  }
  pending_out_ = nullptr;
  TRB_CUDA(cudaEventRecord(consumed_[b], last_reader));  // tracking read the frames too
  if (result_host) {
    const size_t rb = sizeof(int32_t) * S_;
    if (!has_output_) {
      TRB_CUDA(cudaMemsetAsync(ccl_->nblobs(), 0, rb, st));
    }
    if (is_pinned_host(result_host)) {
      TRB_CUDA(cudaMemcpyAsync(result_host, ccl_->nblobs(), rb, cudaMemcpyDeviceToHost, st));
    } else {  // pageable: through a pinned buffer, copied out when the stream gets there
      if (!result_pinned_.p) result_pinned_.alloc(rb);
      TRB_CUDA(cudaMemcpyAsync(result_pinned_.p, ccl_->nblobs(), rb, cudaMemcpyDeviceToHost, st));
      TRB_CUDA(cudaLaunchHostFunc(st, copy_result,
                                  new ResultCopy{static_cast<const int32_t*>(result_pinned_.p), result_host, rb}));
    }
  }
}

void Streams::step_host(const uint8_t* const* frames, int32_t* result_host, cudaStream_t st) {
  if (!st) st = own_;
  step_host_async(frames, result_host, st);
  TRB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace trb
