// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/teamrec/*.hpp, compiled in place with
// -I; no reference source is copied into this repo).  Built by
// oracle/Makefile into oracle/_ref/libteamrec_ref.so, which travels to the
// GPU box with the snapshot.  Used to (a) pin the C restatement
// (oracle/trb_oracle.c) against the reference itself and (b) time the
// reference CPU path for bench.py's cpu_baseline / --impl reference arm.
//
// Flags (oracle/Makefile): -O2 -std=c++20 -ffp-contract=off, default x86-64
// target — SURVEY §0.6: -march=native / FMA contraction changes the
// reference's tracker output.
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "teamrec/motion.hpp"
#include "teamrec/segmentation.hpp"
#include "teamrec/synth.hpp"
#include "teamrec/tracking.hpp"
#include "../include/trb.h"
#include "plane_hash.h"

using namespace teamrec;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return TRB_CONFIG_ERROR;
  if (dynamic_cast<const InvalidArgument*>(&e)) return TRB_INVALID_ARGUMENT;
  if (dynamic_cast<const IoError*>(&e)) return TRB_IO_ERROR;
  return TRB_INVALID_ARGUMENT;
}

MotionConfig to_motion(const trb_motion_config* c) {
  MotionConfig m;
  m.method = c->method == TRB_BG_MODE ? BackgroundMethod::Mode : BackgroundMethod::Mean;
  m.window = c->window;
  m.threshold = c->threshold;
  m.bins = c->bins;
  m.warp = c->warp == 1 ? WarpMode::PerFrameHomography : WarpMode::Identity;
  return m;
}

SegmentationConfig to_seg(const trb_seg_config* c) {
  SegmentationConfig s;
  s.n_blocks = c->n_blocks;
  s.connectivity = c->connectivity == TRB_CONN_FOUR ? Connectivity::Four : Connectivity::Eight;
  s.min_area = c->min_area;
  return s;
}

TrackerConfig to_tracker(const trb_tracker_config* c) {
  TrackerConfig t;
  t.k_clusters = c->k_clusters;
  t.max_iters = c->max_iters;
  t.eps = c->eps;
  t.kmeans_iters = c->kmeans_iters;
  t.seed = c->seed;
  return t;
}

void put_blob(const Blob& b, trb_blob* o) {
  o->label = b.label;
  o->area = b.area;
  o->x_min = b.x_min;
  o->y_min = b.y_min;
  o->x_max = b.x_max;
  o->y_max = b.y_max;
  o->cx = b.cx;
  o->cy = b.cy;
}

Blob get_blob(const trb_blob& b) {
  Blob o;
  o.label = b.label;
  o.area = b.area;
  o.x_min = b.x_min;
  o.y_min = b.y_min;
  o.x_max = b.x_max;
  o.y_max = b.y_max;
  o.cx = b.cx;
  o.cy = b.cy;
  return o;
}

Frame make_frame(const uint8_t* data, int w, int h, int c, int64_t index = 0) {
  Frame f;
  f.width = w;
  f.height = h;
  f.channels = c;
  f.index = index;
  f.data.assign(data, data + static_cast<std::size_t>(w) * h * c);
  return f;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- MotionDetector ----
void* ref_motion_create(const trb_motion_config* c, int w, int h) {
  try {
    return new MotionDetector(to_motion(c), w, h);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_motion_destroy(void* m) { delete static_cast<MotionDetector*>(m); }
int ref_motion_push(void* m, const uint8_t* gray, int w, int h, int c, int64_t index, uint8_t* mask_out,
                    int* has_mask) {
  try {
    auto r = static_cast<MotionDetector*>(m)->push(make_frame(gray, w, h, c, index));
    *has_mask = r.has_value();
    if (r) std::memcpy(mask_out, r->bits.data(), r->bits.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_motion_background(void* m, uint8_t* out) {
  try {
    const Frame bg = static_cast<MotionDetector*>(m)->background();
    std::memcpy(out, bg.data.data(), bg.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- label_blocked / label_sequential ----
int ref_label(const uint8_t* mask, int w, int h, const trb_seg_config* c, int sequential, int workers,
              int32_t* labels_out, trb_blob* blobs_out, int cap, int* n, int64_t* pixels_out) {
  try {
    BinaryMask m = BinaryMask::make(w, h);
    std::memcpy(m.bits.data(), mask, m.bits.size());
    const Backend be = workers > 1 ? Backend::parallel(workers) : Backend::sequential();
    const Labeling lab = sequential ? label_sequential(m, to_seg(c)) : label_blocked(m, to_seg(c), be);
    if (labels_out) std::memcpy(labels_out, lab.labels.data(), lab.labels.size() * sizeof(int32_t));
    *n = static_cast<int>(lab.blobs.size());
    std::size_t off = 0;
    for (std::size_t i = 0; i < lab.blobs.size(); ++i) {
      if (blobs_out && static_cast<int>(i) < cap) put_blob(lab.blobs[i], &blobs_out[i]);
      if (pixels_out)
        for (auto p : lab.blobs[i].pixels) pixels_out[off++] = p;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- warp_frame / stream_detect (motion.hpp:81-119, :260-282) ----
static Homography to_hom(const double* h9) {
  Homography hm;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) hm.h[r][c] = h9[3 * r + c];
  return hm;
}
int ref_warp_frame(const uint8_t* in, int w, int h, int ch, const double* h9, uint8_t* out) {
  try {
    const Frame o = warp_frame(make_frame(in, w, h, ch), to_hom(h9));
    std::memcpy(out, o.data.data(), o.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
// frames: n * w*h*ch bytes; h9s: n * 9 (NULL = no warp); masks_out: (n - W + 1) * w*h
int ref_stream_detect(const uint8_t* frames, int n, int w, int h, int ch, const double* h9s,
                      const trb_motion_config* c, uint8_t* masks_out, int* n_masks) {
  try {
    std::vector<Frame> fr;
    const std::size_t fb = static_cast<std::size_t>(w) * h * ch;
    for (int i = 0; i < n; ++i) fr.push_back(make_frame(frames + fb * i, w, h, ch, i));
    std::vector<Homography> hs;
    if (h9s)
      for (int i = 0; i < n; ++i) hs.push_back(to_hom(h9s + 9 * i));
    const auto masks = stream_detect(fr, h9s ? &hs : nullptr, to_motion(c));
    *n_masks = static_cast<int>(masks.size());
    for (std::size_t i = 0; i < masks.size(); ++i)
      std::memcpy(masks_out + static_cast<std::size_t>(w) * h * i, masks[i].bits.data(), masks[i].bits.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- PNM ingest / track-log interchange (frame.hpp:152-225, tracking.hpp:247-285) ----
int ref_decode_pnm(const uint8_t* bytes, int64_t n, const char* src, int* w, int* h, int* ch, uint8_t* out,
                   int64_t cap) {
  try {
    const Frame f = decode_pnm(std::vector<std::uint8_t>(bytes, bytes + n), src);
    *w = f.width, *h = f.height, *ch = f.channels;
    if (out && static_cast<int64_t>(f.data.size()) <= cap) std::memcpy(out, f.data.data(), f.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_load_frame_sequence(const char* dir, int* n, int* w, int* h, int* ch, int64_t* idx, uint8_t* out,
                            int64_t cap) {
  try {
    const auto fr = load_frame_sequence(dir);
    *n = static_cast<int>(fr.size());
    *w = fr.empty() ? 0 : fr[0].width, *h = fr.empty() ? 0 : fr[0].height, *ch = fr.empty() ? 0 : fr[0].channels;
    int64_t off = 0;
    for (std::size_t i = 0; i < fr.size(); ++i) {
      if (idx) idx[i] = fr[i].index;
      if (out && off + static_cast<int64_t>(fr[i].data.size()) <= cap)
        std::memcpy(out + off, fr[i].data.data(), fr[i].data.size());
      off += static_cast<int64_t>(fr[i].data.size());
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
static TrackLogEntry to_entry(const trb_track_log_entry& e) {
  TrackLogEntry t;
  t.frame = e.frame, t.track_id = e.track_id, t.x = e.x, t.y = e.y, t.w = e.w, t.h = e.h;
  t.status = e.status == 0 ? TrackStatus::Active : TrackStatus::Lost;
  return t;
}
int64_t ref_format_track_log(const trb_track_log_entry* log, int64_t n, char* out, int64_t cap) {
  std::vector<TrackLogEntry> v;
  for (int64_t i = 0; i < n; ++i) v.push_back(to_entry(log[i]));
  const std::string s = format_track_log(v);
  if (out && static_cast<int64_t>(s.size()) < cap) std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int64_t>(s.size());
}
int ref_parse_track_log(const char* text, int64_t len, const char* src, trb_track_log_entry* out, int64_t cap,
                        int64_t* n) {
  try {
    const auto v = parse_track_log(std::string(text, static_cast<std::size_t>(len)), src);
    *n = static_cast<int64_t>(v.size());
    for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) {
      out[i].frame = v[i].frame, out[i].track_id = v[i].track_id, out[i].x = v[i].x, out[i].y = v[i].y;
      out[i].w = v[i].w, out[i].h = v[i].h, out[i].status = v[i].status == TrackStatus::Active ? 0 : 1;
      out[i]._pad = 0;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- extract_blob_features (segmentation.hpp:268-291) ----
// The labelling is rebuilt from the label image + blob records (the
// function reads only labels, width/height and the blob table).
int ref_blob_features(const int32_t* labels, int w, int h, const uint8_t* frame, int fw, int fh, int ch,
                      const trb_blob* blobs, int n, double* mean, double* aspect) {
  try {
    Labeling lab;
    lab.width = w;
    lab.height = h;
    lab.labels.assign(labels, labels + static_cast<std::size_t>(w) * h);
    lab.blobs.resize(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      Blob& b = lab.blobs[static_cast<std::size_t>(i)];
      b.label = blobs[i].label, b.area = blobs[i].area;
      b.x_min = blobs[i].x_min, b.y_min = blobs[i].y_min, b.x_max = blobs[i].x_max, b.y_max = blobs[i].y_max;
      b.cx = blobs[i].cx, b.cy = blobs[i].cy;
    }
    const auto out = extract_blob_features(lab, make_frame(frame, fw, fh, ch));
    for (int i = 0; i < n; ++i) mean[i] = out[i].mean_intensity, aspect[i] = out[i].aspect;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- quantizer / histogram / meanshift ----
int ref_quantize_colors(const double* px, int64_t n, int k, int iters, uint64_t seed, double* centers) {
  try {
    std::vector<std::array<double, 3>> v(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = {px[3 * i], px[3 * i + 1], px[3 * i + 2]};
    const ColorQuantizer q = quantize_colors(v, k, iters, seed);
    for (int c = 0; c < k; ++c)
      for (int j = 0; j < 3; ++j) centers[3 * c + j] = q.centers[c][j];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_histogram(const uint8_t* frame, int fw, int fh, int ch, double cx, double cy, int w, int h,
                  const double* centers, int k, int epan, double* hist) {
  ColorQuantizer q;
  for (int c = 0; c < k; ++c) q.centers.push_back({centers[3 * c], centers[3 * c + 1], centers[3 * c + 2]});
  const Frame f = make_frame(frame, fw, fh, ch);
  auto r = detail::histogram_opt(f, cx, cy, w, h, q, epan ? HistKernel::Epanechnikov : HistKernel::Uniform);
  if (!r) return 0;
  for (int i = 0; i < k; ++i) hist[i] = (*r)[i];
  return 1;
}

void ref_meanshift_step(const uint8_t* frame, int fw, int fh, int ch, double* cx, double* cy, int w, int h,
                        const double* centers, const double* target, int k, int max_iters, double eps,
                        int* status) {
  Track t;
  t.cx = *cx;
  t.cy = *cy;
  t.w = w;
  t.h = h;
  for (int c = 0; c < k; ++c) t.quantizer.centers.push_back({centers[3 * c], centers[3 * c + 1], centers[3 * c + 2]});
  t.target_hist.assign(target, target + k);
  t.status = *status == TRB_TRACK_LOST ? TrackStatus::Lost : TrackStatus::Active;
  TrackerConfig cfg;
  cfg.max_iters = max_iters;
  cfg.eps = eps;
  meanshift_step(make_frame(frame, fw, fh, ch), t, cfg);
  *cx = t.cx;
  *cy = t.cy;
  *status = t.status == TrackStatus::Lost ? TRB_TRACK_LOST : TRB_TRACK_ACTIVE;
}

// ---- Tracker ----
void* ref_tracker_create(const trb_tracker_config* c) {
  try {
    return new Tracker(to_tracker(c));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void ref_tracker_destroy(void* t) { delete static_cast<Tracker*>(t); }
int ref_tracker_process(void* t, const uint8_t* frame, int w, int h, int c, const trb_blob* blobs, int n) {
  try {
    std::vector<Blob> bl;
    for (int i = 0; i < n; ++i) bl.push_back(get_blob(blobs[i]));
    static_cast<Tracker*>(t)->process(make_frame(frame, w, h, c), bl);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_tracker_num_tracks(void* t) { return static_cast<int>(static_cast<Tracker*>(t)->tracks().size()); }
void ref_tracker_tracks(void* t, trb_track* out) {
  const auto& tr = static_cast<Tracker*>(t)->tracks();
  for (std::size_t i = 0; i < tr.size(); ++i) {
    std::memset(&out[i], 0, sizeof(trb_track));
    out[i].track_id = tr[i].track_id;
    out[i].w = tr[i].w;
    out[i].h = tr[i].h;
    out[i].status = tr[i].status == TrackStatus::Lost ? TRB_TRACK_LOST : TRB_TRACK_ACTIVE;
    out[i].lost_frames = tr[i].lost_frames;
    out[i].k = tr[i].quantizer.k();
    out[i].cx = tr[i].cx;
    out[i].cy = tr[i].cy;
  }
}
void ref_tracker_track_model(void* t, int i, double* centers, double* hist) {
  const auto& tr = static_cast<Tracker*>(t)->tracks()[static_cast<std::size_t>(i)];
  for (int c = 0; c < tr.quantizer.k(); ++c)
    for (int j = 0; j < 3; ++j) centers[3 * c + j] = tr.quantizer.centers[c][j];
  for (std::size_t b = 0; b < tr.target_hist.size(); ++b) hist[b] = tr.target_hist[b];
}
int64_t ref_tracker_log_size(void* t) { return static_cast<int64_t>(static_cast<Tracker*>(t)->log().size()); }
void ref_tracker_log(void* t, trb_track_log_entry* out) {
  const auto& log = static_cast<Tracker*>(t)->log();
  for (std::size_t i = 0; i < log.size(); ++i) {
    std::memset(&out[i], 0, sizeof(trb_track_log_entry));
    out[i].frame = log[i].frame;
    out[i].track_id = log[i].track_id;
    out[i].x = log[i].x;
    out[i].y = log[i].y;
    out[i].w = log[i].w;
    out[i].h = log[i].h;
    out[i].status = log[i].status == TrackStatus::Lost ? TRB_TRACK_LOST : TRB_TRACK_ACTIVE;
  }
}

// ---- synth_frames (synth.hpp:45-101) ----
// shape_int: n*{w,h,c0,c1,c2}; shape_dbl: n*{x0,y0,vx,vy,jitter}.  Writes
// n_frames frames (frames_out, n_frames*w*h*ch) and rects (n_frames*n*4).
int ref_synth(int w, int h, int ch, uint8_t bg, int n, const int32_t* si, const double* sd, int n_frames,
              uint64_t seed, uint8_t* frames_out, int32_t* rects_out) {
  try {
    ClipSpec spec;
    spec.width = w;
    spec.height = h;
    spec.channels = ch;
    spec.background = bg;
    for (int k = 0; k < n; ++k) {
      ShapeSpec s;
      s.width = si[5 * k];
      s.height = si[5 * k + 1];
      s.color = {static_cast<uint8_t>(si[5 * k + 2]), static_cast<uint8_t>(si[5 * k + 3]),
                 static_cast<uint8_t>(si[5 * k + 4])};
      s.x0 = sd[5 * k];
      s.y0 = sd[5 * k + 1];
      s.vx = sd[5 * k + 2];
      s.vy = sd[5 * k + 3];
      s.jitter_sigma = sd[5 * k + 4];
      spec.shapes.push_back(s);
    }
    const SynthClip clip = synth_frames(spec, n_frames, seed);
    const std::size_t fb = static_cast<std::size_t>(w) * h * ch;
    for (int t = 0; t < n_frames; ++t) {
      if (frames_out) std::memcpy(frames_out + fb * t, clip.frames[t].data.data(), fb);
      if (rects_out)
        for (int k = 0; k < n; ++k) {
          // centers = ix + (w-1)/2 -> recover ix exactly (synth.hpp:329)
          const auto& c = clip.centers[t][k];
          rects_out[(static_cast<std::size_t>(t) * n + k) * 4 + 0] = static_cast<int32_t>(c[0] - (si[5 * k] - 1) / 2.0);
          rects_out[(static_cast<std::size_t>(t) * n + k) * 4 + 1] =
              static_cast<int32_t>(c[1] - (si[5 * k + 1] - 1) / 2.0);
          rects_out[(static_cast<std::size_t>(t) * n + k) * 4 + 2] = si[5 * k];
          rects_out[(static_cast<std::size_t>(t) * n + k) * 4 + 3] = si[5 * k + 1];
        }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- stepwise multi-stream reference loop (bench.py --impl reference) ----
// Each step advances every stream by one frame: push -> label_blocked
// (sequential backend) -> Tracker::process, streams spread over `threads`
// host threads.  Returns the number of frames that produced a mask.
struct RefStreams {
  int n, w, h, ch;
  std::vector<std::unique_ptr<MotionDetector>> det;
  std::vector<std::unique_ptr<Tracker>> trk;
  SegmentationConfig seg;
  std::vector<int64_t> digest;
};

void* ref_streams_create(int n, int w, int h, int ch, const trb_motion_config* mc, const trb_seg_config* sc,
                         const trb_tracker_config* tc) {
  try {
    auto* r = new RefStreams{n, w, h, ch, {}, {}, to_seg(sc), {}};
    for (int s = 0; s < n; ++s) {
      r->det.push_back(std::make_unique<MotionDetector>(to_motion(mc), w, h));
      r->trk.push_back(std::make_unique<Tracker>(to_tracker(tc)));
    }
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_streams_destroy(void* p) { delete static_cast<RefStreams*>(p); }

int64_t ref_streams_step(void* p, const uint8_t* const* frames, int threads) {
  auto* r = static_cast<RefStreams*>(p);
  std::atomic<int> next{0};
  std::atomic<int64_t> steady{0};
  auto worker = [&]() {
    for (;;) {
      const int s = next.fetch_add(1);
      if (s >= r->n) return;
      Frame f = make_frame(frames[s], r->w, r->h, r->ch);
      auto mask = r->det[s]->push(r->ch == 1 ? f : grayscale(f));
      if (!mask) continue;
      const Labeling lab = label_blocked(*mask, r->seg, Backend::sequential());
      r->trk[s]->process(f, lab.blobs, Backend::sequential());
      steady.fetch_add(1);
    }
  };
  const int nt = std::max(1, std::min(threads, r->n));
  std::vector<std::thread> pool;
  for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  return steady.load();
}

// ---- the reference per-frame loop, used as the CPU baseline ----
// Runs push -> label_blocked(sequential backend) -> Tracker::process over
// n_frames frames of each of n_streams streams (frames[s] = n_frames*w*h*ch
// bytes), one std::thread per stream slot up to `threads`.  Frames before
// the window fills are pushed but not counted.  Returns per-stream
// steady-frame counts in steady_out and total seconds spent in the steady
// frames (summed over streams) in *busy_s; *wall_s is the wall time.
// digest_out (n_streams u64, nullable) receives an FNV-1a over masks,
// labels and the track log so runs can be compared.
int ref_run_streams(int n_streams, int threads, int w, int h, int ch, const uint8_t* const* frames, int n_frames,
                    const trb_motion_config* mc, const trb_seg_config* sc, const trb_tracker_config* tc,
                    int64_t* steady_out, double* wall_s, uint64_t* digest_out, double* stage_s /* 3 */) {
  try {
    std::atomic<int> next{0};
    std::vector<double> st(3 * static_cast<std::size_t>(n_streams), 0.0);
    auto worker = [&]() {
      for (;;) {
        const int s = next.fetch_add(1);
        if (s >= n_streams) return;
        MotionDetector det(to_motion(mc), w, h);
        Tracker tracker(to_tracker(tc));
        const SegmentationConfig seg = to_seg(sc);
        uint64_t hsh = 1469598103934665603ULL;
        auto mix = [&](const void* p, std::size_t n) {
          const auto* b = static_cast<const uint8_t*>(p);
          for (std::size_t i = 0; i < n; ++i) hsh = (hsh ^ b[i]) * 1099511628211ULL;
        };
        int64_t steady = 0;
        const std::size_t fb = static_cast<std::size_t>(w) * h * ch;
        for (int t = 0; t < n_frames; ++t) {
          Frame f = make_frame(frames[s] + fb * t, w, h, ch, t);
          auto t0 = std::chrono::steady_clock::now();
          auto mask = det.push(ch == 1 ? f : grayscale(f));
          auto t1 = std::chrono::steady_clock::now();
          if (!mask) continue;
          const Labeling lab = label_blocked(*mask, seg, Backend::sequential());
          auto t2 = std::chrono::steady_clock::now();
          tracker.process(f, lab.blobs, Backend::sequential());
          auto t3 = std::chrono::steady_clock::now();
          st[3 * s] += std::chrono::duration<double>(t1 - t0).count();
          st[3 * s + 1] += std::chrono::duration<double>(t2 - t1).count();
          st[3 * s + 2] += std::chrono::duration<double>(t3 - t2).count();
          ++steady;
          if (digest_out) {
            mix(mask->bits.data(), mask->bits.size());
            mix(lab.labels.data(), lab.labels.size() * sizeof(int));
          }
        }
        if (digest_out) {
          for (const auto& e : tracker.log()) {
            mix(&e.frame, sizeof(int));
            mix(&e.track_id, sizeof(int));
            mix(&e.x, sizeof(double));
            mix(&e.y, sizeof(double));
            mix(&e.w, sizeof(int));
            mix(&e.h, sizeof(int));
            const int stv = e.status == TrackStatus::Lost;
            mix(&stv, sizeof(int));
          }
          digest_out[s] = hsh;
        }
        steady_out[s] = steady;
      }
    };
    const auto w0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    const int nt = threads < 1 ? 1 : threads;
    for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    if (stage_s) {
      stage_s[0] = stage_s[1] = stage_s[2] = 0.0;
      for (int s = 0; s < n_streams; ++s)
        for (int j = 0; j < 3; ++j) stage_s[j] += st[3 * s + j];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- per-frame detail of the reference per-frame loop (parity tests) ----
// Same loop as ref_run_streams.  For stream s and steady frame k (frames
// with a mask, counted from 0): hashes[(s*n_frames + k)*2 + {0,1}] =
// plane_hash of the mask bytes / the int32 label image, nblobs[s*n_frames+k]
// = blob count, blobs[(s*n_frames + k)*bcap + i] = the first bcap blobs.
// The whole track log goes to logs[s*lcap + i] (first lcap), its length to
// nlog[s].  steady[s] = steady frames.
int ref_run_streams_detail(int n_streams, int threads, int w, int h, int ch, const uint8_t* const* frames,
                           int n_frames, const trb_motion_config* mc, const trb_seg_config* sc,
                           const trb_tracker_config* tc, int64_t* steady, uint64_t* hashes, int32_t* nblobs,
                           trb_blob* blobs, int bcap, trb_track_log_entry* logs, int64_t lcap, int64_t* nlog) {
  std::atomic<int> next{0};
  std::atomic<int> failed{0};
  std::string err;
  auto worker = [&]() {
    try {
      for (;;) {
        const int s = next.fetch_add(1);
        if (s >= n_streams) return;
        MotionDetector det(to_motion(mc), w, h);
        Tracker tracker(to_tracker(tc));
        const SegmentationConfig seg = to_seg(sc);
        const std::size_t fb = static_cast<std::size_t>(w) * h * ch;
        int64_t k = 0;
        for (int t = 0; t < n_frames; ++t) {
          Frame f = make_frame(frames[s] + fb * t, w, h, ch, t);
          auto mask = det.push(ch == 1 ? f : grayscale(f));
          if (!mask) continue;
          const Labeling lab = label_blocked(*mask, seg, Backend::sequential());
          tracker.process(f, lab.blobs, Backend::sequential());
          const int64_t row = static_cast<int64_t>(s) * n_frames + k;
          hashes[2 * row] = trb_plane_hash(mask->bits.data(), static_cast<int64_t>(mask->bits.size()));
          hashes[2 * row + 1] =
              trb_plane_hash(lab.labels.data(), static_cast<int64_t>(lab.labels.size() * sizeof(int)));
          nblobs[row] = static_cast<int32_t>(lab.blobs.size());
          for (int i = 0; i < bcap && i < static_cast<int>(lab.blobs.size()); ++i)
            put_blob(lab.blobs[i], blobs + row * bcap + i);
          ++k;
        }
        steady[s] = k;
        const auto& log = tracker.log();
        nlog[s] = static_cast<int64_t>(log.size());
        for (int64_t i = 0; i < lcap && i < static_cast<int64_t>(log.size()); ++i) {
          trb_track_log_entry& o = logs[static_cast<int64_t>(s) * lcap + i];
          std::memset(&o, 0, sizeof(o));
          o.frame = log[i].frame;
          o.track_id = log[i].track_id;
          o.x = log[i].x;
          o.y = log[i].y;
          o.w = log[i].w;
          o.h = log[i].h;
          o.status = log[i].status == TrackStatus::Lost ? TRB_TRACK_LOST : TRB_TRACK_ACTIVE;
        }
      }
    } catch (const std::exception& e) {
      if (failed.fetch_add(1) == 0) err = e.what();
    }
  };
  std::vector<std::thread> pool;
  const int nt = std::max(1, std::min(threads, n_streams));
  for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  if (failed.load()) {
    g_err = err;
    return TRB_INVALID_ARGUMENT;
  }
  return 0;
}

}  // extern "C"
