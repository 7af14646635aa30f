// teamrec_b200.hpp — the reference's C++ API for the video front end, served
// by the B200 library (include/trb.h, libtrb.so).
//
// Header-only C++ over the C ABI.  It includes the reference's own headers
// for the value types (Frame, BinaryMask, Blob, Labeling, Track, the config
// structs and exception classes), so results are the reference's types and
// failures its exception classes with its messages:
//
//   teamrec_b200::MotionDetector      motion.hpp:149-212   (trb_motion_*)
//   teamrec_b200::background_model    motion.hpp:216-238
//   teamrec_b200::warp_frame          motion.hpp:81-119    (trb_warp_frame)
//   teamrec_b200::stream_detect       motion.hpp:260-282
//   teamrec_b200::detect_motion       motion.hpp:285-287   (frame-sequence overload)
//   teamrec_b200::label_blocked       segmentation.hpp:198-264 (trb_label)
//   teamrec_b200::label_sequential    segmentation.hpp:183-191
//   teamrec_b200::extract_blob_features segmentation.hpp:268-291
//   teamrec_b200::quantize_colors     quantize.hpp:43-118  (trb_quantize_colors)
//   teamrec_b200::histogram           tracking.hpp:106-112 (trb_histogram)
//   teamrec_b200::meanshift_step      tracking.hpp:125-157 (trb_meanshift_step)
//   teamrec_b200::Tracker             tracking.hpp:170-241 (trb_tracker_*)
//
// Every call computes on the device (no CPU fallback: without an sm_100
// device the calls throw teamrec::Error with the CUDA message).  The Backend
// arguments are accepted for signature compatibility; the device decides
// its own parallelism.  teamrec_b200/redirect.hpp makes unmodified reference
// code (its tests, run_vision) call these instead of the CPU versions.
//
// Build: -I<repo>/include -I<reference>/proj/include, link
// <repo>/paper_1310_3322_b200/libtrb.so.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "teamrec/error.hpp"
#include "teamrec/frame.hpp"
#include "teamrec/motion.hpp"
#include "teamrec/parallel.hpp"
#include "teamrec/quantize.hpp"
#include "teamrec/segmentation.hpp"
#include "teamrec/tracking.hpp"
#include "trb.h"

namespace teamrec_b200 {

// device used by objects created from here on (default 0)
inline int& default_device() {
  static int d = 0;
  return d;
}

// trb_status -> the reference's exception class, message from trb_last_error()
[[noreturn]] inline void raise_status(int rc) {
  const std::string m = trb_last_error();
  switch (rc) {
    case TRB_INVALID_ARGUMENT:
      throw teamrec::InvalidArgument(m);
    case TRB_CONFIG_ERROR:
      throw teamrec::ConfigError(m);
    case TRB_IO_ERROR:
      throw teamrec::IoError(m);
    default:
      throw teamrec::Error("trb: " + m);
  }
}
inline void check(int rc) {
  if (rc != TRB_OK) raise_status(rc);
}

inline trb_motion_config to_c(const teamrec::MotionConfig& c) {
  trb_motion_config o{};
  o.method = c.method == teamrec::BackgroundMethod::Mode ? TRB_BG_MODE : TRB_BG_MEAN;
  o.window = c.window;
  o.threshold = c.threshold;
  o.bins = c.bins;
  o.warp = c.warp == teamrec::WarpMode::PerFrameHomography ? 1 : 0;
  o.morph = TRB_MORPH_NONE;
  return o;
}
inline trb_seg_config to_c(const teamrec::SegmentationConfig& c) {
  return trb_seg_config{c.n_blocks, c.connectivity == teamrec::Connectivity::Four ? TRB_CONN_FOUR : TRB_CONN_EIGHT,
                        c.min_area};
}
inline trb_tracker_config to_c(const teamrec::TrackerConfig& c) {
  trb_tracker_config o{};
  o.k_clusters = c.k_clusters;
  o.max_iters = c.max_iters;
  o.eps = c.eps;
  o.kmeans_iters = c.kmeans_iters;
  o.seed = c.seed;
  return o;
}
inline trb_blob to_c(const teamrec::Blob& b) {
  return trb_blob{b.label, b.area, b.x_min, b.y_min, b.x_max, b.y_max, b.cx, b.cy};
}
inline teamrec::Blob from_c(const trb_blob& b) {
  teamrec::Blob o;
  o.label = b.label, o.area = b.area, o.x_min = b.x_min, o.y_min = b.y_min, o.x_max = b.x_max, o.y_max = b.y_max;
  o.cx = b.cx, o.cy = b.cy;
  return o;
}
inline std::vector<double> centers_flat(const teamrec::ColorQuantizer& q) {
  std::vector<double> c;
  c.reserve(q.centers.size() * 3);
  for (const auto& v : q.centers) c.insert(c.end(), v.begin(), v.end());
  return c;
}

// ------------------------------------------------------------ motion
class MotionDetector {  // motion.hpp:149-212
 public:
  MotionDetector(teamrec::MotionConfig cfg, int width, int height) : cfg_(cfg), w_(width), h_(height) {
    const trb_motion_config c = to_c(cfg);
    trb_motion* m = nullptr;
    check(trb_motion_create(&c, width, height, default_device(), &m));
    m_.reset(m, Del{});
  }
  int width() const { return w_; }
  int height() const { return h_; }
  int frames_seen() const {
    int n = 0;
    check(trb_motion_frames_seen(m_.get(), &n));
    return n;
  }
  const teamrec::MotionConfig& config() const { return cfg_; }

  std::optional<teamrec::BinaryMask> push(const teamrec::Frame& gray) {
    teamrec::BinaryMask mask = teamrec::BinaryMask::make(w_, h_);
    int has = 0;
    check(trb_motion_push(m_.get(), gray.data.data(), gray.width, gray.height, gray.channels, gray.index,
                          mask.bits.data(), &has));
    if (!has) return std::nullopt;
    return mask;
  }

  teamrec::Frame background() const {
    teamrec::Frame bg = teamrec::Frame::make(w_, h_, 1);
    check(trb_motion_background(m_.get(), bg.data.data()));
    return bg;
  }

 private:
  struct Del {
    void operator()(trb_motion* m) const { trb_motion_destroy(m); }
  };
  teamrec::MotionConfig cfg_;
  int w_, h_;
  std::shared_ptr<trb_motion> m_;  // copies share the device detector
};

// background over an explicit window (motion.hpp:216-238): the window's
// frames (luma for colour input) pushed through a device detector
inline teamrec::Frame background_model(const std::vector<teamrec::Frame>& window, const teamrec::MotionConfig& cfg) {
  cfg.validate();
  if (static_cast<int>(window.size()) != cfg.window)
    throw teamrec::InvalidArgument("background_model expects " + std::to_string(cfg.window) + " frames, got " +
                                   std::to_string(window.size()));
  const int w = window[0].width, h = window[0].height;
  for (const teamrec::Frame& f : window)
    if (f.width != w || f.height != h)
      throw teamrec::InvalidArgument("frame " + std::to_string(f.index) + " dimensions do not match the window");
  MotionDetector det(cfg, w, h);
  for (const teamrec::Frame& f : window) det.push(f.channels == 1 ? f : teamrec::grayscale(f));
  return det.background();
}

inline teamrec::Frame warp_frame(const teamrec::Frame& f, const teamrec::Homography& hom) {  // motion.hpp:81-119
  double h9[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) h9[3 * r + c] = hom.h[r][c];
  teamrec::Frame out = teamrec::Frame::make(f.width, f.height, f.channels, 0, f.index);
  check(trb_warp_frame(f.data.data(), f.width, f.height, f.channels, h9, default_device(), out.data.data()));
  return out;
}

inline std::vector<teamrec::BinaryMask> stream_detect(const std::vector<teamrec::Frame>& frames,
                                                      const std::vector<teamrec::Homography>* homographies,
                                                      const teamrec::MotionConfig& cfg) {  // motion.hpp:260-282
  cfg.validate();
  if (frames.empty()) throw teamrec::InvalidArgument("stream_detect needs at least one frame");
  if (static_cast<int>(frames.size()) < cfg.window)
    throw teamrec::InvalidArgument("need at least " + std::to_string(cfg.window) + " frames for window, got " +
                                   std::to_string(frames.size()));
  if (homographies && homographies->size() != frames.size())
    throw teamrec::InvalidArgument("homography count " + std::to_string(homographies->size()) +
                                   " does not match frame count " + std::to_string(frames.size()));
  if (cfg.warp == teamrec::WarpMode::PerFrameHomography && !homographies)
    throw teamrec::InvalidArgument("warp mode homography requires per-frame homographies");
  MotionDetector det(cfg, frames[0].width, frames[0].height);
  std::vector<teamrec::BinaryMask> masks;
  masks.reserve(frames.size() - static_cast<std::size_t>(cfg.window) + 1);
  for (std::size_t i = 0; i < frames.size(); ++i) {
    const teamrec::Frame f = homographies ? teamrec_b200::warp_frame(frames[i], (*homographies)[i]) : frames[i];
    if (auto m = det.push(f.channels == 1 ? f : teamrec::grayscale(f))) masks.push_back(std::move(*m));
  }
  return masks;
}

inline std::vector<teamrec::BinaryMask> detect_motion(const std::vector<teamrec::Frame>& frames,
                                                      const teamrec::MotionConfig& cfg) {  // motion.hpp:285-287
  return teamrec_b200::stream_detect(frames, nullptr, cfg);
}

// ------------------------------------------------------------ segmentation
inline teamrec::Labeling label_blocked(const teamrec::BinaryMask& mask, const teamrec::SegmentationConfig& cfg,
                                       const teamrec::Backend& = teamrec::Backend::sequential()) {
  const trb_seg_config c = to_c(cfg);
  teamrec::Labeling out;
  out.width = mask.width;
  out.height = mask.height;
  const std::size_t px = static_cast<std::size_t>(mask.width) * mask.height;
  out.labels.assign(px, 0);
  std::vector<trb_blob> b(px / 2 + 1);
  std::vector<int64_t> pixels(px);
  int n = 0;
  check(trb_label(mask.bits.data(), mask.width, mask.height, &c, default_device(), out.labels.data(), b.data(),
                  static_cast<int>(b.size()), &n, pixels.data(), static_cast<int64_t>(pixels.size())));
  int64_t off = 0;
  out.blobs.reserve(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    teamrec::Blob bl = from_c(b[static_cast<std::size_t>(i)]);
    bl.pixels.assign(pixels.begin() + off, pixels.begin() + off + bl.area);  // Blob::pixels, raster order
    off += bl.area;
    out.blobs.push_back(std::move(bl));
  }
  return out;
}

// label_sequential == label_blocked with one block (the output does not
// depend on n_blocks, segmentation.hpp:183-191)
inline teamrec::Labeling label_sequential(const teamrec::BinaryMask& mask, const teamrec::SegmentationConfig& cfg) {
  teamrec::SegmentationConfig one = cfg;
  one.n_blocks = 1;
  cfg.validate();
  return teamrec_b200::label_blocked(mask, one);
}

inline std::vector<teamrec::Blob> extract_blob_features(const teamrec::Labeling& lab, const teamrec::Frame& frame) {
  std::vector<trb_blob> b;
  b.reserve(lab.blobs.size());
  for (const auto& x : lab.blobs) b.push_back(to_c(x));
  std::vector<double> mean(lab.blobs.size()), aspect(lab.blobs.size());
  check(trb_extract_blob_features(lab.labels.data(), lab.width, lab.height, frame.data.data(), frame.width,
                                  frame.height, frame.channels, b.data(), static_cast<int>(b.size()),
                                  default_device(), mean.data(), aspect.data()));
  std::vector<teamrec::Blob> out = lab.blobs;
  for (std::size_t i = 0; i < out.size(); ++i) out[i].mean_intensity = mean[i], out[i].aspect = aspect[i];
  return out;
}

// ------------------------------------------------------------ tracking
inline teamrec::ColorQuantizer quantize_colors(const std::vector<std::array<double, 3>>& pixels, int k, int iters,
                                               std::uint64_t seed) {  // quantize.hpp:43-118
  if (k < 2) throw teamrec::InvalidArgument("quantize_colors needs k >= 2");
  if (iters < 1) throw teamrec::InvalidArgument("quantize_colors needs iters >= 1");
  if (pixels.size() < static_cast<std::size_t>(k))
    throw teamrec::InvalidArgument("quantize_colors: " + std::to_string(pixels.size()) +
                                   " pixels < k=" + std::to_string(k));
  std::vector<double> flat;
  flat.reserve(pixels.size() * 3);
  for (const auto& p : pixels) flat.insert(flat.end(), p.begin(), p.end());
  std::vector<double> c(static_cast<std::size_t>(3 * k));
  check(trb_quantize_colors(flat.data(), static_cast<int64_t>(pixels.size()), k, iters, seed, c.data(),
                            default_device()));
  teamrec::ColorQuantizer q;
  q.centers.resize(static_cast<std::size_t>(k));
  for (int i = 0; i < k; ++i) q.centers[i] = {c[3 * i], c[3 * i + 1], c[3 * i + 2]};
  return q;
}

inline std::vector<double> histogram(const teamrec::Frame& frame, double cx, double cy, int w, int h,
                                     const teamrec::ColorQuantizer& q,
                                     teamrec::HistKernel kernel = teamrec::HistKernel::Epanechnikov) {
  const std::vector<double> c = centers_flat(q);
  std::vector<double> out(static_cast<std::size_t>(q.k()));
  check(trb_histogram(frame.data.data(), frame.width, frame.height, frame.channels, cx, cy, w, h, c.data(), q.k(),
                      kernel == teamrec::HistKernel::Epanechnikov ? 1 : 0, out.data(), default_device()));
  return out;
}

inline void meanshift_step(const teamrec::Frame& frame, teamrec::Track& track, const teamrec::TrackerConfig& cfg) {
  if (track.status != teamrec::TrackStatus::Active) return;
  const std::vector<double> c = centers_flat(track.quantizer);
  int status = TRB_TRACK_ACTIVE;
  check(trb_meanshift_step(frame.data.data(), frame.width, frame.height, frame.channels, &track.cx, &track.cy,
                           track.w, track.h, c.data(), track.target_hist.data(), track.quantizer.k(), cfg.max_iters,
                           cfg.eps, &status, default_device()));
  track.status = status == TRB_TRACK_LOST ? teamrec::TrackStatus::Lost : teamrec::TrackStatus::Active;
}

class Tracker {  // tracking.hpp:170-241
 public:
  explicit Tracker(teamrec::TrackerConfig cfg) : cfg_(cfg) {
    const trb_tracker_config c = to_c(cfg);
    trb_tracker* t = nullptr;
    check(trb_tracker_create(&c, default_device(), &t));
    t_.reset(t, Del{});
  }
  const teamrec::TrackerConfig& config() const { return cfg_; }
  const std::vector<teamrec::Track>& tracks() const {
    refresh_();
    return tracks_;
  }
  const std::vector<teamrec::TrackLogEntry>& log() const {
    refresh_();
    return log_;
  }
  int frames_processed() const {
    int n = 0;
    check(trb_tracker_frames_processed(t_.get(), &n));
    return n;
  }
  void process(const teamrec::Frame& frame, const std::vector<teamrec::Blob>& blobs,
               const teamrec::Backend& = teamrec::Backend::sequential()) {
    std::vector<trb_blob> b;
    b.reserve(blobs.size());
    for (const auto& x : blobs) b.push_back(to_c(x));
    check(trb_tracker_process(t_.get(), frame.data.data(), frame.width, frame.height, frame.channels, b.data(),
                              static_cast<int>(b.size())));
    stale_ = true;
  }

 private:
  struct Del {
    void operator()(trb_tracker* t) const { trb_tracker_destroy(t); }
  };
  void refresh_() const {
    if (!stale_) return;
    int n = 0;
    check(trb_tracker_num_tracks(t_.get(), &n));
    std::vector<trb_track> tr(static_cast<std::size_t>(n > 0 ? n : 1));
    check(trb_tracker_tracks(t_.get(), tr.data(), n));
    tracks_.clear();
    for (int i = 0; i < n; ++i) {
      const trb_track& s = tr[static_cast<std::size_t>(i)];
      teamrec::Track t;
      t.track_id = s.track_id, t.cx = s.cx, t.cy = s.cy, t.w = s.w, t.h = s.h, t.lost_frames = s.lost_frames;
      t.status = s.status == TRB_TRACK_LOST ? teamrec::TrackStatus::Lost : teamrec::TrackStatus::Active;
      std::vector<double> c(static_cast<std::size_t>(3 * s.k)), hist(static_cast<std::size_t>(s.k));
      check(trb_tracker_track_model(t_.get(), i, c.data(), hist.data()));
      t.quantizer.centers.resize(static_cast<std::size_t>(s.k));
      for (int k = 0; k < s.k; ++k) t.quantizer.centers[k] = {c[3 * k], c[3 * k + 1], c[3 * k + 2]};
      t.target_hist = std::move(hist);
      tracks_.push_back(std::move(t));
    }
    int64_t nl = 0;
    check(trb_tracker_log_size(t_.get(), &nl));
    std::vector<trb_track_log_entry> lg(static_cast<std::size_t>(nl > 0 ? nl : 1));
    check(trb_tracker_log(t_.get(), lg.data(), nl));
    log_.clear();
    for (int64_t i = 0; i < nl; ++i) {
      const trb_track_log_entry& e = lg[static_cast<std::size_t>(i)];
      log_.push_back({e.frame, e.track_id, e.x, e.y, e.w, e.h,
                      e.status == TRB_TRACK_LOST ? teamrec::TrackStatus::Lost : teamrec::TrackStatus::Active});
    }
    stale_ = false;
  }
  teamrec::TrackerConfig cfg_;
  std::shared_ptr<trb_tracker> t_;
  mutable std::vector<teamrec::Track> tracks_;
  mutable std::vector<teamrec::TrackLogEntry> log_;
  mutable bool stale_ = true;
};

}  // namespace teamrec_b200
