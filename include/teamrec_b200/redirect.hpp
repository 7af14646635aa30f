// redirect.hpp — run UNMODIFIED reference code on the B200 library.
//
// Force-include it (g++ -include teamrec_b200/redirect.hpp) ahead of a
// reference translation unit (its unit tests, a run_vision caller): it
// parses the reference headers first (so their own definitions stay
// intact), puts the device implementations of teamrec_b200.hpp into
// namespace teamrec under gpu_ names, and then renames the hot-path
// identifiers with macros, so every later `MotionDetector`, `label_blocked`,
// `Tracker`, ... — in the test file and in headers parsed afterwards such as
// harness.hpp's run_vision (harness.hpp:412-450) — is the device version.
// harness.hpp is deliberately NOT included here: parsed after the macros,
// its run_vision pipeline stages (make_stage, pipeline.hpp:44-54) construct
// the device MotionDetector / label_blocked / Tracker.
#pragma once

#include "teamrec/config.hpp"
#include "teamrec/discretize.hpp"
#include "teamrec/evaluation.hpp"
#include "teamrec/hmm.hpp"
#include "teamrec/id3.hpp"
#include "teamrec/pipeline.hpp"
#include "teamrec/rng.hpp"
#include "teamrec/synth.hpp"
#include "teamrec/trajectory.hpp"
#include "teamrec_b200/teamrec_b200.hpp"

namespace teamrec {
using gpu_MotionDetector = teamrec_b200::MotionDetector;
using gpu_Tracker = teamrec_b200::Tracker;
inline Frame gpu_background_model(const std::vector<Frame>& w, const MotionConfig& c) {
  return teamrec_b200::background_model(w, c);
}
inline Frame gpu_warp_frame(const Frame& f, const Homography& h) { return teamrec_b200::warp_frame(f, h); }
inline std::vector<BinaryMask> gpu_stream_detect(const std::vector<Frame>& f, const std::vector<Homography>* h,
                                                 const MotionConfig& c) {
  return teamrec_b200::stream_detect(f, h, c);
}
// both detect_motion overloads: the frame-sequence one on the device, the
// single frame-vs-background threshold (motion.hpp:241-257) stays the reference's
inline std::vector<BinaryMask> gpu_detect_motion(const std::vector<Frame>& f, const MotionConfig& c) {
  return teamrec_b200::detect_motion(f, c);
}
inline BinaryMask gpu_detect_motion(const Frame& f, const Frame& bg, const MotionConfig& c) {
  return detect_motion(f, bg, c);
}
inline Labeling gpu_label_blocked(const BinaryMask& m, const SegmentationConfig& c,
                                  const Backend& b = Backend::sequential()) {
  return teamrec_b200::label_blocked(m, c, b);
}
inline Labeling gpu_label_sequential(const BinaryMask& m, const SegmentationConfig& c) {
  return teamrec_b200::label_sequential(m, c);
}
inline std::vector<Blob> gpu_extract_blob_features(const Labeling& l, const Frame& f) {
  return teamrec_b200::extract_blob_features(l, f);
}
inline ColorQuantizer gpu_quantize_colors(const std::vector<std::array<double, 3>>& p, int k, int iters,
                                          std::uint64_t seed) {
  return teamrec_b200::quantize_colors(p, k, iters, seed);
}
inline std::vector<double> gpu_histogram(const Frame& f, double cx, double cy, int w, int h, const ColorQuantizer& q,
                                         HistKernel k = HistKernel::Epanechnikov) {
  return teamrec_b200::histogram(f, cx, cy, w, h, q, k);
}
inline void gpu_meanshift_step(const Frame& f, Track& t, const TrackerConfig& c) {
  teamrec_b200::meanshift_step(f, t, c);
}
}  // namespace teamrec

#define MotionDetector gpu_MotionDetector
#define Tracker gpu_Tracker
#define background_model gpu_background_model
#define warp_frame gpu_warp_frame
#define stream_detect gpu_stream_detect
#define detect_motion gpu_detect_motion
#define label_blocked gpu_label_blocked
#define label_sequential gpu_label_sequential
#define extract_blob_features gpu_extract_blob_features
#define quantize_colors gpu_quantize_colors
#define histogram gpu_histogram
#define meanshift_step gpu_meanshift_step
