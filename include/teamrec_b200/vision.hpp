// vision.hpp — run_vision (harness.hpp:412-450) with device stages.
//
// The reference assembles the video front end as three type-erased pipeline
// stages (make_stage<In, Out>, pipeline.hpp:44-54) around a MotionDetector,
// label_blocked and a Tracker, and runs them through its Pipeline in
// Sequential or Pipelined mode (one thread per stage).  make_vision_stages()
// returns the same three StageSpecs ("motion", "segmentation", "tracking";
// Frame -> VisionItem -> VisionItem -> VisionItem) backed by the device
// objects of teamrec_b200.hpp, so a caller's Pipeline::assemble /
// run_pipeline work unchanged; run_vision() is the reference's entry point
// over them.  Each stage object is touched by one stage thread at a time,
// as the C ABI requires.
//
// (Do not combine with redirect.hpp in one translation unit: that header
// renames these identifiers.)
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "teamrec/harness.hpp"
#include "teamrec_b200/teamrec_b200.hpp"

namespace teamrec_b200 {

// The three run_vision stages over device objects; *tracker_out (optional)
// receives the tracker so its log can be read after the run.
inline std::vector<teamrec::StageSpec> make_vision_stages(const teamrec::FrameworkConfig& cfg, int width, int height,
                                                          const teamrec::Backend& backend,
                                                          std::shared_ptr<Tracker>* tracker_out = nullptr) {
  auto detector = std::make_shared<MotionDetector>(cfg.motion, width, height);
  auto tracker = std::make_shared<Tracker>(cfg.tracker);
  if (tracker_out) *tracker_out = tracker;
  std::vector<teamrec::StageSpec> stages;
  stages.push_back(teamrec::make_stage<teamrec::Frame, teamrec::VisionItem>(
      "motion",
      [detector](teamrec::Frame f) {
        teamrec::VisionItem item;
        item.mask = detector->push(f.channels == 1 ? f : teamrec::grayscale(f));
        item.frame = std::move(f);
        return item;
      },
      teamrec::Backend::sequential(), cfg.queue_capacity));
  const teamrec::SegmentationConfig seg = cfg.segmentation;
  stages.push_back(teamrec::make_stage<teamrec::VisionItem, teamrec::VisionItem>(
      "segmentation",
      [seg](teamrec::VisionItem item) {
        if (item.mask) item.labeling = teamrec_b200::label_blocked(*item.mask, seg);
        return item;
      },
      backend, cfg.queue_capacity));
  stages.push_back(teamrec::make_stage<teamrec::VisionItem, teamrec::VisionItem>(
      "tracking",
      [tracker](teamrec::VisionItem item) {
        if (item.labeling) tracker->process(item.frame, item.labeling->blobs);
        return item;
      },
      backend, cfg.queue_capacity));
  return stages;
}

// harness.hpp:412-450 on the device stages: same outputs (items, track log,
// per-stage timing) as the reference's run_vision.
inline teamrec::VisionOutputs run_vision(const teamrec::FrameworkConfig& cfg, const std::vector<teamrec::Frame>& frames,
                                         const teamrec::Backend& backend, teamrec::PipelineMode mode) {
  std::shared_ptr<Tracker> tracker;
  auto stages = make_vision_stages(cfg, frames.empty() ? 1 : frames[0].width, frames.empty() ? 1 : frames[0].height,
                                   backend, &tracker);
  const teamrec::Pipeline p = teamrec::Pipeline::assemble(std::move(stages));
  auto [items, timing] = teamrec::run_pipeline<teamrec::Frame, teamrec::VisionItem>(p, frames, mode);
  teamrec::VisionOutputs out;
  out.items = std::move(items);
  out.track_log = tracker->log();
  out.timing = std::move(timing);
  return out;
}

}  // namespace teamrec_b200
