// TEST INFRASTRUCTURE: the device run_vision (include/teamrec_b200/vision.hpp)
// against the reference's run_vision (harness.hpp:412-450) on clips of the
// reference's generator: identical vision_digest (every mask bit, every
// label, the %.17g track log), in Sequential and Pipelined mode, plus the
// stage names / item counts of the timing report.  Exit code 0 = identical.
#include <cstdio>
#include <string>

#include "teamrec_b200/vision.hpp"

using namespace teamrec;

static int compare(const char* name, const FrameworkConfig& cfg, const std::vector<Frame>& frames) {
  int bad = 0;
  const VisionOutputs want = run_vision(cfg, frames, Backend::sequential(), PipelineMode::Sequential);
  const std::string wd = vision_digest(want);
  for (PipelineMode mode : {PipelineMode::Sequential, PipelineMode::Pipelined}) {
    const VisionOutputs got = teamrec_b200::run_vision(cfg, frames, Backend::parallel(2), mode);
    const bool same = vision_digest(got) == wd;
    const bool stages = got.timing.stages.size() == 3 && got.timing.stages[0].name == "motion" &&
                        got.timing.stages[1].name == "segmentation" && got.timing.stages[2].name == "tracking" &&
                        got.timing.stages[0].items == frames.size();
    std::printf("%s %s %s: digest %s (%zu bytes, %zu log entries), stages %s\n", same && stages ? "PASS" : "FAIL",
                name, pipeline_mode_name(mode).c_str(), same ? "identical" : "DIFFERS", wd.size(),
                got.track_log.size(), stages ? "ok" : "BAD");
    bad += !(same && stages);
  }
  return bad;
}

int main() {
  int bad = 0;
  {  // harness_test.cpp:377-410's clip: 48x36 RGB, two shapes, window 9
    FrameworkConfig cfg;
    cfg.motion.window = 9;
    ClipSpec clip;
    clip.width = 48;
    clip.height = 36;
    clip.channels = 3;
    const int n_frames = cfg.motion.window + 20;
    const double span = n_frames - 1;
    clip.shapes.push_back({7, 7, {220, 60, 40}, 3.0, 3.0, (28.0 - 3.0) / span, (20.0 - 3.0) / span, 0.0});
    clip.shapes.push_back({6, 6, {40, 80, 230}, 38.0, 26.0, (4.0 - 38.0) / span, (6.0 - 26.0) / span, 0.0});
    bad += compare("harness-clip", cfg, synth_frames(clip, n_frames, 4321).frames);
  }
  {  // a gray 320x240 clip with three crossing shapes, default window (91)
    FrameworkConfig cfg;
    ClipSpec clip;
    clip.width = 320;
    clip.height = 240;
    clip.channels = 1;
    clip.background = 16;
    const int n_frames = 130;
    const double span = n_frames - 1;
    clip.shapes.push_back({16, 14, {200, 200, 200}, 20.0, 30.0, 250.0 / span, 160.0 / span, 0.0});
    clip.shapes.push_back({12, 18, {120, 120, 120}, 270.0, 190.0, -250.0 / span, -160.0 / span, 0.0});
    clip.shapes.push_back({20, 12, {250, 250, 250}, 150.0, 20.0, 10.0 / span, 190.0 / span, 0.0});
    bad += compare("gray-320x240", cfg, synth_frames(clip, n_frames, 77).frames);
  }
  std::printf("%s\n", bad ? "FAILED" : "ALL IDENTICAL");
  return bad;
}
