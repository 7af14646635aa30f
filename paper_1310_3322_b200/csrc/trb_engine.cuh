// trb_engine.cuh — host-side state machines over the kernels.  One object
// per reference object: MotionState ~ MotionDetector (motion.hpp:149-212),
// CclState ~ label_blocked's workspace (segmentation.hpp:198-264),
// TrackerState ~ Tracker (tracking.hpp:170-241).  Each holds a batch of
// S independent streams so one launch serves every stream of a GPU.
#pragma once

#include <memory>
#include <vector>

#include "trb_kernels.cuh"

namespace trb {

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t bytes, bool zero = true) {
    if (bytes <= n && p) return;
    release();
    TRB_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    n = bytes;
    if (zero) {
      // Every consumer runs on a non-blocking stream, which does not order
      // after the legacy stream: finish the clear before anyone can launch.
      TRB_CUDA(cudaMemsetAsync(p, 0, bytes ? bytes : 16, 0));
      TRB_CUDA(cudaStreamSynchronize(0));
    }
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void alloc(size_t bytes) {
    if (bytes <= n && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    TRB_CUDA(cudaMallocHost(&p, bytes ? bytes : 16));
    n = bytes;
  }
  // mapped pinned memory: kernels store into it directly (its device address)
  void alloc_mapped(size_t bytes) {
    if (p) cudaFreeHost(p);
    p = nullptr;
    TRB_CUDA(cudaHostAlloc(&p, bytes ? bytes : 16, cudaHostAllocMapped));
    n = bytes;
  }
  void* device_ptr() const {
    void* d = nullptr;
    TRB_CUDA(cudaHostGetDevicePointer(&d, p, 0));
    return d;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

bool is_pinned_host(const void* p);
void* pinned_device_alias(const void* p);
bool pinned_unmapped(const void* p);
void validate_motion(const trb_motion_config& c);
void validate_seg(const trb_seg_config& c, int w, int h);
void validate_tracker(const trb_tracker_config& c);

class MotionState {
 public:
  MotionState(const trb_motion_config& cfg, int S, int w, int h, int ch);
  // frames_dev: device array [S] of device frame pointers.  Writes the
  // masks (device, S*px) when the window is full; returns true then.
  // frames_aligned: every frame pointer is 16-byte aligned (the 16-byte
  // vector path needs it; otherwise the scalar path runs)
  bool push(const uint8_t* const* frames_dev, uint8_t* mask, uint8_t* tmp, cudaStream_t st, int* launches,
            bool frames_aligned = true);
  void background(uint8_t* out_dev, cudaStream_t st);  // stream 0 only
  int frames_seen() const { return frames_seen_; }
  const trb_motion_config& cfg() const { return cfg_; }

 private:
  trb_motion_config cfg_;
  int S_, w_, h_, ch_;
  int64_t px_;
  bool wide_;
  int frames_seen_ = 0;
  bool mode_inc_ = false;
  DevBuf ring_, sums_, cnt_, bsum_, mode_;  // cnt_/bsum_/mode_: incremental Mode state
};

class CclState {
 public:
  CclState(int S, int w, int h, const trb_seg_config& cfg);
  // mask: device [S][px].  Labels, blobs and counts stay on the device.
  // The blob table is double-buffered: run() writes the buffer the previous
  // run did not, so a tracker may still read the last table while the next
  // frame is labelled.  blobs()/nblobs() = the table of the latest run.
  void run(const uint8_t* mask, cudaStream_t st, int* launches);
  int32_t* labels() const { return labels_.as<int32_t>(); }
  trb_blob* blobs() const { return blobs_[cur_].as<trb_blob>(); }
  int32_t* nblobs() const { return nblobs_[cur_].as<int32_t>(); }
  int next_buffer() const { return cur_ ^ 1; }
  int64_t blob_cap() const { return blob_cap_; }
  int64_t px() const { return px_; }

 private:
  CclArgs args_{};
  int S_, w_, h_;
  int64_t px_, slot_cap_, blob_cap_;
  DevBuf labg_, labels_, slots_, nslots_, rowcount_, bitmap_, blobs_[2], nblobs_[2], tiles_, tile_state_;
  int cur_ = 0;
};

class TrackerState;  // trb_track.cu

// The batched front end: motion -> morph -> CCL -> tracking for S streams.
class Streams {
 public:
  Streams(int S, int w, int h, int ch, const trb_motion_config& mc, const trb_seg_config& sc,
          const trb_tracker_config& tc, bool with_tracker, int track_cap = 256, int64_t log_cap = 1 << 16);
  ~Streams();
  void step_device(const uint8_t* const* frames_host_array_of_dev_ptrs, cudaStream_t st);
  // MotionConfig::warp == per-frame homography (stream_detect, motion.hpp:
  // 260-282): every frame is first warped into the reference plane by its
  // homography h9s[s*9 .. s*9+8] (row-major, host memory).
  void step_device_warp(const uint8_t* const* frames_host_array_of_dev_ptrs, const double* h9s, cudaStream_t st);
  // synchronous: result_host (S blob counts) valid on return
  void step_host(const uint8_t* const* frames_host, int32_t* result_host, cudaStream_t st);
  // pipelined: the H2D copy of this step's frames runs on a copy stream
  // (overlapping the previous step's kernels) into one of two staging
  // buffers; result_host is written when `st` reaches this step (valid after
  // synchronize()); frames_host must stay untouched until then.
  void step_host_async(const uint8_t* const* frames_host, int32_t* result_host, cudaStream_t st,
                       const trb_step_output* out = nullptr);
  // Throws the tracker's sticky capacity error once the device reported it
  // (mirrored into pinned memory after every step: raised at most a step
  // or two after the step that overflowed, and at synchronize()).
  void check_sticky_errors();
  // Make `st` wait for every step issued so far (the tracker of the last
  // step runs on an internal stream; see run_).
  void join(cudaStream_t st);
  void set_overlap(bool on) { overlap_ = on; }
  cudaStream_t stream() const { return own_; }
  int S() const { return S_; }
  int w() const { return w_; }
  int h() const { return h_; }
  int ch() const { return ch_; }
  int64_t px() const { return px_; }
  int frames_seen() const { return motion_->frames_seen(); }
  bool has_output() const { return has_output_; }
  int last_launches() const { return last_launches_; }
  uint8_t* mask(int s) const { return mask_.as<uint8_t>() + px_ * s; }
  CclState& ccl() { return *ccl_; }
  TrackerState* tracker() { return tracker_.get(); }
  // per-stage device time (motion, ccl, tracking) accumulated over steps
  static constexpr int kStages = 4;  // motion, ccl+stats, track schedule+meanshift, gate+spawn
  void set_profiling(bool on);
  const double* profile_ms() const { return prof_ms_; }
  int profile_steps() const { return prof_steps_; }

 private:
  static constexpr int kPtrSlots = 16;
  static constexpr int kStaging = 3;  // host-path staging ring (step t's tracker reads its frames during t+1)
  // frames_dev stays valid until `done` (an event recorded after the last
  // read of the frames: the tracker's stream when it overlaps)
  // returns the stream of the frames' last reader
  cudaStream_t run_(const uint8_t* const* frames_dev, cudaStream_t st, bool overlap, cudaEvent_t done);
  const uint8_t* const* upload_ptrs_(const uint8_t* const* frames, cudaStream_t st);
  int S_, w_, h_, ch_;
  int64_t px_;
  trb_motion_config mc_;
  bool frames_aligned_ = true;  // the current step's frame pointers are 16-byte aligned
  std::unique_ptr<MotionState> motion_;
  std::unique_ptr<CclState> ccl_;
  std::unique_ptr<TrackerState> tracker_;
  DevBuf mask_, mask_tmp_, frame_ptrs_, staging_[kStaging];
  DevBuf staging_ptrs_;  // [kStaging][S] device pointer tables of the staging planes (constant)
  // step overlap: the tracker of step t runs on trk_ while motion + CCL of
  // step t+1 run on the caller's stream (blob tables double-buffered)
  cudaStream_t trk_ = nullptr;
  cudaEvent_t ccl_ev_[2] = {}, trk_ev_[2] = {}, mot_ev_[2] = {};
  bool early_ms_ = true;
  bool direct_out_ = true;  // step outputs stored by the pack kernel into the caller's pinned buffers (TRB_DIRECT_OUT=0: copies)  // mean-shift waits for the step's motion only, the gate for its CCL (TRB_EARLY_MS=0: both for CCL)
  bool trk_pending_[2] = {false, false};
  int last_trk_ = -1;
  bool overlap_ = true;  // TRB_OVERLAP=0 disables (A/B)
  DevBuf warp_buf_, warp_ptrs_, invs_dev_;  // warped frames, their pointer table, inverses [slot][S][9]
  PinnedBuf invs_host_;
  PinnedBuf result_pinned_;
  DevBuf out_dev_;              // packed step output (trb_step_output regions)
  int out_bcap_ = -1, out_lcap_ = -1;
  PinnedBuf out_bounce_;        // pageable trb_step_output targets go through here
  void output_(const trb_step_output* out, cudaStream_t last_reader, int* launches);
  const trb_step_output* pending_out_ = nullptr;  // set by step_host_async for run_
  cudaStream_t copy_ = nullptr;
  cudaEvent_t copied_[kStaging] = {}, consumed_[kStaging] = {};
  int host_step_ = 0;
  PinnedBuf ptrs_host_;
  cudaStream_t own_ = nullptr;
  bool has_output_ = false;
  int last_launches_ = 0;
  int ptr_slot_ = 0;
  cudaEvent_t slot_ev_[kPtrSlots] = {};
  cudaEvent_t prof_ev_[kStages + 1] = {};
  bool profiling_ = false;
  double prof_ms_[kStages] = {};
  int prof_steps_ = 0;
};

}  // namespace trb
