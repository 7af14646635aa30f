// trb_track.cuh — device-resident multi-object tracker (north-star kernel
// (5): nearest-centroid track association, plus the mean-shift update and
// the k-means colour model it depends on).
//
// Reference: Tracker (tracking.hpp:170-241), meanshift_step (:125-157),
// histogram_opt (:79-102), spawn_track (:208-234), quantize_colors
// (quantize.hpp:43-118).  Bit-exact: every fp64 operation is an explicit
// round-to-nearest intrinsic, sequential sums go through ordered_sums()
// (trb_osum.cuh), hypot is glibc's algorithm (trb_exact.cuh).
//
// State layout (per stream s, slot capacity T, K clusters), all in HBM:
//   list[s][T]      slot ids in the reference's track-list order
//   slot arrays     id, w, h, status, lost, pending, cx, cy,
//                   centers[K][3], hist[K], lut[256] (gray -> bin)
//   log[s][cap]     TrackLogEntry records (tracking.hpp:159-165)
// Per frame: meanshift (one CTA per active track, persistent grid) ->
// gate (one CTA per stream: association, spawn decisions, retire, log) ->
// spawn (one CTA per new track: k-means++ / Lloyd / target histogram).
#pragma once

#include "trb_engine.cuh"
#include "trb_osum.cuh"

namespace trb {

struct TrackDev {
  int S, T, K;
  int max_iters, kmeans_iters;
  double eps;
  uint64_t seed;
  int W, H, CH;  // frame geometry
  const uint8_t* const* frames;  // [S] device frame pointers
  // per stream
  int32_t* n_list;
  int32_t* list;  // [S][T]
  int32_t* next_id;
  int32_t* frame_no;
  int32_t* err;  // bit0 track-capacity overflow, bit1 log overflow
  int32_t* err_any;  // OR of every stream's err
  // mapped pinned host words the kernels store into (no per-step D2H copy):
  // [0] active tracks of the frame (schedule), [1] / [2] track / log
  // capacity exceeded (gate; sticky)
  volatile int32_t* host_mirror;
  // per slot [S][T]
  int32_t *id, *w, *h, *status, *lost, *used, *pending;
  int32_t* iters;  // mean-shift iterations of the last frame (scheduling hint)
  double *cx, *cy;
  double* centers;  // [S][T][K][3]
  double* hist;     // [S][T][K]
  uint8_t* lut;     // [S][T][256]
  // blobs of the current frame
  const trb_blob* blobs;
  int64_t blob_stride;
  const int32_t* nblobs;
  uint8_t* matched;  // [S][blob_stride] scratch
  // log
  trb_track_log_entry* log;  // [S][log_cap] ring
  int64_t log_cap;
  int64_t* n_log;     // [S] head: entries ever logged
  int64_t* log_tail;  // [S] entries drained by the host
  int64_t* step_log_base;  // [S] head before the last frame's entries
  // meanshift work queue (largest window first)
  int32_t* work;       // [S*T]
  int32_t* work_n;
  int32_t* work_head;
  // tracks spawned this frame (gate kernel appends, spawn kernel claims)
  int32_t* spawn_list;  // [S*T] slot indices
  int32_t* spawn_n;
  int32_t* spawn_head;
  int G;               // CTAs per cluster
  int iter_floor;      // scheduling: iterations assumed at least
  int iter_decay;      // scheduling: iteration hint = max(now, prev - prev*decay/8); 0 = this frame's
  double split_us;     // tracks estimated below this (single-CTA us) run in split mode
  double split_fix, split_perpx;  // single-CTA cost model: us per iteration + us per window pixel
  int order_fix;       // queue order: cost = iterations x (order_fix + window px)
  // per-cluster scratch (breakpoint list, partitioned weights, bin cache)
  unsigned char* scratch;
  size_t scratch_stride;
  int64_t maxN;
  double* u2;  // v2 engine: per-CTA ux2 / uy2 (W + H + 1 doubles each)
  uint32_t* words2;  // v2 engine: per-cluster staged bin words
  int stream_groups;  // schedule: streams in this many contiguous groups, processed group after group
};

class TrackerState {
 public:
  TrackerState(const trb_tracker_config& cfg, int S, int track_cap = 256, int64_t log_cap = 1 << 16);
  ~TrackerState();
  // One Tracker::process for every stream.  blobs: device [S][blob_stride].
  // blobs_ready (optional): `st` waits for it before the gate kernel, the
  // first reader of the blob table (mean-shift itself needs only the
  // frames and the track state).
  // after_meanshift (optional) is recorded on `st` right after the
  // mean-shift kernel (per-stage profiling)
  void process(const uint8_t* const* frames_dev, int w, int h, int ch, const trb_blob* blobs, int64_t blob_stride,
               const int32_t* nblobs, cudaStream_t st, int* launches, cudaEvent_t after_meanshift = nullptr,
               cudaEvent_t blobs_ready = nullptr);
  // host-side readers (synchronise `st`)
  int num_tracks(int s, cudaStream_t st);
  void tracks(int s, trb_track* out, int cap, cudaStream_t st);
  void track_model(int s, int i, double* centers, double* hist, cudaStream_t st);
  // entries logged and not drained yet (the whole log when never drained)
  int64_t log_size(int s, cudaStream_t st);
  void log(int s, trb_track_log_entry* out, int64_t cap, cudaStream_t st);
  // copy up to cap undrained entries out and release them; returns the count
  int64_t drain_log(int s, trb_track_log_entry* out, int64_t cap, cudaStream_t st);
  // the last processed frame's results packed for one D2H: per stream the
  // blob count, the first bcap blobs, the number of log entries of the frame
  // and its first lcap entries (regions as trb_step_output, device memory)
  void pack_step(const trb_blob* blobs, int64_t blob_stride, const int32_t* nblobs, int32_t* n_blobs_out,
                 trb_blob* blobs_out, int bcap, int32_t* n_log_out, trb_track_log_entry* log_out, int lcap,
                 cudaStream_t st);
  const int32_t* err_word() const { return d_.err_any; }
  // the sticky error bits as the kernels left them in host memory (no sync):
  // 1 track capacity, 2 log capacity
  int32_t host_errors() const {
    const volatile int32_t* m = static_cast<const volatile int32_t*>(mirror_.p);
    return (m[1] ? 1 : 0) | (m[2] ? 2 : 0);
  }
  int track_cap() const { return T_; }
  int64_t log_cap() const { return log_cap_; }
  int frames_processed(int s, cudaStream_t st);
  void check_errors(cudaStream_t st, bool log_too = true);
  const trb_tracker_config& cfg() const { return cfg_; }

 private:
  trb_tracker_config cfg_;
  int S_, T_, K_;
  int64_t log_cap_;
  DevBuf i32_, f64_, lut_, log_, nlog_, matched_, bp_, work_, u2_, words2_;
  TrackDev d_{};
  int64_t matched_cap_ = 0;
  int grid_ = 0, grid2_ = 0;
  int grid_big_[2] = {0, 0};  // clusters of 16 and of 12 CTAs (few-track frames)
  PinnedBuf mirror_;          // TrackDev::host_mirror (mapped)
  size_t smem_set_ = 0, smem2_ = 0;
};

// device diagnostics counters (see g_trb_stats in trb_track.cu)
void read_debug_stats(unsigned long long* out, bool reset);

// ---- standalone device ops behind the C ABI (tests and compat layer) ----
// meanshift_step (tracking.hpp:125-157) on one track; frame on the device.
void device_meanshift_step(const uint8_t* frame_dev, int w, int h, int ch, double* cx, double* cy, int tw, int th,
                           const double* centers, const double* target, int k, int max_iters, double eps,
                           int* status, cudaStream_t st);
// histogram_opt (tracking.hpp:79-102); returns false for nullopt.
bool device_histogram(const uint8_t* frame_dev, int w, int h, int ch, double cx, double cy, int tw, int th,
                      const double* centers, int k, int epanechnikov, double* hist, cudaStream_t st);
// quantize_colors (quantize.hpp:43-118) for integer-valued samples.
void device_quantize_colors(const double* pixels, int64_t n, int k, int iters, uint64_t seed, double* centers,
                            cudaStream_t st);

}  // namespace trb

namespace trb {
// hang diagnostics: host-mapped progress records [n_ctas][4]
int* enable_progress(int n_ctas);
void enable_itlog(bool on);
int64_t read_itlog(long long* out, int64_t cap);
void read_phases(unsigned long long* out128);
void read_cta_times(unsigned long long* out2048, bool reset);
void read_warpwalk(unsigned long long* out128, bool reset);
}  // namespace trb
