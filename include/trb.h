/*
 * trb.h — C ABI of the B200-native video front end (motion -> 3x3 morphology
 * -> connected components -> blob statistics -> mean-shift tracking).
 *
 * This is the drop-in boundary for the hot path of the reference
 * ("teamrec", arXiv 1310.3322).  Every entry point replaces one reference
 * C++ call; the reference file:line is cited beside it (paths relative to
 * /root/reference/proj/include/teamrec/).  Plain pointers and sizes only:
 * no torch or C++ types cross this boundary.
 *
 * Conventions
 *   - Every function returns a trb_status; 0 is success.  On failure the
 *     message is available from trb_last_error() (thread-local), with the
 *     reference's own wording where the reference throws
 *     (e.g. "motion detector expects grayscale frames", motion.hpp:165).
 *   - The caller owns every buffer.  There is no cross-ABI free.
 *   - Handles are not internally synchronised (same as the reference
 *     objects, which are touched by one pipeline stage thread each,
 *     pipeline.hpp:259-286).  Each handle owns a CUDA stream.
 *   - There is no CPU fallback: without a usable sm_100 device every call
 *     that computes returns TRB_CUDA_ERROR.
 */
#ifndef TRB_H_
#define TRB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum trb_status {
  TRB_OK = 0,
  TRB_INVALID_ARGUMENT = 1, /* teamrec::InvalidArgument (error.hpp:15-18) */
  TRB_CONFIG_ERROR = 2,     /* teamrec::ConfigError (error.hpp:27-30)     */
  TRB_IO_ERROR = 3,         /* teamrec::IoError (error.hpp:21-24)         */
  TRB_CUDA_ERROR = 4,       /* device missing / kernel fault              */
  TRB_OUT_OF_MEMORY = 5,
  TRB_CAPACITY = 6          /* caller buffer too small; *n holds the need */
} trb_status;

/* ---- configuration structs (field-for-field the reference structs) ---- */

enum { TRB_BG_MEAN = 0, TRB_BG_MODE = 1 };       /* BackgroundMethod, motion.hpp:18 */
enum { TRB_CONN_FOUR = 0, TRB_CONN_EIGHT = 1 };   /* Connectivity, segmentation.hpp:15 */
enum { TRB_TRACK_ACTIVE = 0, TRB_TRACK_LOST = 1 }; /* TrackStatus, tracking.hpp:36 */
/* 3x3 morphology is NOT in the reference; default OFF keeps parity. */
enum { TRB_MORPH_NONE = 0, TRB_MORPH_ERODE = 1, TRB_MORPH_DILATE = 2, TRB_MORPH_OPEN = 3, TRB_MORPH_CLOSE = 4 };

/* MotionConfig (motion.hpp:44-56).  warp: 0 identity, 1 per-frame
 * homography (stream_detect, motion.hpp:260-282): the batched handle then
 * takes frames through trb_streams_step_device_warp. */
typedef struct trb_motion_config {
  int32_t method;    /* TRB_BG_MEAN | TRB_BG_MODE, default mean */
  int32_t window;    /* default 91 */
  int32_t threshold; /* default 25 */
  int32_t bins;      /* default 32 */
  int32_t warp;      /* 0 = identity, 1 = per-frame homography */
  int32_t morph;     /* extension: TRB_MORPH_*, default none */
} trb_motion_config;

/* SegmentationConfig (segmentation.hpp:25-34). */
typedef struct trb_seg_config {
  int32_t n_blocks;     /* default 4; validated, never changes the output */
  int32_t connectivity; /* default eight */
  int32_t min_area;     /* default 4 */
} trb_seg_config;

/* TrackerConfig (tracking.hpp:21-34). */
typedef struct trb_tracker_config {
  int32_t k_clusters;   /* default 16 */
  int32_t max_iters;    /* default 20 */
  double eps;           /* default 0.5 */
  int32_t kmeans_iters; /* default 20 */
  int32_t _pad;
  uint64_t seed;        /* default 0 */
} trb_tracker_config;

/* Blob (segmentation.hpp:36-45) without the pixel list. */
typedef struct trb_blob {
  int32_t label, area, x_min, y_min, x_max, y_max;
  double cx, cy;
} trb_blob;

/* TrackLogEntry (tracking.hpp:159-165). */
typedef struct trb_track_log_entry {
  int32_t frame, track_id;
  double x, y;
  int32_t w, h, status, _pad;
} trb_track_log_entry;

/* Track (tracking.hpp:40-50) scalar part; quantizer centres and the
 * target histogram are read with trb_tracker_track_model(). */
typedef struct trb_track {
  int32_t track_id, w, h, status, lost_frames, k;
  double cx, cy;
} trb_track;

/* ---- process-wide ---- */
const char* trb_last_error(void);
const char* trb_version(void);
int trb_device_count(int* n);
void trb_default_motion_config(trb_motion_config* c);
void trb_default_seg_config(trb_seg_config* c);
void trb_default_tracker_config(trb_tracker_config* c);
/* validate() of each config: MotionConfig::validate motion.hpp:51-55,
 * SegmentationConfig::validate segmentation.hpp:30-33,
 * TrackerConfig::validate tracking.hpp:28-33. */
int trb_motion_config_validate(const trb_motion_config* c);
int trb_seg_config_validate(const trb_seg_config* c);
int trb_tracker_config_validate(const trb_tracker_config* c);

/* ---- MotionDetector (motion.hpp:149-212) ---- */
typedef struct trb_motion trb_motion;
/* MotionDetector(cfg, w, h), motion.hpp:151-157 */
int trb_motion_create(const trb_motion_config* cfg, int width, int height, int device, trb_motion** out);
int trb_motion_destroy(trb_motion* m);
/* push(gray), motion.hpp:164-193.  gray: width*height bytes on the host,
 * channels must be 1.  *has_mask = 0 until `window` frames arrived
 * (std::nullopt), then mask_out (host, width*height bytes of 0/1) is
 * written. */
int trb_motion_push(trb_motion* m, const uint8_t* gray, int width, int height, int channels, int64_t frame_index,
                    uint8_t* mask_out, int* has_mask);
/* background(), motion.hpp:196-203 */
int trb_motion_background(trb_motion* m, uint8_t* out);
int trb_motion_frames_seen(const trb_motion* m, int* n);

/* ---- label_blocked / label_sequential (segmentation.hpp:183-264) ----
 * mask: host, w*h bytes (nonzero = foreground).  labels_out: host, w*h
 * int32 (nullable).  blobs_out: host, blob_cap entries (nullable); the
 * number of blobs is always written to *n_blobs; TRB_CAPACITY when
 * blob_cap is too small.  pixels_out (nullable) receives the per-blob
 * raster pixel lists (Blob::pixels, segmentation.hpp:141) concatenated in
 * label order: sum(area) int64 entries. */
int trb_label(const uint8_t* mask, int width, int height, const trb_seg_config* cfg, int device, int32_t* labels_out,
              trb_blob* blobs_out, int blob_cap, int* n_blobs, int64_t* pixels_out, int64_t pixels_cap);

/* ---- frame / track-log I/O (host side, no device) ----
 * decode_pnm / load_pnm (frame.hpp:152-183): binary P5 (gray) / P6 (RGB),
 * maxval 255, '#' comments in the header.  out == NULL queries the shape.
 * load_frame_sequence (:198-225): every .pgm/.ppm of `dir`, ordered by the
 * trailing digits of the file stem; out receives n_frames frames back to
 * back, indices (nullable) their indices.  Errors: TRB_IO_ERROR with the
 * reference's IoError messages. */
int trb_decode_pnm(const uint8_t* bytes, int64_t n, const char* source_name, int* width, int* height, int* channels,
                   uint8_t* out, int64_t out_cap);
int trb_load_pnm(const char* path, int* width, int* height, int* channels, uint8_t* out, int64_t out_cap);
int trb_load_frame_sequence(const char* dir, int* n_frames, int* width, int* height, int* channels,
                            int64_t* indices, uint8_t* out, int64_t out_cap);
/* Track-log interchange (tracking.hpp:244-285): text lines
 * `frame track_id x y w h status` (x, y as %.17g).  format: *len = text
 * length (out NULL = query; cap includes the terminating NUL). */
int trb_format_track_log(const trb_track_log_entry* log, int64_t n, char* out, int64_t cap, int64_t* len);
int trb_parse_track_log(const char* text, int64_t len, const char* source, trb_track_log_entry* out, int64_t cap,
                        int64_t* n);
int trb_save_track_log(const char* path, const trb_track_log_entry* log, int64_t n);
int trb_load_track_log(const char* path, trb_track_log_entry* out, int64_t cap, int64_t* n);

/* ---- 3x3 morphology on device masks (extension, not in the reference) ----
 * n_planes masks of width x height bytes (0/1), back to back in device memory;
 * out-of-image neighbours are ignored.  op: TRB_MORPH_*.  Widths that are a
 * multiple of 16 take the fused row-strip kernel (open/close in one pass);
 * `in` and `out` must not overlap.  cuda_stream: NULL = legacy stream. */
int trb_morph_device(const uint8_t* in, uint8_t* out, int width, int height, int n_planes, int op,
                     void* cuda_stream);

/* ---- warp_frame (motion.hpp:81-119) ----
 * Inverse-mapped bilinear resampling of one frame (host buffers) by the
 * homography h (row-major 3x3); samples off the source plane read 0. */
int trb_warp_frame(const uint8_t* frame, int width, int height, int channels, const double* homography, int device,
                   uint8_t* out);

/* ---- extract_blob_features (segmentation.hpp:266-291) ----
 * Per blob: mean intensity (luma for RGB frames) and bbox aspect
 * (width / height), as the reference fills Blob::mean_intensity / aspect.
 * Host buffers; labels is the w*h label image, blobs its n_blobs records.
 * TRB_INVALID_ARGUMENT "label image dimensions do not match frame" when the
 * sizes differ (:270-271). */
int trb_extract_blob_features(const int32_t* labels, int width, int height, const uint8_t* frame, int frame_width,
                              int frame_height, int channels, const trb_blob* blobs, int n_blobs, int device,
                              double* mean_intensity, double* aspect);

/* ---- Tracker (tracking.hpp:170-241) ---- */
typedef struct trb_tracker trb_tracker;
int trb_tracker_create(const trb_tracker_config* cfg, int device, trb_tracker** out);
int trb_tracker_destroy(trb_tracker* t);
/* process(frame, blobs), tracking.hpp:179-205.  frame: host, w*h*channels. */
int trb_tracker_process(trb_tracker* t, const uint8_t* frame, int width, int height, int channels,
                        const trb_blob* blobs, int n_blobs);
int trb_tracker_num_tracks(const trb_tracker* t, int* n);
int trb_tracker_tracks(const trb_tracker* t, trb_track* out, int cap);
/* centers: k*3 doubles, target_hist: k doubles, for track i (list order) */
int trb_tracker_track_model(const trb_tracker* t, int i, double* centers, double* target_hist);
int trb_tracker_log_size(const trb_tracker* t, int64_t* n);
int trb_tracker_log(const trb_tracker* t, trb_track_log_entry* out, int64_t cap);
int trb_tracker_frames_processed(const trb_tracker* t, int* n);

/* ---- batched device-resident front end (run_vision, harness.hpp:412-450) ----
 * n_streams independent camera streams of one geometry advance one frame
 * per step: motion -> (morph) -> CCL -> blob stats -> tracking, each stage
 * one launch for all streams.  Outputs stay in HBM until downloaded. */
typedef struct trb_streams trb_streams;
int trb_streams_create(int n_streams, int width, int height, int channels, const trb_motion_config* mc,
                       const trb_seg_config* sc, const trb_tracker_config* tc, int device, trb_streams** out);
/* Capacities of a streams handle.  The reference's track list and log are
 * unbounded std::vectors (tracking.hpp:237-238); on the device they are
 * bounded per stream.  A step that would exceed either bound FAILS: the
 * device records a sticky error, and the next step / synchronize /
 * download call returns TRB_CAPACITY (the tracker state is no longer the
 * reference's).  The log is a ring: entries stay until drained
 * (trb_streams_drain_log), so a long-running stream that drains now and
 * then never overflows. */
typedef struct trb_streams_options {
  int32_t track_cap; /* live tracks per stream, default 256 */
  int32_t _pad;
  int64_t log_cap;   /* undrained log entries held per stream, default 65536 */
} trb_streams_options;
void trb_default_streams_options(trb_streams_options* o);
int trb_streams_create_ex(int n_streams, int width, int height, int channels, const trb_motion_config* mc,
                          const trb_seg_config* sc, const trb_tracker_config* tc, const trb_streams_options* opt,
                          int device, trb_streams** out);
/* Per-step results of the host path, what Tracker::process / label_blocked
 * hand back to the reference's caller for the frame: every stream's blob
 * count and blob table (the first blob_cap records; n_blobs may exceed it),
 * and the log entries the frame appended (tracking.hpp:203; the first
 * log_cap of n_log).  All pointers are PINNED host memory (cudaMallocHost)
 * or NULL (region skipped); arrays are [n_streams] / [n_streams][cap]. */
typedef struct trb_step_output {
  int32_t* n_blobs;
  trb_blob* blobs;
  int32_t blob_cap;
  int32_t log_cap;
  int32_t* n_log;
  trb_track_log_entry* log;
} trb_step_output;
int trb_streams_destroy(trb_streams* s);
/* frames: host array of n_streams DEVICE pointers (w*h*channels bytes each;
 * any alignment — 16-byte aligned frames take the vector path).
 * cuda_stream: cudaStream_t to launch on (NULL = the handle's own).
 * Step overlap: motion + CCL of a step run on cuda_stream; its tracking runs
 * on the handle's internal stream and overlaps the NEXT step's motion + CCL.
 * cuda_stream covers all work up to the previous step's tracking;
 * trb_streams_join makes a stream wait for everything issued so far
 * (trb_streams_synchronize and the download calls wait for everything).
 * The frames must stay valid until the step's tracking has run. */
int trb_streams_step_device(trb_streams* s, const uint8_t* const* frames, void* cuda_stream);
/* cuda_stream waits (on the device) for every step issued so far. */
int trb_streams_join(trb_streams* s, void* cuda_stream);
/* step_device for MotionConfig::warp = homography: every frame is warped
 * into the reference plane (warp_frame, motion.hpp:81-119) by its
 * homography (homographies: host, n_streams * 9 doubles, row-major) before
 * it enters the window (stream_detect, motion.hpp:279).  Errors are the
 * reference's ("homography has a non-finite entry", "... not normalizable
 * (h[2][2] = 0)", "... not invertible"). */
int trb_streams_step_device_warp(trb_streams* s, const uint8_t* const* frames, const double* homographies,
                                 void* cuda_stream);
/* frames: host array of n_streams HOST pointers (pinned for best speed);
 * the H2D copy is part of the call.  If result_host is not NULL it
 * receives n_streams int32 blob counts (the D2H read of the step). */
int trb_streams_step_host(trb_streams* s, const uint8_t* const* frames, int32_t* result_host, void* cuda_stream);
/* Pipelined step_host: returns once the work is queued.  The frames' H2D
 * copy runs on the handle's copy stream into one of three staging buffers and
 * overlaps the previous step's kernels; result_host (if not NULL) is written
 * when cuda_stream reaches this step.  frames and result_host must stay
 * valid until trb_streams_synchronize (or a later synchronous call). */
int trb_streams_step_host_async(trb_streams* s, const uint8_t* const* frames, int32_t* result_host,
                                void* cuda_stream);
/* step_host_async with the step's results (trb_step_output) copied back
 * on the device's own schedule: valid after trb_streams_synchronize. */
int trb_streams_step_host_async_out(trb_streams* s, const uint8_t* const* frames, const trb_step_output* out,
                                    void* cuda_stream);
int trb_streams_synchronize(trb_streams* s);
/* Copy up to cap undrained track-log entries of `stream` (oldest first)
 * into out, release them from the device ring; *n = entries copied.
 * trb_streams_download_log / log_size see only undrained entries. */
int trb_streams_drain_log(trb_streams* s, int stream, trb_track_log_entry* out, int64_t cap, int64_t* n);
int trb_streams_frames_seen(const trb_streams* s, int* n);
/* 1 once the window is full (a mask/labels/blobs exist for the last step) */
int trb_streams_has_output(const trb_streams* s, int* has);
int trb_streams_download_mask(trb_streams* s, int stream, uint8_t* out);
int trb_streams_download_labels(trb_streams* s, int stream, int32_t* out);
int trb_streams_download_blobs(trb_streams* s, int stream, trb_blob* out, int cap, int* n);
int trb_streams_log_size(trb_streams* s, int stream, int64_t* n);
int trb_streams_download_log(trb_streams* s, int stream, trb_track_log_entry* out, int64_t cap);
int trb_streams_num_tracks(trb_streams* s, int stream, int* n);
/* Kernel launches issued by the last step (for the bench's gpu_launches). */
int trb_streams_last_step_launches(const trb_streams* s, int* n);
/* Per-stage device time (CUDA events on the launch stream around the
 * motion, CCL+statistics, tracker schedule+mean-shift and tracker
 * gate+spawn stages), summed over the profiled steps: ms_out[4].
 * Profiling synchronises after every step. */
int trb_streams_profile(trb_streams* s, int enable);
int trb_streams_profile_read(const trb_streams* s, double* ms_out, int* steps);
/* extract_blob_features for stream `stream`'s last step, from its labels and
 * blob table in HBM and `frame_dev` (device pointer to that step's frame):
 * *n = blob count; mean_intensity / aspect (host, cap entries). */
int trb_streams_blob_features(trb_streams* s, int stream, const uint8_t* frame_dev, double* mean_intensity,
                              double* aspect, int cap, int* n);
/* Device pointers of the per-stream output planes (for device consumers). */
int trb_streams_device_planes(trb_streams* s, int stream, uint8_t** mask, int32_t** labels);

/* ---- synthetic input (synth.hpp:45-101), device rasteriser ----
 * rects: n_shapes * 4 int32 (ix, iy, w, h) already rounded with lround on
 * the host (synth.hpp:313-314); colors: n_shapes * 3 bytes.  Later shapes
 * overwrite earlier ones.  out: DEVICE buffer w*h*channels. */
int trb_synth_raster(uint8_t* out_device, int width, int height, int channels, uint8_t background,
                     const int32_t* rects, const uint8_t* colors, int n_shapes, void* cuda_stream);
/* n_frames frames in one launch: rects is n_frames * n_shapes * 4, frame f
 * is written at out_device + f*frame_stride. */
int trb_synth_raster_frames(uint8_t* out_device, int64_t frame_stride, int n_frames, int width, int height,
                            int channels, uint8_t background, const int32_t* rects, const uint8_t* colors,
                            int n_shapes, void* cuda_stream);


/* ---- standalone tracker operations (public reference functions) ----
 * frame: host, w*h*channels bytes.  Device-computed, bit-exact. */
/* meanshift_step(frame, track, cfg), tracking.hpp:125-157.  *status is
 * TRB_TRACK_ACTIVE / TRB_TRACK_LOST, in and out. */
int trb_meanshift_step(const uint8_t* frame, int width, int height, int channels, double* cx, double* cy, int w,
                       int h, const double* centers, const double* target_hist, int k, int max_iters, double eps,
                       int* status, int device);
/* histogram(frame, cx, cy, w, h, q, kernel), tracking.hpp:106-112
 * (epanechnikov = 1, uniform = 0).  Errors as the reference:
 * "histogram window must be >= 3x3", "histogram window does not intersect
 * the frame". */
int trb_histogram(const uint8_t* frame, int width, int height, int channels, double cx, double cy, int w, int h,
                  const double* centers, int k, int epanechnikov, double* hist_out, int device);
/* quantize_colors(pixels, k, iters, seed), quantize.hpp:43-118; samples must
 * be integer-valued in [0, 65535] (as rgb_at produces). */
int trb_quantize_colors(const double* pixels, int64_t n, int k, int iters, uint64_t seed, double* centers_out,
                        int device);

/* ---- self tests of the exact-arithmetic replicas (host build of the same
 * header the kernels use; on_device = 1 runs the device build) ---- */
int trb_selftest_hypot(const double* x, const double* y, int64_t n, double* out, int on_device);
/* device diagnostics: [0] ordered-sum calls [1] sums [2] sums replayed by the
 * exact serial fallback [3] breakpoints [4] elements [5] mean-shift
 * iterations [6] spawns [7] Lloyd iterations [8] empty-cluster passes
 * [9] tracks advanced, [16..25] ordered-sum failure reasons by bit.
 * reset != 0 zeroes them after reading. */
int trb_debug_stats(uint64_t* out32, int reset);
/* hang diagnostics: tracker CTAs publish {kernel, item, iteration, stage}
 * into host-mapped memory; *host_out points at n_ctas*4 ints. */
int trb_debug_progress(int n_ctas, int** host_out);
/* per mean-shift-iteration timing log: enable (1/0, -1 = keep), read up to
 * cap {window pixels, SM cycles} pairs */
int trb_debug_itlog(int enable, int64_t* out_pairs, int64_t cap, int64_t* n);
/* per-phase SM cycles of the mean-shift iterations while the log is on:
 * [bucket][64] by window size (<5k, <50k, <150k, larger pixels); entry 0 of
 * a bucket counts its iterations (256 entries) */
int trb_debug_phases(uint64_t* out256);
/* diagnostics build: per mean-shift CTA [busy ns, last item end
 * (globaltimer ns)] while the log is on (2048 entries) */
int trb_debug_cta_times(uint64_t* out2048, int reset);
/* diagnostics build: per (cluster rank 0..7, warp 0..7, [histogram,
 * centroid]) the sum over 8-CTA engine runs of the warp's phase-B walk
 * cycles (slowest lane) while the log is on (128 entries) */
int trb_debug_warp_walks(uint64_t* out128, int reset);

#ifdef __cplusplus
}
#endif

#endif /* TRB_H_ */
