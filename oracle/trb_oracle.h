/*
 * trb_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's per-frame video front end
 * (teamrec, /root/reference/proj/include/teamrec/ headers).  It is the checker
 * the CUDA path is compared against; it is never linked into the product
 * library (paper_1310_3322_b200/csrc) and only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.
 *
 * Parity of this restatement is PINNED two ways (see tests/test_oracle_*.py):
 *   1. the reference's own golden vectors / known-answer tests
 *      (motion_test.cpp, segmentation_test.cpp, tracking_test.cpp), and
 *   2. the unmodified reference compiled from its headers into
 *      oracle/_ref/libteamrec_ref.so (oracle/ref_driver.cpp), compared on
 *      the synthetic recipes.
 * Build with default x86-64 flags and -ffp-contract=off: the
 * tracker is FMA-sensitive.
 *
 * Struct layouts are shared with the product ABI (include/trb.h).
 */
#ifndef TRB_ORACLE_H_
#define TRB_ORACLE_H_

#include <stdint.h>

#include "../include/trb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- motion (motion.hpp:127-212) ---- */
typedef struct orc_motion orc_motion;
orc_motion* orc_motion_create(const trb_motion_config* cfg, int width, int height);
void orc_motion_destroy(orc_motion* m);
/* returns 1 when a mask was written, 0 while the window fills */
int orc_motion_push(orc_motion* m, const uint8_t* gray, uint8_t* mask_out);
void orc_motion_background(const orc_motion* m, uint8_t* out);
uint8_t orc_window_background(const uint8_t* vals, int n, int method, int bins);
/* luma / grayscale (frame.hpp:91-104) */
void orc_grayscale(const uint8_t* rgb, int64_t n_px, uint8_t* out);
/* 3x3 morphology (NOT in the reference; north-star kernel (2)).  Rule:
 * out-of-image neighbours are ignored (erode = AND, dilate = OR over the
 * in-bounds 3x3 neighbourhood).  Parity unpinned by the reference. */
void orc_morph(const uint8_t* in, int width, int height, int op, uint8_t* out);

/* ---- labelling (segmentation.hpp:88-264) ----
 * Returns the number of blobs; labels (w*h) and blobs (cap) are written.
 * Independent algorithm (BFS flood fill seeded in raster order), same
 * output contract as finalize_labels.  pixels (nullable) receives the
 * concatenated per-blob raster pixel lists. */
int orc_label(const uint8_t* mask, int width, int height, int connectivity, int min_area, int32_t* labels,
              trb_blob* blobs, int cap, int64_t* pixels);

/* warp_frame (motion.hpp:81-119): inverse-mapped bilinear resampling under
 * the homography h9 (row-major 3x3), samples off the source read 0.
 * Returns 0, or 1 non-finite entry, 2 h[2][2] == 0, 3 not invertible
 * (the reference's InvalidArgument cases). */
int orc_warp_frame(const uint8_t* in, int width, int height, int channels, const double* h9, uint8_t* out);

/* extract_blob_features (segmentation.hpp:266-291): per blob the mean
 * intensity (luma for RGB frames; the double sum of byte values is exact)
 * and the bbox aspect (width / height).  Returns -1 when the label image
 * and the frame sizes differ (InvalidArgument). */
int orc_blob_features(const int32_t* labels, int width, int height, const uint8_t* frame, int frame_width,
                      int frame_height, int channels, const trb_blob* blobs, int n_blobs, double* mean_intensity,
                      double* aspect);

/* ---- quantizer / tracker (quantize.hpp, tracking.hpp) ---- */
void orc_quantize_colors(const double* pixels /* n*3 */, int64_t n, int k, int iters, uint64_t seed,
                         double* centers /* k*3 out */);
int orc_quantizer_assign(const double* centers, int k, double r, double g, double b);
/* histogram_opt (tracking.hpp:79-102): returns 0 for nullopt */
int orc_histogram(const uint8_t* frame, int width, int height, int channels, double cx, double cy, int w, int h,
                  const double* centers, int k, int epanechnikov, double* hist);
uint64_t orc_mix_seed(uint64_t seed, uint64_t salt);

typedef struct orc_tracker orc_tracker;
orc_tracker* orc_tracker_create(const trb_tracker_config* cfg);
void orc_tracker_destroy(orc_tracker* t);
void orc_tracker_process(orc_tracker* t, const uint8_t* frame, int width, int height, int channels,
                         const trb_blob* blobs, int n_blobs);
int orc_tracker_num_tracks(const orc_tracker* t);
void orc_tracker_tracks(const orc_tracker* t, trb_track* out);
void orc_tracker_track_model(const orc_tracker* t, int i, double* centers, double* hist);
int64_t orc_tracker_log_size(const orc_tracker* t);
void orc_tracker_log(const orc_tracker* t, trb_track_log_entry* out);
/* meanshift_step on an explicit track (tracking.hpp:125-157); status in/out */
void orc_meanshift_step(const uint8_t* frame, int width, int height, int channels, double* cx, double* cy, int w,
                        int h, const double* centers, const double* target, int k, int max_iters, double eps,
                        int* status);

/* ---- synthetic clips (synth.hpp:45-101) ----
 * shapes: n * {w, h, c0, c1, c2} int32 and n * {x0, y0, vx, vy, jitter}
 * doubles.  Writes frame t into out (w*h*channels) and the per-shape
 * integer top-left corners into rects (n*4: ix, iy, w, h) when not NULL.
 * Returns 0, or -1 when a shape leaves the frame.  Rng draws (jitter) are
 * consumed per frame in order, so frames must be generated t = 0,1,2,...
 * through one orc_synth handle. */
typedef struct orc_synth orc_synth;
orc_synth* orc_synth_create(int width, int height, int channels, uint8_t background, int n_shapes,
                            const int32_t* shape_int, const double* shape_dbl, uint64_t seed);
void orc_synth_destroy(orc_synth* s);
int orc_synth_next(orc_synth* s, uint8_t* out, int32_t* rects);

/* libm hypot (what std::hypot resolves to); tests pin the product's
 * device replica of glibc's algorithm against it. */
double orc_libm_hypot(double x, double y);
void orc_libm_hypot_n(const double* x, const double* y, int64_t n, double* out);
/* plane_hash.h digest of n bytes (test infrastructure: GPU planes vs the
 * reference's, oracle/ref_driver.cpp ref_run_streams_detail) */
uint64_t orc_plane_hash(const void* data, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* TRB_ORACLE_H_ */
