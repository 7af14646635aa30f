// trb_kernels.cuh — kernel argument blocks and launchers shared by the
// kernel translation units and the host engine (trb_engine.cu).
#pragma once

#include "trb_common.cuh"

namespace trb {

// ---------------------------------------------------------------- motion
struct MotionArgs {
  const uint8_t* const* frames;  // device array [n_streams] of frame pointers
  uint8_t* ring;                 // stream s ring at ring + s*ring_stride, slot plane at + slot*px
  int64_t ring_stride;
  void* sums;                    // u16 or u32 [n_streams][px]
  uint8_t* mask;                 // [n_streams][px]
  int64_t px;
  int slot;
  int full_before;  // window was already full before this push (evict)
  int emit;         // a mask is produced by this push
  int threshold;
  uint32_t W;
  FastDiv div;      // divides by 2W
  int vec_ok;       // 16-byte aligned planes
};

struct ModeArgs {
  const uint8_t* ring;
  int64_t ring_stride;
  int64_t px;
  int W, bins, threshold, newest;
  uint8_t* mask;    // [n_streams][px] (unused when bg_out is set)
  uint8_t* bg_out;  // when set: write the background image instead of the mask
};

// Incremental Mode background (window_background Mode, motion.hpp:134-143,
// maintained per push instead of re-reading the W-sample ring): per pixel
// and bin the sample count (u8, W <= 255) and sample sum (u16), and the
// current mode bin.  Planes are bin-major: cnt[s][bin][px], bsum[s][bin][px].
struct ModeIncArgs {
  const uint8_t* const* frames;
  uint8_t* ring;  // as MotionArgs
  int64_t ring_stride;
  uint8_t* cnt;
  uint16_t* bsum;
  uint8_t* mode;  // [n_streams][px]
  uint8_t* mask;
  int64_t px;
  int slot, full_before, emit, threshold, bins;
};
void launch_motion_mode_inc(const ModeIncArgs& a, int channels, int n_streams, cudaStream_t st);
void launch_motion_mean(const MotionArgs& a, int channels, bool wide_sums, int n_streams, cudaStream_t st);
void launch_ring_update(const MotionArgs& a, int channels, bool wide_sums, int n_streams, cudaStream_t st);
void launch_motion_mode(const ModeArgs& a, int n_streams, cudaStream_t st);
void launch_mean_background(const void* sums, int64_t px, int W, bool wide_sums, uint8_t* out, cudaStream_t st);
// returns the number of launches issued
int launch_morph(const uint8_t* in, uint8_t* out, uint8_t* scratch, int w, int h, int n_streams, int op,
                 cudaStream_t st);
// warp_frame (motion.hpp:81-119): host inverse (throws the reference's
// InvalidArgument messages) and the per-pixel resampling of S frames.
void homography_inverse(const double* h9, double* inv9);
void launch_warp_frames(const uint8_t* const* in_dev, uint8_t* out, int64_t stride, const double* invs_dev, int w,
                        int h, int ch, int n_streams, cudaStream_t st);
void launch_synth_raster(uint8_t* out, int w, int h, int ch, uint8_t bg, const int32_t* rects, const uint8_t* colors,
                         int n, cudaStream_t st, int n_frames = 1, int64_t frame_stride = 0);

// ------------------------------------------------------------------- CCL
// Per-stream slot table: one slot per tile-local component ("tile
// component"); the global union-find runs over slots.
struct SlotTable {
  int32_t* parent;  // union-find parent slot (min slot id is the set root)
  int32_t* root;    // resolved set root
  int32_t* area;
  int32_t* x0;
  int32_t* y0;
  int32_t* x1;
  int32_t* y1;
  unsigned long long* sx;
  unsigned long long* sy;
  int32_t* minpix;  // smallest linear pixel index (component's raster-first pixel)
  int32_t* dense;   // final label of the slot's component (0 = dropped)
};

struct CclArgs {
  const uint8_t* mask;  // [S][px]
  int32_t* labg;        // [S][px] slot id of every foreground pixel
  int32_t* labels;      // [S][px] final labels
  int w, h;
  int64_t px;
  int conn;  // TRB_CONN_*
  int min_area;
  int tiles_x, tiles_y;
  SlotTable slots;      // base pointers; stream s at + s*slot_cap
  int64_t slot_cap;
  int32_t* nslots;      // [S]
  int32_t* rowcount;    // [S][h] survivors per row, then exclusive prefix
  uint32_t* bitmap;     // [S][h][wpr] survivor root bits
  int wpr;              // bitmap words per row
  trb_blob* blobs;      // [S][blob_cap]
  int64_t blob_cap;
  int32_t* nblobs;      // [S]
  int32_t* tile_list;   // [S * tiles] tiles holding foreground (s * tiles + ty * tiles_x + tx)
  int32_t* tile_count;  // [1]
  uint8_t* tile_state;  // [S * tiles] bit 0: holds foreground this frame; bit 1: its labels may be nonzero
};

// Launches the full CCL + blob-statistics chain; returns launches issued.
int launch_ccl(const CclArgs& a, int n_streams, cudaStream_t st);
// the first bcap blobs of every stream's table into out[S][bcap]
void launch_pack_blobs(const trb_blob* blobs, int64_t stride, const int32_t* nblobs, trb_blob* out, int bcap,
                       int n_streams, cudaStream_t st);

// ------------------------------------------------------------ tracking
struct TrackerDev;  // defined in trb_track.cu
}  // namespace trb
