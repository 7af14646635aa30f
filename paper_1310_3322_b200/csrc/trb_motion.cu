// trb_motion.cu — north-star kernel (1): fused background-model update,
// frame differencing and thresholding; plus the Mode estimator, the 3x3
// morphology stage (north-star (2)) and the synthetic-frame rasteriser.
//
// Reference: MotionDetector::push (motion.hpp:164-193), window_background
// (motion.hpp:127-144), luma (frame.hpp:91-93).
//
// HBM layout (per stream, all frame-major so every access is a coalesced
// 16-byte vector stream):
//   ring  [W][px] u8   slot = frames_seen % W (the reference keeps the same
//                      samples pixel-major, ring_[p*W+slot], motion.hpp:173)
//   sums  [px]    u16 when W <= 257 (255*257 < 2^16), else u32
//   mask  [px]    u8 0/1
// Algorithmic bytes per pixel per frame (Mean, gray): frame 1 + evicted
// sample 1 + new sample 1 + sum 2+2 + mask 1 = 8.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "trb_kernels.cuh"

namespace trb {

namespace {

__device__ __forceinline__ uint32_t luma3(uint32_t r, uint32_t g, uint32_t b) {
  return (77u * r + 150u * g + 29u * b + 128u) >> 8;  // frame.hpp:92
}

// Load 16 consecutive pixels of the input frame as gray bytes.
template <int CH>
__device__ __forceinline__ void load16(const uint8_t* __restrict__ f, int64_t p0, uint8_t (&v)[16]) {
  if constexpr (CH == 1) {
    const uint4 q = __ldcs(reinterpret_cast<const uint4*>(f + p0));
    const uint8_t* b = reinterpret_cast<const uint8_t*>(&q);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = b[i];
  } else {
    uint4 q[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) q[j] = __ldcs(reinterpret_cast<const uint4*>(f + 3 * p0) + j);
    const uint8_t* b = reinterpret_cast<const uint8_t*>(q);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = static_cast<uint8_t>(luma3(b[3 * i], b[3 * i + 1], b[3 * i + 2]));
  }
}

template <int CH>
__device__ __forceinline__ uint8_t load1(const uint8_t* __restrict__ f, int64_t p) {
  if constexpr (CH == 1) return f[p];
  return static_cast<uint8_t>(luma3(f[3 * p], f[3 * p + 1], f[3 * p + 2]));
}

__device__ __forceinline__ uint8_t thr_mask(uint32_t v, uint32_t bg, int thr) {
  const int diff = static_cast<int>(v) - static_cast<int>(bg);
  return (diff > thr || -diff > thr) ? 1 : 0;  // motion.hpp:189-190, strict
}

}  // namespace

// One thread = kMotionItems x 16 pixels (block-strided 16-pixel chunks, so
// every load / store instruction of a warp is one coalesced 512-byte run).
// grid.y = stream.
#ifndef TRB_MOTION_ITEMS
#define TRB_MOTION_ITEMS 1
#endif
constexpr int kMotionItems = TRB_MOTION_ITEMS;
template <int CH, typename SumT>
__global__ void __launch_bounds__(256) motion_mean_kernel(MotionArgs a) {
  const int s = blockIdx.y;
  const uint8_t* __restrict__ frame = a.frames[s];
  uint8_t* __restrict__ ring = a.ring + static_cast<int64_t>(s) * a.ring_stride + static_cast<int64_t>(a.slot) * a.px;
  SumT* __restrict__ sums = reinterpret_cast<SumT*>(a.sums) + static_cast<int64_t>(s) * a.px;
  uint8_t* __restrict__ mask = a.mask + static_cast<int64_t>(s) * a.px;
#pragma unroll
  for (int item = 0; item < kMotionItems; ++item) {
  const int64_t chunk = (static_cast<int64_t>(blockIdx.x) * kMotionItems + item) * blockDim.x + threadIdx.x;
  const int64_t p0 = chunk * 16;
  if (p0 >= a.px) return;
  if (p0 + 16 <= a.px && a.vec_ok) {
    uint8_t v[16];
    load16<CH>(frame, p0, v);
    uint4 old_q = make_uint4(0, 0, 0, 0);
    if (a.full_before) old_q = __ldcs(reinterpret_cast<const uint4*>(ring + p0));
    const uint8_t* old = reinterpret_cast<const uint8_t*>(&old_q);
    uint4 new_q;
    uint8_t* nb = reinterpret_cast<uint8_t*>(&new_q);
#pragma unroll
    for (int i = 0; i < 16; ++i) nb[i] = v[i];
    __stcs(reinterpret_cast<uint4*>(ring + p0), new_q);
    constexpr int kSumVec = 16 * sizeof(SumT) / 16;
    uint4 sq[kSumVec];
#pragma unroll
    for (int j = 0; j < kSumVec; ++j) sq[j] = __ldcs(reinterpret_cast<const uint4*>(sums + p0) + j);
    SumT* sv = reinterpret_cast<SumT*>(sq);
    uint4 mq;
    uint8_t* mb = reinterpret_cast<uint8_t*>(&mq);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t sum = static_cast<uint32_t>(sv[i]) - old[i] + v[i];
      sv[i] = static_cast<SumT>(sum);
      uint32_t bg;
      if constexpr (sizeof(SumT) == 2) bg = a.div.div(2u * sum + a.W);
      else bg = static_cast<uint32_t>((2ull * sum + a.W) / (2ull * a.W));
      mb[i] = thr_mask(v[i], bg, a.threshold);
    }
#pragma unroll
    for (int j = 0; j < kSumVec; ++j) __stcs(reinterpret_cast<uint4*>(sums + p0) + j, sq[j]);
    if (a.emit) __stcs(reinterpret_cast<uint4*>(mask + p0), mq);
  } else {
    const int64_t p1 = min(p0 + 16, a.px);
    for (int64_t p = p0; p < p1; ++p) {
      const uint8_t v = load1<CH>(frame, p);
      const uint8_t old = a.full_before ? ring[p] : 0;
      ring[p] = v;
      const uint32_t sum = static_cast<uint32_t>(sums[p]) - old + v;
      sums[p] = static_cast<SumT>(sum);
      if (a.emit) {
        const uint32_t bg = static_cast<uint32_t>((2ull * sum + a.W) / (2ull * a.W));
        mask[p] = thr_mask(v, bg, a.threshold);
      }
    }
  }
  }
}

// ---- bulk-async variant (gray frames, u16 sums: the C5 workload) ----
// Persistent CTAs stream tiles of kBulkTile pixels through shared memory
// with the Blackwell bulk-copy engine: one thread issues cp.async.bulk loads
// of the next tile's frame / evicted ring samples / sums (completion counted
// on an mbarrier) while the CTA computes the current tile from shared memory,
// then bulk-stores the new ring samples (the frame tile itself), sums and
// mask.  Two stages; a load into a stage waits for the stores that last read
// it (cp.async.bulk.wait_group.read).
constexpr int kBulkThreads = 256;
constexpr int kBulkTile = 16 * kBulkThreads;  // pixels per tile (16 per thread)
struct BulkStage {
  alignas(128) uint8_t frame[kBulkTile];
  alignas(128) uint8_t ring[kBulkTile];
  alignas(128) uint16_t sums[kBulkTile];
  alignas(128) uint8_t mask[kBulkTile];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void __launch_bounds__(kBulkThreads) motion_mean_bulk_kernel(MotionArgs a, int tiles_per_stream,
                                                                        int n_tiles) {
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  BulkStage* stage = reinterpret_cast<BulkStage*>(bulk_smem);
  __shared__ __align__(8) uint64_t bar[2];
  const int t = threadIdx.x;
  auto tile_of = [&](int i, int& s, int64_t& p0, uint32_t& n) {
    s = i / tiles_per_stream;
    p0 = static_cast<int64_t>(i - s * tiles_per_stream) * kBulkTile;
    n = static_cast<uint32_t>(min(static_cast<int64_t>(kBulkTile), a.px - p0));
  };
  auto issue = [&](int i, int st) {  // loads of tile i into stage st (one thread)
    int s;
    int64_t p0;
    uint32_t n;
    tile_of(i, s, p0, n);
    const uint32_t bytes = n * (a.full_before ? 4u : 3u);
    mbar_expect_tx(&bar[st], bytes);
    bulk_load(stage[st].frame, a.frames[s] + p0, n, &bar[st]);
    if (a.full_before)
      bulk_load(stage[st].ring, a.ring + static_cast<int64_t>(s) * a.ring_stride + static_cast<int64_t>(a.slot) * a.px + p0,
                n, &bar[st]);
    bulk_load(stage[st].sums, reinterpret_cast<const uint16_t*>(a.sums) + static_cast<int64_t>(s) * a.px + p0, 2 * n,
              &bar[st]);
  };
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int k = 0;  // tiles this CTA processed
  if (t == 0 && static_cast<int>(blockIdx.x) < n_tiles) issue(blockIdx.x, 0);
  for (int i = blockIdx.x; i < n_tiles; i += gridDim.x, ++k) {
    const int st = k & 1;
    if (t == 0) {
      const int nx = i + gridDim.x;
      if (nx < n_tiles) {
        bulk_wait_read0();  // the stores of the previous tile (other stage) have read their smem
        issue(nx, st ^ 1);
      }
    }
    mbar_wait(&bar[st], (k >> 1) & 1);
    int s;
    int64_t p0;
    uint32_t n;
    tile_of(i, s, p0, n);
    BulkStage& S = stage[st];
    const uint32_t q0 = 16u * t;
    if (q0 < n) {
      const uint4 fq = *reinterpret_cast<const uint4*>(S.frame + q0);
      const uint8_t* v = reinterpret_cast<const uint8_t*>(&fq);
      uint4 oq = make_uint4(0, 0, 0, 0);
      if (a.full_before) oq = *reinterpret_cast<const uint4*>(S.ring + q0);
      const uint8_t* old = reinterpret_cast<const uint8_t*>(&oq);
      uint4 sq[2];
      sq[0] = *reinterpret_cast<const uint4*>(S.sums + q0);
      sq[1] = *reinterpret_cast<const uint4*>(S.sums + q0 + 8);
      uint16_t* sv = reinterpret_cast<uint16_t*>(sq);
      uint4 mq;
      uint8_t* mb = reinterpret_cast<uint8_t*>(&mq);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t sum = static_cast<uint32_t>(sv[j]) - old[j] + v[j];
        sv[j] = static_cast<uint16_t>(sum);
        mb[j] = thr_mask(v[j], a.div.div(2u * sum + a.W), a.threshold);
      }
      *reinterpret_cast<uint4*>(S.sums + q0) = sq[0];
      *reinterpret_cast<uint4*>(S.sums + q0 + 8) = sq[1];
      *reinterpret_cast<uint4*>(S.mask + q0) = mq;
    }
    fence_proxy_async();  // this thread's smem writes -> visible to the bulk (async proxy) reads
    __syncthreads();
    if (t == 0) {
      bulk_store(a.ring + static_cast<int64_t>(s) * a.ring_stride + static_cast<int64_t>(a.slot) * a.px + p0, S.frame, n);
      bulk_store(reinterpret_cast<uint16_t*>(a.sums) + static_cast<int64_t>(s) * a.px + p0, S.sums, 2 * n);
      if (a.emit) bulk_store(a.mask + static_cast<int64_t>(s) * a.px + p0, S.mask, n);
      bulk_commit();
    }
  }
  if (t == 0) bulk_wait0();  // every store has landed before the kernel ends
}

// Mode estimator (window_background Mode path, motion.hpp:134-143): per
// pixel histogram of the W ring samples into `bins` equal bins, most
// populated bin (strict >, lower bin wins ties), rounded mean of that bin's
// samples.  Per-thread bin counters live in shared memory ([bin][thread]
// so lanes never conflict).  One thread = one pixel.
__global__ void __launch_bounds__(64) motion_mode_kernel(ModeArgs a) {
  extern __shared__ uint16_t counts[];  // [bins][64]
  const int s = blockIdx.y;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint8_t* ring = a.ring + static_cast<int64_t>(s) * a.ring_stride;
  const int t = threadIdx.x;
  for (int b = 0; b < a.bins; ++b) counts[b * 64 + t] = 0;
  if (p >= a.px) return;
  for (int i = 0; i < a.W; ++i) {
    const uint32_t v = ring[static_cast<int64_t>(i) * a.px + p];
    counts[((v * a.bins) >> 8) * 64 + t] += 1;
  }
  int best = 0;
  uint32_t bestc = counts[t];
  for (int b = 1; b < a.bins; ++b) {
    const uint32_t c = counts[b * 64 + t];
    if (c > bestc) bestc = c, best = b;
  }
  uint64_t sum = 0, cnt = 0;
  for (int i = 0; i < a.W; ++i) {
    const uint32_t v = ring[static_cast<int64_t>(i) * a.px + p];
    if (static_cast<int>((v * a.bins) >> 8) == best) sum += v, ++cnt;
  }
  const uint32_t bg = static_cast<uint32_t>((2 * sum + cnt) / (2 * cnt));
  if (a.bg_out) {
    a.bg_out[static_cast<int64_t>(s) * a.px + p] = static_cast<uint8_t>(bg);
    return;
  }
  // the newest sample sits in slot a.newest
  const uint32_t v = ring[static_cast<int64_t>(a.newest) * a.px + p];
  a.mask[static_cast<int64_t>(s) * a.px + p] = thr_mask(v, bg, a.threshold);
}

// Incremental Mode push (one thread per pixel).  The evicted sample leaves
// its bin, the new one enters its bin; the mode bin m (argmax, strict >, the
// lowest bin wins ties) changes only if the new sample's bin overtakes it
// (compare), or if m itself lost a sample to another bin (rescan of the
// pixel's `bins` counters — bin-major planes, so a warp's rescan loads are
// coalesced).  Background = rounded mean of the mode bin's samples,
// (2*sum + cnt) / (2*cnt) as window_background (motion.hpp:142-143); the mask
// is |v - bg| > threshold (:189-190).  Per push ~12 B/px plus 1 B per bin
// for the pixels that rescan, instead of the W-byte ring re-read.
// P pixels per thread (block-strided, so every load instruction of a warp
// is one coalesced run), in three rounds per thread: (1) the samples, the
// evicted ring samples and the mode bins of all P pixels; (2) every touched
// counter of all P pixels — no store before the last load, so the loads of
// a round are all in flight together (the kernel is latency-bound: two
// dependent DRAM round trips per pixel); (3) arithmetic with the aliasing
// between the old, new and mode bins resolved in registers, the rare
// rescans, and the stores — counters, mode bin and ring slot only where
// they change.
// floor(n / d) for n < 2^17, 1 <= d < 2^9 (the Mode background's rounded
// mean): a float reciprocal estimate and one correction step each way.
__device__ __forceinline__ uint32_t div_small(uint32_t n, uint32_t d) {
  uint32_t q = static_cast<uint32_t>(__fmul_rz(static_cast<float>(n), __frcp_rn(static_cast<float>(d))));
  if (q * d > n) --q;
  if ((q + 1) * d <= n) ++q;
  return q;
}

// One pixel's push given its loaded state: sample v, evicted sample old, mode
// bin m0 and the counters of the new / mode / evicted bins (c_m / s_m valid
// when m0 != bn, c_bo / s_bo when bo differs from both).  Stores the changed
// counters (the rare rescan loads the pixel's other bins) and returns the
// new mode bin with its count and sum.
struct ModeOut {
  uint32_t mm;
  int cm;
  uint32_t sm;
};
__device__ __forceinline__ ModeOut mode_push(uint32_t v, uint32_t old, uint32_t m0, int cbn, uint32_t sbn, int cm,
                                             uint32_t sm_, int cbo, uint32_t sbo, bool full, uint32_t nb,
                                             uint8_t* __restrict__ cnt, uint16_t* __restrict__ bsum, int64_t px,
                                             int64_t p) {
  const uint32_t bn = (v * nb) >> 8, bo = (old * nb) >> 8;
  if (m0 == bn) cm = cbn, sm_ = sbn;
  if (full && bo != bn && bo == m0) cbo = cm, sbo = sm_;
  const bool moved = !full || bo != bn;  // counts change
  if (!moved) {
    sbn = sbn + v - old;
  } else {
    if (full) cbo -= 1, sbo -= old;
    cbn += 1, sbn += v;
  }
  if (m0 == bn) cm = cbn, sm_ = sbn;
  if (full && m0 == bo && bo != bn) cm = cbo, sm_ = sbo;
  uint32_t mm = m0;
  if (full && bo != bn && bo == m0) {  // the mode bin lost a sample: rescan (new values for bo / bn)
    uint32_t best = 0;
    int bc = -1;
#pragma unroll 8
    for (uint32_t b = 0; b < nb; ++b) {
      const int c = b == bo ? cbo : (b == bn ? cbn : cnt[b * px + p]);
      if (c > bc) bc = c, best = b;
    }
    mm = best, cm = bc;
    sm_ = mm == bo ? sbo : (mm == bn ? sbn : bsum[mm * px + p]);
  } else if (moved && bn != m0 && (cbn > cm || (cbn == cm && bn < m0))) {
    mm = bn, cm = cbn, sm_ = sbn;
  }
  if (moved) cnt[bn * px + p] = static_cast<uint8_t>(cbn);
  if (moved || v != old) bsum[bn * px + p] = static_cast<uint16_t>(sbn);
  if (full && bo != bn) cnt[bo * px + p] = static_cast<uint8_t>(cbo), bsum[bo * px + p] = static_cast<uint16_t>(sbo);
  return ModeOut{mm, cm, sm_};
}

// The touched counters of one pixel (round 2 of the kernels below).
__device__ __forceinline__ void mode_loads(uint32_t v, uint32_t old, uint32_t m, bool full, uint32_t nb,
                                           const uint8_t* __restrict__ cnt, const uint16_t* __restrict__ bsum,
                                           int64_t px, int64_t p, int& c_bn, uint32_t& s_bn, int& c_m,
                                           uint32_t& s_m, int& c_bo, uint32_t& s_bo) {
  const uint32_t bn = (v * nb) >> 8, bo = (old * nb) >> 8;
  c_m = c_bo = 0, s_m = s_bo = 0;
  c_bn = cnt[bn * px + p], s_bn = bsum[bn * px + p];
  if (m != bn) c_m = cnt[m * px + p], s_m = bsum[m * px + p];
  if (full && bo != bn && bo != m) c_bo = cnt[bo * px + p], s_bo = bsum[bo * px + p];
}

template <int CH, int P>
__global__ void __launch_bounds__(256) motion_mode_inc_kernel(ModeIncArgs a) {
  const int s = blockIdx.y;
  // (64-bit offsets: 32-bit ones measured 10-25 % slower — extra widening per address)
  using Off = int64_t;
  const Off px = a.px;
  const Off base = static_cast<Off>(blockIdx.x) * 256 * P + threadIdx.x;
  uint8_t* __restrict__ ring = a.ring + static_cast<int64_t>(s) * a.ring_stride + static_cast<int64_t>(a.slot) * px;
  uint8_t* __restrict__ cnt = a.cnt + static_cast<int64_t>(s) * a.bins * px;
  uint16_t* __restrict__ bsum = a.bsum + static_cast<int64_t>(s) * a.bins * px;
  uint8_t* __restrict__ mode = a.mode + static_cast<int64_t>(s) * px;
  uint8_t* __restrict__ mask = a.mask + static_cast<int64_t>(s) * px;
  const uint8_t* __restrict__ frame = a.frames[s];
  const bool full = a.full_before != 0;
  const uint32_t nb = static_cast<uint32_t>(a.bins);
  uint32_t v[P], old[P];
  uint32_t m[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const Off p = base + k * 256;
    v[k] = 0, old[k] = 0, m[k] = 0;
    if (p < px) {
      v[k] = load1<CH>(frame, p);
      if (full) old[k] = ring[p];
      m[k] = mode[p];
    }
  }
  int c_bn[P], c_m[P], c_bo[P];
  uint32_t s_bn[P], s_m[P], s_bo[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const Off p = base + k * 256;
    if (p < px) mode_loads(v[k], old[k], m[k], full, nb, cnt, bsum, px, p, c_bn[k], s_bn[k], c_m[k], s_m[k], c_bo[k], s_bo[k]);
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const Off p = base + k * 256;
    if (p >= px) continue;
    const ModeOut o = mode_push(v[k], old[k], m[k], c_bn[k], s_bn[k], c_m[k], s_m[k], c_bo[k], s_bo[k], full, nb, cnt,
                                bsum, px, p);
    if (o.mm != m[k]) mode[p] = static_cast<uint8_t>(o.mm);
    if (!full || v[k] != old[k]) ring[p] = static_cast<uint8_t>(v[k]);
    if (a.emit) {
      const uint32_t bg = div_small(2 * o.sm + static_cast<uint32_t>(o.cm), 2 * static_cast<uint32_t>(o.cm));
      mask[p] = thr_mask(v[k], bg, a.threshold);
    }
  }
}

// Ring update only (Mode path): write the new sample, keep the sums.
template <int CH, typename SumT>
__global__ void __launch_bounds__(256) ring_update_kernel(MotionArgs a) {
  const int s = blockIdx.y;
  const uint8_t* __restrict__ frame = a.frames[s];
  uint8_t* __restrict__ ring = a.ring + static_cast<int64_t>(s) * a.ring_stride + static_cast<int64_t>(a.slot) * a.px;
  SumT* __restrict__ sums = reinterpret_cast<SumT*>(a.sums) + static_cast<int64_t>(s) * a.px;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= a.px) return;
  const uint8_t v = load1<CH>(frame, p);
  const uint8_t old = a.full_before ? ring[p] : 0;
  ring[p] = v;
  sums[p] = static_cast<SumT>(static_cast<uint32_t>(sums[p]) - old + v);
}

// Mean background image from the sums (MotionDetector::background, :196-203).
template <typename SumT>
__global__ void mean_background_kernel(const void* sums_v, int64_t px, int W, uint8_t* out) {
  const SumT* sums = reinterpret_cast<const SumT*>(sums_v);
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= px) return;
  out[p] = static_cast<uint8_t>((2ull * sums[p] + W) / (2ull * W));
}

// 3x3 binary erosion / dilation (north-star kernel (2); not in the
// reference).  Out-of-image neighbours are ignored.  One CTA = 32x8 output
// pixels; the (32+2)x(8+2) input tile with halo is staged in shared memory.
__global__ void __launch_bounds__(256) morph3x3_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                                      int w, int h, int64_t stride, int dilate) {
  __shared__ uint8_t tile[10][34];
  const int s = blockIdx.z;
  in += static_cast<int64_t>(s) * stride;
  out += static_cast<int64_t>(s) * stride;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
  const uint8_t pad = dilate ? 0 : 1;  // neutral element for ignored neighbours
  for (int i = threadIdx.x; i < 10 * 34; i += blockDim.x) {
    const int ty = i / 34, tx = i % 34;
    const int gx = x0 + tx - 1, gy = y0 + ty - 1;
    tile[ty][tx] = (gx >= 0 && gy >= 0 && gx < w && gy < h) ? (in[static_cast<int64_t>(gy) * w + gx] != 0) : pad;
  }
  __syncthreads();
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int gx = x0 + tx, gy = y0 + ty;
  if (gx >= w || gy >= h) return;
  uint32_t acc = dilate ? 0u : 1u;
#pragma unroll
  for (int dy = 0; dy < 3; ++dy)
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      const uint32_t v = tile[ty + dy][tx + dx];
      acc = dilate ? (acc | v) : (acc & v);
    }
  out[static_cast<int64_t>(gy) * w + gx] = static_cast<uint8_t>(acc);
}

// Row-strip 3x3 morphology for widths that are a multiple of 16 (the HBM
// path): a lane owns a 16-pixel column block (one 16-byte vector per row)
// and walks a strip of kStripRows rows with a sliding window, so each mask
// byte is read ~(R+4)/R times and written once.  The horizontal 3-tap runs
// on two u64 words with byte shifts; the neighbours' edge bytes come from
// the adjacent lanes (__shfl), so a warp covers 32 blocks but stores only
// its 30 inner ones (lanes 0 and 31 are halo).  OP: 0 erode, 1 dilate,
// 2 open (erode then dilate), 3 close (dilate then erode) — the two-stage
// ops run fused (the eroded rows never leave registers).  Out-of-image
// neighbours are ignored (neutral element), as morph3x3_kernel.
#ifndef TRB_MORPH_ROWS
#define TRB_MORPH_ROWS 8
#endif
constexpr int kStripRows = TRB_MORPH_ROWS;
constexpr uint64_t kOnes = 0x0101010101010101ull;

template <bool AND>
__device__ __forceinline__ uint64_t bop(uint64_t a, uint64_t b) {
  return AND ? (a & b) : (a | b);
}

// horizontal 3-tap over this lane's 16 bytes (all 32 lanes must call it)
template <bool AND>
__device__ __forceinline__ void horiz3(uint64_t& lo, uint64_t& hi, int lane) {
  const uint64_t nb = AND ? 1ull : 0ull;
  uint64_t lb = __shfl_up_sync(0xffffffffu, hi >> 56, 1);
  uint64_t rb = __shfl_down_sync(0xffffffffu, lo & 0xffull, 1);
  if (lane == 0) lb = nb;
  if (lane == 31) rb = nb;
  const uint64_t l_lo = (lo << 8) | lb, l_hi = (hi << 8) | (lo >> 56);
  const uint64_t r_lo = (lo >> 8) | (hi << 56), r_hi = (hi >> 8) | (rb << 56);
  lo = bop<AND>(bop<AND>(lo, l_lo), r_lo);
  hi = bop<AND>(bop<AND>(hi, l_hi), r_hi);
}

#ifndef TRB_MORPH_LD
#define TRB_MORPH_LD __ldg  // halo rows are re-read by the neighbouring strip: keep them in L2
#define TRB_MORPH_ST __stcs
#endif

template <int OP>
__global__ void __launch_bounds__(128) morph_strip_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                                          int w, int h, int64_t stride) {
  constexpr bool A1 = (OP == 0 || OP == 2);  // stage 1 erodes (AND) or dilates (OR)
  constexpr bool TWO = OP >= 2;
  constexpr bool A2 = (OP == 3);             // stage 2 of open dilates, of close erodes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s = blockIdx.z;
  in += s * stride;
  out += s * stride;
  const int bx = (blockIdx.x * 4 + warp) * 30 + lane - 1;  // this lane's 16-pixel block
  const bool colok = bx >= 0 && bx * 16 < w;
  const bool store = colok && lane >= 1 && lane <= 30;
  const int y0 = blockIdx.y * kStripRows, y1 = min(h, y0 + kStripRows);
  const uint64_t n1 = A1 ? kOnes : 0ull, n2 = A2 ? kOnes : 0ull;
  // horizontal stage-1 tap of raw row y (neutral outside the image)
  auto h1 = [&](int y, uint64_t& lo, uint64_t& hi) {
    lo = hi = n1;
    if (colok && y >= 0 && y < h) {
      const uint4 q = TRB_MORPH_LD(reinterpret_cast<const uint4*>(in + static_cast<int64_t>(y) * w) + bx);
      lo = (static_cast<uint64_t>(q.y) << 32) | q.x;
      hi = (static_cast<uint64_t>(q.w) << 32) | q.z;
    }
    horiz3<A1>(lo, hi, lane);
  };
  auto put = [&](int y, uint64_t lo, uint64_t hi) {
    if (store) {
      uint4 q;
      q.x = static_cast<uint32_t>(lo), q.y = static_cast<uint32_t>(lo >> 32);
      q.z = static_cast<uint32_t>(hi), q.w = static_cast<uint32_t>(hi >> 32);
      TRB_MORPH_ST(reinterpret_cast<uint4*>(out + static_cast<int64_t>(y) * w) + bx, q);
    }
  };
  uint64_t al, ah, bl, bh, cl, ch;  // stage-1 taps of rows e-1, e, e+1
  if (!TWO) {
    h1(y0 - 1, al, ah);
    h1(y0, bl, bh);
    for (int y = y0; y < y1; ++y) {
      h1(y + 1, cl, ch);
      put(y, bop<A1>(bop<A1>(al, bl), cl), bop<A1>(bop<A1>(ah, bh), ch));
      al = bl, ah = bh, bl = cl, bh = ch;
    }
  } else {
    // stage-1 rows e = y0-1 .. y1 (neutral for stage 2 outside the image),
    // each through the stage-2 horizontal tap
    auto e_row = [&](int e, uint64_t& lo, uint64_t& hi) {
      lo = bop<A1>(bop<A1>(al, bl), cl), hi = bop<A1>(bop<A1>(ah, bh), ch);
      if (!(colok && e >= 0 && e < h)) lo = hi = n2;
      horiz3<A2>(lo, hi, lane);
    };
    uint64_t pl, ph, ql, qh, rl, rh;  // stage-2 taps of stage-1 rows y-1, y, y+1
    h1(y0 - 2, al, ah);
    h1(y0 - 1, bl, bh);
    h1(y0, cl, ch);
    e_row(y0 - 1, pl, ph);
    al = bl, ah = bh, bl = cl, bh = ch;
    h1(y0 + 1, cl, ch);
    e_row(y0, ql, qh);
    for (int y = y0; y < y1; ++y) {
      al = bl, ah = bh, bl = cl, bh = ch;
      h1(y + 2, cl, ch);
      e_row(y + 1, rl, rh);
      put(y, bop<A2>(bop<A2>(pl, ql), rl), bop<A2>(bop<A2>(ph, qh), rh));
      pl = ql, ph = qh, ql = rl, qh = rh;
    }
  }
}

// Synthetic frame raster (synth.hpp:295-328): background fill, then every
// shape's rectangle in order (later shapes overwrite earlier ones).
// grid.y = frame: frame f uses rects + f*n*4 and writes out + f*frame_stride.
__global__ void synth_raster_kernel(uint8_t* out, int w, int h, int ch, uint8_t bg, const int32_t* rects,
                                    const uint8_t* colors, int n, int64_t frame_stride) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= static_cast<int64_t>(w) * h) return;
  out += frame_stride * blockIdx.y;
  rects += static_cast<int64_t>(4) * n * blockIdx.y;
  const int x = static_cast<int>(p % w), y = static_cast<int>(p / w);
  int hit = -1;
  for (int k = 0; k < n; ++k) {
    const int ix = rects[4 * k], iy = rects[4 * k + 1], rw = rects[4 * k + 2], rh = rects[4 * k + 3];
    if (x >= ix && x < ix + rw && y >= iy && y < iy + rh) hit = k;
  }
  for (int c = 0; c < ch; ++c) out[p * ch + c] = hit < 0 ? bg : colors[3 * hit + c];
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int bulk_mode() {  // TRB_MOTION_BULK=0 selects the register-streaming kernel (A/B)
  static const int m = [] {
    const char* e = getenv("TRB_MOTION_BULK");
    return e ? atoi(e) : 1;
  }();
  return m;
}

void launch_motion_mean(const MotionArgs& a, int channels, bool wide_sums, int n_streams, cudaStream_t st) {
  if (channels == 1 && !wide_sums && a.vec_ok && bulk_mode()) {
    static int grid = 0;
    const size_t smem = 2 * sizeof(BulkStage);
    if (!grid) {
      TRB_CUDA(cudaFuncSetAttribute(motion_mean_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      int per_sm = 0, sms = 0, dev = 0;
      TRB_CUDA(cudaGetDevice(&dev));
      TRB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      TRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, motion_mean_bulk_kernel, kBulkThreads, smem));
      // a few CTAs per SM keep enough bytes in flight (2 stages x 20 KB each)
      // and leave the SMs' shared memory to the tracker of the previous step,
      // which runs concurrently (step overlap)
      const char* e = getenv("TRB_MOTION_BULK_CTAS");
      grid = std::max(1, std::min(per_sm, e ? atoi(e) : 3)) * sms;  // A/B: 1 -> 63 %, 2 -> 87 %, 3 -> 93 % of the measured copy peak
    }
    const int tiles_per_stream = static_cast<int>(ceil_div64(a.px, kBulkTile));
    const int n_tiles = tiles_per_stream * n_streams;
    motion_mean_bulk_kernel<<<std::min(grid, n_tiles), kBulkThreads, smem, st>>>(a, tiles_per_stream, n_tiles);
    TRB_LAUNCH_CHECK("motion_mean_bulk_kernel");
    return;
  }
  const int64_t chunks = ceil_div64(a.px, 16);
  dim3 grid(static_cast<unsigned>(ceil_div64(chunks, 256 * kMotionItems)), n_streams);
  if (channels == 1) {
    if (wide_sums) motion_mean_kernel<1, uint32_t><<<grid, 256, 0, st>>>(a);
    else motion_mean_kernel<1, uint16_t><<<grid, 256, 0, st>>>(a);
  } else {
    if (wide_sums) motion_mean_kernel<3, uint32_t><<<grid, 256, 0, st>>>(a);
    else motion_mean_kernel<3, uint16_t><<<grid, 256, 0, st>>>(a);
  }
  TRB_LAUNCH_CHECK("motion_mean_kernel");
}

template <int P>
static void launch_mode_inc_p(const ModeIncArgs& a, int channels, int n_streams, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div64(a.px, 256 * P)), n_streams);
  if (channels == 1) motion_mode_inc_kernel<1, P><<<grid, 256, 0, st>>>(a);
  else motion_mode_inc_kernel<3, P><<<grid, 256, 0, st>>>(a);
}

void launch_motion_mode_inc(const ModeIncArgs& a, int channels, int n_streams, cudaStream_t st) {
  static const int pix = [] {  // pixels per thread (A/B knob)
    // A/B (C5MODE): 2 ahead of 1, 4, 8; 4 CONSECUTIVE pixels with 32-bit
    // sample / ring / mode / mask words measured 1.9x slower (the per-pixel
    // counter accesses then spread over 4x the sectors per warp instruction)
    const char* e = getenv("TRB_MODE_PIX");
    return e ? atoi(e) : 2;
  }();
  if (pix == 1) launch_mode_inc_p<1>(a, channels, n_streams, st);
  else if (pix == 2) launch_mode_inc_p<2>(a, channels, n_streams, st);
  else if (pix == 8) launch_mode_inc_p<8>(a, channels, n_streams, st);
  else launch_mode_inc_p<4>(a, channels, n_streams, st);
  TRB_LAUNCH_CHECK("motion_mode_inc_kernel");
}

void launch_ring_update(const MotionArgs& a, int channels, bool wide_sums, int n_streams, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div64(a.px, 256)), n_streams);
  if (channels == 1) {
    if (wide_sums) ring_update_kernel<1, uint32_t><<<grid, 256, 0, st>>>(a);
    else ring_update_kernel<1, uint16_t><<<grid, 256, 0, st>>>(a);
  } else {
    if (wide_sums) ring_update_kernel<3, uint32_t><<<grid, 256, 0, st>>>(a);
    else ring_update_kernel<3, uint16_t><<<grid, 256, 0, st>>>(a);
  }
  TRB_LAUNCH_CHECK("ring_update_kernel");
}

void launch_motion_mode(const ModeArgs& a, int n_streams, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div64(a.px, 64)), n_streams);
  const size_t smem = static_cast<size_t>(a.bins) * 64 * sizeof(uint16_t);
  motion_mode_kernel<<<grid, 64, smem, st>>>(a);
  TRB_LAUNCH_CHECK("motion_mode_kernel");
}

void launch_mean_background(const void* sums, int64_t px, int W, bool wide_sums, uint8_t* out, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(ceil_div64(px, 256));
  if (wide_sums) mean_background_kernel<uint32_t><<<grid, 256, 0, st>>>(sums, px, W, out);
  else mean_background_kernel<uint16_t><<<grid, 256, 0, st>>>(sums, px, W, out);
  TRB_LAUNCH_CHECK("mean_background_kernel");
}

// in -> out (distinct buffers).  Returns the number of launches.
int launch_morph(const uint8_t* in, uint8_t* out, uint8_t* scratch, int w, int h, int n_streams, int op,
                 cudaStream_t st) {
  if (op < TRB_MORPH_ERODE || op > TRB_MORPH_CLOSE) throw Error(TRB_CONFIG_ERROR, "unknown morphology op");
  const int64_t stride = static_cast<int64_t>(w) * h;
  if (w % 16 == 0) {  // HBM path: one fused launch for every op
    const int warps_per_row = ceil_div(w / 16, 30);
    dim3 grid(ceil_div(warps_per_row, 4), ceil_div(h, kStripRows), n_streams);
    switch (op) {
      case TRB_MORPH_ERODE: morph_strip_kernel<0><<<grid, 128, 0, st>>>(in, out, w, h, stride); break;
      case TRB_MORPH_DILATE: morph_strip_kernel<1><<<grid, 128, 0, st>>>(in, out, w, h, stride); break;
      case TRB_MORPH_OPEN: morph_strip_kernel<2><<<grid, 128, 0, st>>>(in, out, w, h, stride); break;
      default: morph_strip_kernel<3><<<grid, 128, 0, st>>>(in, out, w, h, stride); break;
    }
    TRB_LAUNCH_CHECK("morph_strip_kernel");
    return 1;
  }
  dim3 grid(ceil_div(w, 32), ceil_div(h, 8), n_streams);
  auto pass = [&](const uint8_t* src, uint8_t* dst, int dilate) {
    morph3x3_kernel<<<grid, 256, 0, st>>>(src, dst, w, h, stride, dilate);
    TRB_LAUNCH_CHECK("morph3x3_kernel");
  };
  switch (op) {
    case TRB_MORPH_ERODE: pass(in, out, 0); return 1;
    case TRB_MORPH_DILATE: pass(in, out, 1); return 1;
    case TRB_MORPH_OPEN: pass(in, scratch, 0); pass(scratch, out, 1); return 2;
    default: pass(in, scratch, 1); pass(scratch, out, 0); return 2;
  }
}

// ------------------------------------------------------------------- warp
// warp_frame (motion.hpp:81-119): inverse-mapped bilinear resampling, one
// thread per output pixel (all channels).  The inverse is computed on the
// host with the reference's cofactor expressions; here every fp64 op is an
// explicit round-to-nearest intrinsic in the reference's left-to-right
// order (no contraction), floor / lround as std::floor / std::lround.
__global__ void __launch_bounds__(256) warp_frame_kernel(const uint8_t* const* in, int64_t in_stride,
                                                         uint8_t* out, const double* invs, int w, int h, int ch) {
  const int s = blockIdx.y;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= static_cast<int64_t>(w) * h) return;
  const uint8_t* f = in[s];
  uint8_t* o = out + in_stride * s;
  const double* inv = invs + 9 * s;
  const int y = static_cast<int>(p / w), x = static_cast<int>(p - static_cast<int64_t>(y) * w);
  const double xd = x, yd = y;
  const double ww = __dadd_rn(__dadd_rn(__dmul_rn(inv[6], xd), __dmul_rn(inv[7], yd)), inv[8]);
  if (fabs(ww) < 1e-12) {  // projects to infinity; stays 0
    for (int c = 0; c < ch; ++c) o[p * ch + c] = 0;
    return;
  }
  const double sx = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(inv[0], xd), __dmul_rn(inv[1], yd)), inv[2]), ww);
  const double sy = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(inv[3], xd), __dmul_rn(inv[4], yd)), inv[5]), ww);
  const int x0 = __double2int_rz(floor(sx)), y0 = __double2int_rz(floor(sy));
  const double dx = __dsub_rn(sx, static_cast<double>(x0)), dy = __dsub_rn(sy, static_cast<double>(y0));
  const double ex = __dsub_rn(1.0, dx), ey = __dsub_rn(1.0, dy);
  const double w00 = __dmul_rn(ex, ey), w10 = __dmul_rn(dx, ey), w01 = __dmul_rn(ex, dy), w11 = __dmul_rn(dx, dy);
  auto tap = [&](int tx, int ty, int c) -> double {
    if (tx < 0 || ty < 0 || tx >= w || ty >= h) return 0.0;
    return f[(static_cast<int64_t>(ty) * w + tx) * ch + c];
  };
  for (int c = 0; c < ch; ++c) {
    double v = __dmul_rn(w00, tap(x0, y0, c));
    v = __dadd_rn(v, __dmul_rn(w10, tap(x0 + 1, y0, c)));
    v = __dadd_rn(v, __dmul_rn(w01, tap(x0, y0 + 1, c)));
    v = __dadd_rn(v, __dmul_rn(w11, tap(x0 + 1, y0 + 1, c)));
    const double lo = (0.0 < v) ? v : 0.0;        // std::max(0.0, v)
    const double cl = (lo < 255.0) ? lo : 255.0;  // std::min(255.0, .)
    o[p * ch + c] = static_cast<uint8_t>(llround(cl));
  }
}

// Homography::validate + the inverse of warp_frame (motion.hpp:73-95); host.
void homography_inverse(const double* hm, double* inv) {
  for (int i = 0; i < 9; ++i)
    if (!std::isfinite(hm[i])) throw Error(TRB_INVALID_ARGUMENT, "homography has a non-finite entry");
  if (hm[8] == 0.0) throw Error(TRB_INVALID_ARGUMENT, "homography is not normalizable (h[2][2] = 0)");
  auto H = [&](int r, int c) { return hm[3 * r + c]; };
  const double det = H(0, 0) * (H(1, 1) * H(2, 2) - H(1, 2) * H(2, 1)) -
                     H(0, 1) * (H(1, 0) * H(2, 2) - H(1, 2) * H(2, 0)) +
                     H(0, 2) * (H(1, 0) * H(2, 1) - H(1, 1) * H(2, 0));
  if (std::abs(det) < 1e-12) throw Error(TRB_INVALID_ARGUMENT, "homography is not invertible");
  const double r[9] = {(H(1, 1) * H(2, 2) - H(1, 2) * H(2, 1)) / det, (H(0, 2) * H(2, 1) - H(0, 1) * H(2, 2)) / det,
                       (H(0, 1) * H(1, 2) - H(0, 2) * H(1, 1)) / det, (H(1, 2) * H(2, 0) - H(1, 0) * H(2, 2)) / det,
                       (H(0, 0) * H(2, 2) - H(0, 2) * H(2, 0)) / det, (H(0, 2) * H(1, 0) - H(0, 0) * H(1, 2)) / det,
                       (H(1, 0) * H(2, 1) - H(1, 1) * H(2, 0)) / det, (H(0, 1) * H(2, 0) - H(0, 0) * H(2, 1)) / det,
                       (H(0, 0) * H(1, 1) - H(0, 1) * H(1, 0)) / det};
  for (int i = 0; i < 9; ++i) inv[i] = r[i];
}

void launch_warp_frames(const uint8_t* const* in_dev, uint8_t* out, int64_t stride, const double* invs_dev, int w,
                        int h, int ch, int n_streams, cudaStream_t st) {
  const int64_t px = static_cast<int64_t>(w) * h;
  dim3 grid(static_cast<unsigned>(ceil_div64(px, 256)), n_streams);
  warp_frame_kernel<<<grid, 256, 0, st>>>(in_dev, stride, out, invs_dev, w, h, ch);
  TRB_LAUNCH_CHECK("warp_frame_kernel");
}

void launch_synth_raster(uint8_t* out, int w, int h, int ch, uint8_t bg, const int32_t* rects, const uint8_t* colors,
                         int n, cudaStream_t st, int n_frames, int64_t frame_stride) {
  const int64_t px = static_cast<int64_t>(w) * h;
  dim3 grid(static_cast<unsigned>(ceil_div64(px, 256)), n_frames);
  synth_raster_kernel<<<grid, 256, 0, st>>>(out, w, h, ch, bg, rects, colors, n, frame_stride);
  TRB_LAUNCH_CHECK("synth_raster_kernel");
}

}  // namespace trb
