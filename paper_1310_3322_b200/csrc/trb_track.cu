// trb_track.cu — tracker kernels (see trb_track.cuh for the layout).
#include <algorithm>
#include <cstring>
#include <vector>

namespace trb {
// Optional hang diagnostics: host-mapped [cta][4] = {kernel, item, iter, stage}.
__device__ int* g_progress;
}  // namespace trb
namespace trb {
// Optional per-phase cycle accounting (enabled with the iteration log):
// [bucket][phase], bucket = window-size class of the iteration (<5k, <50k,
// <150k, larger pixels); thread 0 of the group's rank-0 CTA adds the cycles
// since its previous mark; [bucket][0] counts iterations.
__device__ unsigned long long g_phase[256];
__device__ int g_phase_on;
__shared__ long long s_ph_last;
__shared__ int s_ph_bucket;
__shared__ unsigned long long s_item_t0;
// per-CTA [busy ns, last item end (globaltimer)] of the mean-shift kernel
__device__ unsigned long long g_cta_time[2 * 1024];
// per (cluster rank, warp, hist/cent): sum over runs of the warp's phase-B walk cycles (8-CTA runs)
__device__ unsigned long long g_warpwalk[8 * 8 * 2];
}  // namespace trb
// The device-side instrumentation below compiles only into the diagnostics
// build (make diag -> libtrb_diag.so, -DTRB_DIAG); the product build has no
// progress/phase/iteration-log code in its kernels.
#ifdef TRB_DIAG
#define TRB_PHASE(k, rank_, G_)                                                                   \
  do {                                                                                            \
    if (::trb::g_phase_on && threadIdx.x == 0 && (rank_) == 0) {                                  \
      const long long n_ = clock64();                                                             \
      if ((k) >= 0) atomicAdd(&::trb::g_phase[(k) + 64 * ::trb::s_ph_bucket], n_ - ::trb::s_ph_last); \
      ::trb::s_ph_last = n_;                                                                      \
    }                                                                                             \
  } while (0)
#define TRB_PHASE_BEGIN(n_px, rank_)                                                              \
  do {                                                                                            \
    if (::trb::g_phase_on && threadIdx.x == 0 && (rank_) == 0) {                                  \
      const int b_ = (n_px) < 5000 ? 0 : (n_px) < 50000 ? 1 : (n_px) < 150000 ? 2 : 3;            \
      ::trb::s_ph_bucket = b_;                                                                    \
      atomicAdd(&::trb::g_phase[64 * b_], 1ull);                                                  \
      ::trb::s_ph_last = clock64();                                                               \
    }                                                                                             \
  } while (0)
// per-thread phase-B walk cycles of rank-0 CTAs: [40 + 2*(L==3)] max, [41 + 2*(L==3)] sum
#define TRB_OSUM_WALK_BEGIN() \
  const bool walk_on_ = ::trb::g_phase_on != 0;             \
  const long long walk_t0_ = walk_on_ ? clock64() : 0;       \
  long long walk_t1_ = walk_t0_;                                 \
  unsigned long long nslow_ = 0, nbp_ = 0
// per-element timestamps of a typical walking thread (CTA 1, thread 100; L == 3 only): g_phase[192 + k]
#define TRB_OSUM_ELEM_TRACE(k, dep) \
  if (walk_on_ && L == 3 && rank == 1 && threadIdx.x == 100 && (k) < 32) \
    ::trb::g_phase[192 + (k)] = clock64() - walk_t0_ + ((dep) != (dep) ? 1 : 0)
// time to the first element's data (cursor start-up); `dep` forces the wait
#define TRB_OSUM_WALK_FIRST(cond, dep) \
  if ((cond) && walk_on_) walk_t1_ = clock64() + ((dep) != (dep) ? 1 : 0)
#define TRB_OSUM_COUNT(v) ++(v)
#define TRB_OSUM_WALK_END()                                                                        \
  do {                                                                                             \
    if (walk_on_ && G == 8) { /* by the warp's slow-path events: walk cycles summed, counted */     \
      const unsigned wm_ = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(clock64() - walk_t0_)); \
      const bool work_ = __any_sync(0xffffffffu, j0 < j1);                                         \
      const unsigned ns_ = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(nslow_));          \
      if ((threadIdx.x & 31) == 0 && work_) {                                                      \
        const int c_ = ns_ == 0 ? 0 : ns_ <= 2 ? 1 : ns_ <= 5 ? 2 : ns_ <= 10 ? 3 : ns_ <= 20 ? 4 : ns_ <= 40 ? 5 : 6; \
        atomicAdd(&::trb::g_warpwalk[(L == 3) * 16 + c_ * 2], wm_);                                 \
        atomicAdd(&::trb::g_warpwalk[(L == 3) * 16 + c_ * 2 + 1], 1ull);                            \
      }                                                                                            \
    }                                                                                              \
    if (walk_on_ && rank == 0 && j0 < j1) {                                                        \
      const unsigned long long d_ = clock64() - walk_t0_;                                          \
      unsigned long long* ph_ = ::trb::g_phase + 64 * ::trb::s_ph_bucket;                         \
      atomicMax(&ph_[40 + 2 * (L == 3)], d_);                                                      \
      atomicAdd(&ph_[41 + 2 * (L == 3)], d_);                                                      \
      atomicMax(&ph_[44 + 4 * (L == 3)], nslow_);                                                  \
      atomicAdd(&ph_[45 + 4 * (L == 3)], nslow_);                                                  \
      atomicMax(&ph_[46 + 4 * (L == 3)], nbp_);                                                    \
      atomicAdd(&ph_[47 + 4 * (L == 3)], nbp_);                                                    \
      atomicAdd(&ph_[52 + (L == 3)], 1ull);                                                        \
      atomicAdd(&ph_[54 + (L == 3)], static_cast<unsigned long long>(walk_t1_ - walk_t0_));       \
    }                                                                                              \
  } while (0)
#define TRB_OSUM_MARK(stage)                                                                   \
  do {                                                                                         \
    if (::trb::g_progress && threadIdx.x == 0)                                                 \
      (reinterpret_cast<volatile int*>(::trb::g_progress))[4 * blockIdx.x + 3] = 100 + (stage); \
    TRB_PHASE((stage) >= 20 ? ((L == 1 ? 11 : 13) + (stage)) : ((L == 1 ? 7 : 18) + (stage)), rank, G); \
  } while (0)

#else
#define TRB_PHASE(k, rank_, G_) ((void)0)
#define TRB_PHASE_BEGIN(n_px, rank_) ((void)0)
#define TRB_OSUM_WALK_BEGIN()
#define TRB_OSUM_WALK_END() ((void)0)
#define TRB_OSUM_COUNT(v) ((void)0)
#define TRB_OSUM_WALK_FIRST(cond, dep) ((void)0)
#define TRB_OSUM_ELEM_TRACE(k, dep) ((void)0)
#define TRB_OSUM_MARK(stage) ((void)0)
#endif

#include "trb_track.cuh"
// v2 engine phase marks (diagnostics build): hist run slots 1..7, centroid 9..15
#define TRB_XS_MARK(k) TRB_PHASE(1 + (k) + (NF == 1 ? 0 : 8), rank, G)
#include "trb_xsum.cuh"

namespace trb {

// Device-side diagnostics: [0..4] ordered_sums stats (see trb_osum.cuh),
// [5] mean-shift iterations, [6] spawns, [7] Lloyd iterations, [8] farthest
// point passes, [9] tracks advanced, [11] window pixels of the mean-shift
// iterations (the tracker's algorithmic frame reads, one byte per pixel).
// [16..25] ordered_sums failure reasons (bit index of the `bad` mask).
__device__ unsigned long long g_trb_stats[32];
// Optional per-iteration timing log: {window pixels, cycles} pairs.
__device__ long long* g_itlog;
__device__ unsigned long long g_itlog_n;
#ifdef TRB_DIAG
#define TRB_PROGRESS(slot, a, b, c, d)                                                      \
  do {                                                                                      \
    if (g_progress && threadIdx.x == 0) {                                                   \
      volatile int* p_ = g_progress + 4 * (slot);                                           \
      p_[0] = (a), p_[1] = (b), p_[2] = (c), p_[3] = (d);                                   \
    }                                                                                       \
  } while (0)
#else
#define TRB_PROGRESS(slot, a, b, c, d) ((void)0)
#endif

namespace {

constexpr int NT = kOsumThreads;

// Exact u32 division by a runtime divisor (Granlund-Montgomery): used to
// turn a raster element index into (x, y) inside a window.
struct UDiv32 {
  uint32_t m;
  int sh1, sh2;
  __device__ static UDiv32 make(uint32_t d) {
    int l = 0;
    while ((1ull << l) < d) ++l;
    UDiv32 r;
    r.m = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    r.sh1 = l > 0 ? 1 : 0;
    r.sh2 = l > 0 ? l - 1 : 0;
    return r;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> sh1)) >> sh2;
  }
};

struct Win {
  int x0, y0, x1, y1;
  __device__ bool empty() const { return x0 >= x1 || y0 >= y1; }
};

// clip_window, tracking.hpp:61-66
__device__ __forceinline__ Win clip_window(int fw, int fh, double cx, double cy, int w, int h) {
  const int x0 = static_cast<int>(xlround(cx)) - w / 2;
  const int y0 = static_cast<int>(xlround(cy)) - h / 2;
  return Win{max(0, x0), max(0, y0), min(fw, x0 + w), min(fh, y0 + h)};
}

// ColorQuantizer::assign, quantize.hpp:20-29 (strict <, lowest index wins)
__device__ __forceinline__ int q_assign(const double* c, int k, double r, double g, double b) {
  int best = 0;
  double best_d = __longlong_as_double(0x7ff0000000000000LL);
  for (int i = 0; i < k; ++i) {
    const double dr = xsub(r, c[3 * i]), dg = xsub(g, c[3 * i + 1]), db = xsub(b, c[3 * i + 2]);
    const double d = xadd(xadd(xmul(dr, dr), xmul(dg, dg)), xmul(db, db));
    if (d < best_d) best_d = d, best = i;
  }
  return best;
}

// Per-cluster global scratch of the tracker kernels.
// Both arrays hold thread chunks INTERLEAVED (element gt*C + i at i*GT + gt,
// 4-pixel words for bins), so a warp's loads at step i are coalesced; the
// slack covers chunk rounding and the cursors' read-ahead.
constexpr int64_t kValsSlack = 32768;  // doubles
constexpr int64_t kBinsSlack = 262144;  // bytes
struct TrackScratch {
  double* vals;    // [2*maxN + slack] positive Epanechnikov weights, partitioned by bin, then raster
  uint8_t* bins;   // [maxN + slack] bin of every window pixel (raster order, as words)
  static __host__ __device__ size_t bytes(int G, int64_t maxN) {
    (void)G;
    return sizeof(double) * (2 * maxN + kValsSlack) + maxN + kBinsSlack + 256;
  }
};

// Shared-memory map for the tracker CTAs (dynamic part; the engine's
// OsumShared is static).
struct TrackSmem {
  OsumShared* os;
  Grp grp;       // the CTAs sharing this track (cluster, or this CTA alone)
  double* ux2;   // [W]
  double* uy2;   // [H]
  double* cen;   // [K*3]
  double* old;   // [K*3]
  double* q;     // [K]
  double* p;     // [K]
  double* wsq;   // [K]
  double* scal;  // [16] broadcast scalars
  long long* red;  // [2*NT] reduction scratch
  int* cnt;      // [K+1][NT] per-thread segment counts, then scatter cursors
  int* binoff;   // [K+2] segment offsets in the partitioned sequence
  int* bincta;   // [K+1] this CTA's per-segment totals
  int* gcnt;     // [kMaxCluster][K+1] gathered per-CTA segment totals
  int* iscal;    // [16]
  uint8_t* lut;  // [256]
  static size_t bytes(int K, int W, int H) {
    return sizeof(OsumShared) + 16 + sizeof(double) * (W + H + 9 * K + 16) + sizeof(long long) * 2 * NT +
           sizeof(int) * ((K + 1) * NT + 2 * K + 3 + 16 + kMaxCluster * (K + 1)) + 256 + 16 * 16;
  }
  __device__ void carve(void* base, OsumShared* /*unused*/, int K, int W, int H) {
    char* p_ = static_cast<char*>(base);
    auto take = [&](size_t n) {
      char* r = p_;
      p_ += (n + 15) & ~size_t(15);
      return r;
    };
    // the engine's workspace (> 48 KB, so it must be dynamic shared memory)
    OsumShared* osh = reinterpret_cast<OsumShared*>(take(sizeof(OsumShared)));
    os = osh;
    grp = Grp::cluster();
    ux2 = reinterpret_cast<double*>(take(sizeof(double) * W));
    uy2 = reinterpret_cast<double*>(take(sizeof(double) * H));
    cen = reinterpret_cast<double*>(take(sizeof(double) * 3 * K));
    old = reinterpret_cast<double*>(take(sizeof(double) * 3 * K));
    q = reinterpret_cast<double*>(take(sizeof(double) * K));
    p = reinterpret_cast<double*>(take(sizeof(double) * K));
    wsq = reinterpret_cast<double*>(take(sizeof(double) * K));
    scal = reinterpret_cast<double*>(take(sizeof(double) * 16));
    red = reinterpret_cast<long long*>(take(sizeof(long long) * 2 * NT));
    cnt = reinterpret_cast<int*>(take(sizeof(int) * (K + 1) * NT));
    binoff = reinterpret_cast<int*>(take(sizeof(int) * (K + 2)));
    bincta = reinterpret_cast<int*>(take(sizeof(int) * (K + 1)));
    gcnt = reinterpret_cast<int*>(take(sizeof(int) * kMaxCluster * (K + 1)));
    iscal = reinterpret_cast<int*>(take(sizeof(int) * 16));
    lut = reinterpret_cast<uint8_t*>(take(256));
    if (threadIdx.x == 0) osh->phase = 0;
  }
};

// Fill ux2/uy2 for window r around (cx, cy) with half-sizes w/2.0, h/2.0:
// ux = (x - cx) / hx; ux*ux  (tracking.hpp:84-91, same operations).
__device__ void fill_u2(TrackSmem& sm, const Win& r, double cx, double cy, int w, int h) {
  const double hx = static_cast<double>(w) / 2.0, hy = static_cast<double>(h) / 2.0;
  for (int i = threadIdx.x; i < r.x1 - r.x0; i += blockDim.x) {
    const double ux = xdiv(xsub(static_cast<double>(r.x0 + i), cx), hx);
    sm.ux2[i] = xmul(ux, ux);
  }
  for (int i = threadIdx.x; i < r.y1 - r.y0; i += blockDim.x) {
    const double uy = xdiv(xsub(static_cast<double>(r.y0 + i), cy), hy);
    sm.uy2[i] = xmul(uy, uy);
  }
}

__device__ __forceinline__ double epan_weight(const TrackSmem& sm, int xx, int yy, int epan) {
  if (!epan) return 1.0;
  const double t = xsub(1.0, xadd(sm.ux2[xx], sm.uy2[yy]));
  return (0.0 < t) ? t : 0.0;  // std::max(0.0, t)
}

// --- element sources for the engine (cursor walks from j0 upward) ---
// histogram bins: the positive weights stably partitioned by bin; one
// segment per non-empty bin.  vals holds thread chunks interleaved in
// 2-element blocks: block b of thread gt is the double2 at b*GT + gt.  The
// cursor streams blocks through a ring of kRing cp.async slots per thread.
struct BinsSrc {
  static constexpr int kUnroll = 1;
  static constexpr int kRing = 5;
  const double* vals;
  const int* off;  // [K+1]
  int K;
  uint4* stage;    // [kRing][blockDim.x] 16-byte slots
  static __device__ __forceinline__ int chunk(int N, int GT) { return (N + GT - 1) / GT; }
  static __device__ __forceinline__ int max_chunk(int N, int GT) { return chunk(N, GT); }
  static __device__ __forceinline__ void bounds(int N, int GT, int gt, int& j0, int& j1) {
    const int C = chunk(N, GT);
    j0 = min(N, gt * C), j1 = min(N, j0 + C);
  }
  struct Cursor {
    const BinsSrc* s;
    const double2* p;  // next block to request
    int j, b, sb, nb, GT, blk;  // current segment b = [sb, nb); blk = ring slot of the block being consumed
    int k;                      // element of the current 2-element block
    double c0, c1;
    __device__ __forceinline__ void next(int /*k*/, bool& start, int& seg, bool& has, double* v) {
      if (k == 0) {
        cp_async_wait<kRing - 2>();  // the block in slot blk has landed
        const uint4* slot = s->stage + blk * blockDim.x + threadIdx.x;
        const double2 d = *reinterpret_cast<const double2*>(slot);
        c0 = d.x, c1 = d.y;
        const int refill = blk == 0 ? kRing - 1 : blk - 1;  // (blk + kRing - 1) % kRing
        cp_async16(s->stage + refill * blockDim.x + threadIdx.x, p);
        cp_async_commit();
        p += GT;
        blk = blk == kRing - 1 ? 0 : blk + 1;
      }
      if (j >= nb) {
        do ++b;
        while (j >= s->off[b + 1]);
        sb = s->off[b], nb = s->off[b + 1];
      }
      TRB_CHECK(b < s->K, "BinsSrc segment", b, j);
      start = (j == sb), seg = b, has = true, v[0] = k == 0 ? c0 : c1;
      ++j;
      k ^= 1;
    }
  };
  __device__ Cursor begin(int j0, int gt, int /*C*/, int GT) const {
    int b = 0;
    while (b < K - 1 && off[b + 1] <= j0) ++b;
    Cursor c;
    c.s = this, c.j = j0, c.b = b, c.sb = off[b], c.nb = off[b + 1], c.GT = GT, c.blk = 0, c.k = 0;
    c.c0 = c.c1 = 0.0;
    cp_async_wait<0>();  // nothing of an earlier walk is still landing
    const double2* p = reinterpret_cast<const double2*>(vals) + gt;
#pragma unroll
    for (int r = 0; r < kRing - 1; ++r, p += GT) {
      cp_async16(stage + r * blockDim.x + threadIdx.x, p);
      cp_async_commit();
    }
    c.p = p;
    return c;
  }
};
static_assert(BinsSrc::kRing * 16 * NT <= kOsumStageBytes, "staging ring exceeds the gather list");

__device__ __forceinline__ unsigned u4_byte(const uint4& u, int k) {
  const unsigned lo = (k & 4) ? u.y : u.x, hi = (k & 4) ? u.w : u.z;
  return (((k & 8) ? hi : lo) >> (8 * (k & 3))) & 0xffu;
}

// mean-shift centroid: every window pixel, weight sqrt(q/p) of its bin;
// bins are 4-pixel words, chunk-interleaved (word i of thread gt at
// i*GT + gt, so a warp's loads are coalesced), streamed through a ring of
// kRing 4-byte cp.async slots per thread.  Chunks are multiples of 4 pixels
// (not 16), so small and medium windows spread over all the cluster's
// threads.  The loop stays rolled (kUnroll 1).
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
struct CentroidSrc {
  static constexpr int kUnroll = 1;
  static constexpr int kRing = 8;
  const uint8_t* bins;
  const double* wsq;  // < 0 when p[b] <= 0
  int x0, y0, ww;
  uint32_t* stage;    // [kRing][blockDim.x] 4-byte slots
  static __device__ __forceinline__ int chunk(int N, int GT) { return ((N + GT - 1) / GT + 3) & ~3; }
  // The first warp of the group (the young sum: its running sums still cross
  // a binade every few chunks, one divergent slow step per crossing) takes a
  // quarter-length chunk each; the other threads share the rest evenly.
  // Every chunk is a multiple of 4 pixels and they stay in thread order.
  static constexpr int kYoung = 32;
  static __device__ __forceinline__ int young_chunk(int N, int GT) { return max(4, (chunk(N, GT) >> 2) & ~3); }
  static __device__ __forceinline__ int half_chunk(int N, int GT) { return max(4, (chunk(N, GT) >> 1) & ~3); }
  static __device__ __forceinline__ int rest_chunk(int N, int GT) {
    const int Y = kYoung * (young_chunk(N, GT) + half_chunk(N, GT));
    return N <= Y ? 4 : ((N - Y + (GT - 2 * kYoung) - 1) / (GT - 2 * kYoung) + 3) & ~3;
  }
  static __device__ __forceinline__ int max_chunk(int N, int GT) {
    return max(max(young_chunk(N, GT), half_chunk(N, GT)), rest_chunk(N, GT));
  }
  // warp 0: quarter chunks, warp 1: half chunks, the rest evenly
  static __device__ __forceinline__ void bounds(int N, int GT, int gt, int& j0, int& j1) {
    const int Cy = young_chunk(N, GT), Ch = half_chunk(N, GT);
    if (gt < kYoung) {
      j0 = min(N, gt * Cy), j1 = min(N, j0 + Cy);
    } else if (gt < 2 * kYoung) {
      j0 = min(N, kYoung * Cy + (gt - kYoung) * Ch), j1 = min(N, j0 + Ch);
    } else {
      const int C1 = rest_chunk(N, GT);
      j0 = min(N, kYoung * (Cy + Ch) + (gt - 2 * kYoung) * C1), j1 = min(N, j0 + C1);
    }
  }
  struct Cursor {
    const CentroidSrc* s;
    const uint32_t* p;  // next word to request
    int i, xx, GT;      // i = element index inside the chunk
    double xd, yd;      // pixel coordinates as doubles (exact integers)
    uint32_t cur;
    __device__ __forceinline__ void next(int /*k*/, bool& start, int& seg, bool& has, double* v) {
      const int k = i & 3;
      if (k == 0) {
        const int w = i >> 2;
        cp_async_wait<kRing - 2>();  // word w has landed
        cur = s->stage[(w & (kRing - 1)) * blockDim.x + threadIdx.x];
        cp_async4(s->stage + ((w + kRing - 1) & (kRing - 1)) * blockDim.x + threadIdx.x, p);
        cp_async_commit();
        p += GT;
      }
      const double w = s->wsq[(cur >> (8 * k)) & 0xffu];
      start = false, seg = 0, has = w >= 0.0;
      v[0] = w;
      v[1] = xmul(w, xd);
      v[2] = xmul(w, yd);
      ++i;
      xd = xadd(xd, 1.0);
      if (++xx == s->ww) xx = 0, xd = static_cast<double>(s->x0), yd = xadd(yd, 1.0);
    }
  };
  // j0 = gt * C with C a multiple of 4
  __device__ Cursor begin(int j0, int gt, int /*C*/, int GT) const {
    const int xx = j0 % ww, yy = j0 / ww;
    const uint32_t* p = reinterpret_cast<const uint32_t*>(bins) + gt;
    Cursor c;
    c.s = this, c.i = 0, c.xx = xx, c.GT = GT;
    c.xd = static_cast<double>(x0 + xx), c.yd = static_cast<double>(y0 + yy);
    c.cur = 0;
    cp_async_wait<0>();
#pragma unroll
    for (int r = 0; r < kRing - 1; ++r, p += GT) {
      cp_async4(stage + r * blockDim.x + threadIdx.x, p);
      cp_async_commit();
    }
    c.p = p;
    return c;
  }
};
static_assert(CentroidSrc::kRing * 4 * NT <= kOsumStageBytes, "centroid staging ring exceeds the gather list");

__device__ __forceinline__ int bin_of(const uint8_t* frame, int fw, int ch, int x, int y, const TrackSmem& sm, int K,
                                      bool use_lut) {
  if (ch == 1) {
    const int v = frame[static_cast<int64_t>(y) * fw + x];
    if (use_lut) return sm.lut[v];
    const double d = v;
    return q_assign(sm.cen, K, d, d, d);
  }
  const uint8_t* p = frame + (static_cast<int64_t>(y) * fw + x) * 3;
  return q_assign(sm.cen, K, p[0], p[1], p[2]);
}

// Bin every window pixel (cached for the centroid pass) and stably
// Per-cluster scratch (partitioned weights, bin words) is rewritten every
// iteration at the same addresses: its stores carry an L2 evict_last policy
// so the lines stay in L2 between iterations instead of being written back
// to HBM while the overlapped motion/CCL kernels stream through L2
// (TRB_SCRATCH_HINT=0 at build time disables it for A/B).
#ifndef TRB_SCRATCH_HINT
#define TRB_SCRATCH_HINT 1
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol = 0;
#if TRB_SCRATCH_HINT
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
#if TRB_SCRATCH_HINT
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_keep(uint32_t* p, uint32_t v, uint64_t pol) {
#if TRB_SCRATCH_HINT
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
#else
  *p = v;
#endif
}

// partition the positive-weight pixels by bin across the cluster:
// sm.binoff[b] = start of bin b, scratch.vals = weights in (bin, raster)
// order.  Returns the number of positive-weight pixels.
__device__ int partition_window(const uint8_t* frame, int fw, int ch, const Win& r, int K, int epan, bool use_lut,
                                TrackSmem& sm, const TrackScratch& scr) {
  const Grp& cl = sm.grp;
  // Segments of the partitioned sequence: bins 0..K-1 (positive weights of
  // each bin, raster order), then segment K = all positive weights in raster
  // order (the histogram total, tracking.hpp:96).  One engine run then
  // yields hist[0..K-1] and total.
  const int NT_ = blockDim.x, t = threadIdx.x;
  const int rank = static_cast<int>(cl.block_rank()), G = static_cast<int>(cl.num_blocks());
  const int ww = r.x1 - r.x0, N = ww * (r.y1 - r.y0);
  // chunks of a multiple of 4 pixels (CentroidSrc's chunking): every thread
  // owns whole words of bins, stored chunk-interleaved
  const int GT = G * NT_, gt = rank * NT_ + t;
  int j0, j1;
  CentroidSrc::bounds(N, GT, gt, j0, j1);
  const int NB = K + 1;
  for (int b = 0; b < NB; ++b) sm.cnt[b * NT_ + t] = 0;
  {
    int xx = j0 % ww, yy = j0 / ww, npos = 0;
    unsigned wacc = 0;
    uint32_t* bw = reinterpret_cast<uint32_t*>(scr.bins) + gt;
    const uint64_t pol = l2_keep_policy();
    // a 4-pixel word of bins is complete: store it (word-interleaved)
    auto put_word = [&](int /*j*/, bool /*last*/) {
      st_keep(bw, wacc, pol);
      bw += GT;
      wacc = 0;
    };
    if (ch == 1 && use_lut) {
      // gray + LUT (the tracker's case): pixels are loaded one step ahead
      const uint8_t* row = frame + static_cast<int64_t>(r.y0 + yy) * fw + r.x0;
      int pix = j0 < j1 ? row[xx] : 0;
      for (int j = j0; j < j1; ++j) {
        const int b = sm.lut[pix];
        const bool pos = epan_weight(sm, xx, yy, epan) > 0.0;
        if (++xx == ww) xx = 0, ++yy, row += fw;
        if (j + 1 < j1) pix = row[xx];
        wacc |= static_cast<unsigned>(b) << (8 * (j & 3));
        if ((j & 3) == 3 || j + 1 == j1) put_word(j, j + 1 == j1);
        if (pos) sm.cnt[b * NT_ + t] += 1, ++npos;
      }
    } else {
      for (int j = j0; j < j1; ++j) {
        const int b = bin_of(frame, fw, ch, r.x0 + xx, r.y0 + yy, sm, K, use_lut);
        wacc |= static_cast<unsigned>(b) << (8 * (j & 3));
        if ((j & 3) == 3 || j + 1 == j1) put_word(j, j + 1 == j1);
        if (epan_weight(sm, xx, yy, epan) > 0.0) sm.cnt[b * NT_ + t] += 1, ++npos;
        if (++xx == ww) xx = 0, ++yy;
      }
    }
    sm.cnt[K * NT_ + t] = npos;
  }
  __syncthreads();
  TRB_PHASE(2, rank, G);
  // exclusive scan of the counts of every segment over the CTA's threads
  const int lane = t & 31, wid = t >> 5, nw = NT_ >> 5, per = NT_ >> 5;
  for (int b = wid; b < NB; b += nw) {
    int* row = sm.cnt + b * NT_;
    int acc = 0;
    for (int i = 0; i < per; ++i) acc += row[lane * per + i];
    int incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int run = incl - acc;
    if (lane == 31) sm.bincta[b] = incl;
    for (int i = 0; i < per; ++i) {
      const int v = row[lane * per + i];
      row[lane * per + i] = run;
      run += v;
    }
  }
  cl.sync();
  TRB_PHASE(3, rank, G);
  // segment offsets (cluster totals) and this CTA's carry per segment
  // (parallel DSMEM loads into gcnt[q][b], then one thread combines locally)
  for (int i = t; i < G * NB; i += NT_) sm.gcnt[i] = *cl.map_shared_rank(&sm.bincta[i % NB], i / NB);
  __syncthreads();
  for (int b = t; b < NB; b += NT_) {  // per segment: this CTA's carry and the cluster total
    int carry = 0, tot = 0;
    for (int q = 0; q < G; ++q) {
      const int c = sm.gcnt[q * NB + b];
      if (q < rank) carry += c;
      tot += c;
    }
    sm.red[b] = carry, sm.red[NT_ + b] = tot;
  }
  __syncthreads();
  if (t == 0) {
    int off = 0;
    for (int b = 0; b < NB; ++b) {
      sm.binoff[b] = off;
      sm.red[b] += off;  // where this CTA's segment-b run starts
      off += static_cast<int>(sm.red[NT_ + b]);
    }
    sm.binoff[NB] = off;
  }
  __syncthreads();
  TRB_PHASE(4, rank, G);
  for (int b = 0; b < NB; ++b) sm.cnt[b * NT_ + t] += static_cast<int>(sm.red[b]);
  {
    int xx = j0 % ww, yy = j0 / ww;
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(scr.bins) + gt;
    uint32_t word = bw[0], wnext = bw[GT];  // (slack past N)
    bw += 2 * GT;
    // vals in BinsSrc's interleaved layout for its chunk size: a sequence
    // position p lives in chunk g = p / Cv at offset i = p % Cv.  The
    // cursors carry (g, i) and advance incrementally (no division per
    // store): per bin packed g << 20 | i in shared memory (Cv < 2^20, g <
    // 2^11), the total segment's in registers.
    const int nseq = sm.binoff[NB], Cv = BinsSrc::chunk(nseq, GT);
    const UDiv32 divC = UDiv32::make(static_cast<uint32_t>(max(1, Cv)));
    for (int b = 0; b < NB; ++b) {
      const uint32_t pos = static_cast<uint32_t>(sm.cnt[b * NT_ + t]);
      const uint32_t g = divC.div(pos);
      sm.cnt[b * NT_ + t] = static_cast<int>((g << 20) | (pos - g * static_cast<uint32_t>(Cv)));
    }
    const uint32_t cK = static_cast<uint32_t>(sm.cnt[K * NT_ + t]);
    int gT = static_cast<int>(cK >> 20), iT = static_cast<int>(cK & 0xfffffu);
    auto at = [&](int g, int i) { return (static_cast<int64_t>(i >> 1) * GT + g) * 2 + (i & 1); };
    const uint64_t pol = l2_keep_policy();
    for (int j = j0; j < j1; ++j) {
      const double w = epan_weight(sm, xx, yy, epan);
      const int b = (word >> (8 * (j & 3))) & 0xffu;
      if ((j & 3) == 3) word = wnext, wnext = *bw, bw += GT;
      if (w > 0.0) {
        TRB_CHECK(b < K, "partition scatter", b, j);
        const uint32_t cb = static_cast<uint32_t>(sm.cnt[b * NT_ + t]);
        int g = static_cast<int>(cb >> 20), i = static_cast<int>(cb & 0xfffffu);
        st_keep(&scr.vals[at(g, i)], w, pol);
        if (++i == Cv) i = 0, ++g;
        sm.cnt[b * NT_ + t] = static_cast<int>((static_cast<uint32_t>(g) << 20) | static_cast<uint32_t>(i));
        st_keep(&scr.vals[at(gT, iT)], w, pol);
        if (++iT == Cv) iT = 0, ++gT;
      }
      if (++xx == ww) xx = 0, ++yy;
    }
  }
  cl.sync();  // every CTA reads the other CTAs' bincta before it is reused; vals complete
  TRB_PHASE(5, rank, G);
  return sm.binoff[NB];
}

// histogram_opt (tracking.hpp:79-102) with the quantizer in sm.cen (and
// sm.lut when use_lut).  Writes the normalised histogram to out[K];
// returns false for std::nullopt.  Cluster-uniform.
__device__ bool window_histogram(const uint8_t* frame, int fw, int fh, int ch, double cx, double cy, int w, int h,
                                 int K, int epan, bool use_lut, TrackSmem& sm, const TrackScratch& scr, double* out) {
  const Win r = clip_window(fw, fh, cx, cy, w, h);
  if (r.empty()) return false;
  TRB_PHASE_BEGIN((r.x1 - r.x0) * (r.y1 - r.y0), sm.grp.rank_);
  fill_u2(sm, r, cx, cy, w, h);
  __syncthreads();
  TRB_PHASE(1, sm.grp.rank_, sm.grp.size_);
  const int nseq = partition_window(frame, fw, ch, r, K, epan, use_lut, sm, scr);
  // per-bin sums (segments 0..K-1) and the total (segment K), each a
  // sequential sum in its reference order
  if (nseq == 0) return false;  // no positive weight: total == 0
  BinsSrc bs{scr.vals, sm.binoff, K + 1, osum_stage(*sm.os)};
  osum_run<1, true>(sm.grp, nseq, K + 1, bs, *sm.os, g_trb_stats);
  const double total = sm.os->result[K];
  if (!(total > 0.0)) return false;
  for (int b = threadIdx.x; b < K; b += blockDim.x) out[b] = xdiv(sm.os->result[b], total);
  __syncthreads();
  return true;
}

// meanshift_step (tracking.hpp:125-157) on the track whose model sits in
// sm.cen / sm.q (and sm.lut).  cx, cy, status updated in place (uniform).
__device__ void meanshift_device(const uint8_t* frame, int fw, int fh, int ch, double& cx, double& cy, int w, int h,
                                 int& status, int K, int max_iters, double eps, bool use_lut, TrackSmem& sm,
                                 const TrackScratch& scr) {
  if (threadIdx.x == 0) sm.iscal[10] = 0;
  if (status != TRB_TRACK_ACTIVE) return;
  if (threadIdx.x == 0) atomicAdd(&g_trb_stats[9], 1ull);
  for (int it = 0; it < max_iters; ++it) {
    if (threadIdx.x == 0) {
      sm.iscal[10] = it + 1;
      if (sm.grp.rank_ == 0) {
        const Win rw = clip_window(fw, fh, cx, cy, w, h);
        atomicAdd(&g_trb_stats[5], 1ull);
        atomicAdd(&g_trb_stats[11], static_cast<unsigned long long>(rw.empty() ? 0 : (rw.x1 - rw.x0) * (rw.y1 - rw.y0)));
      }
    }
    TRB_PROGRESS(blockIdx.x, 1, -1, it, 1);
    const long long t_it0 = clock64();
    const bool ok = window_histogram(frame, fw, fh, ch, cx, cy, w, h, K, 1, use_lut, sm, scr, sm.p);
    TRB_PROGRESS(blockIdx.x, 1, -1, it, 2);
    double* bct = reinterpret_cast<double*>(sm.red);  // per-bin bhattacharyya terms
    if (ok)
      for (int b = threadIdx.x; b < K; b += blockDim.x) {
        bct[b] = xsqrt(xmul(sm.p[b], sm.q[b]));
        sm.wsq[b] = sm.p[b] <= 0.0 ? -1.0 : xsqrt(xdiv(sm.q[b], sm.p[b]));
      }
    __syncthreads();
    if (threadIdx.x == 0) {
      int lost = !ok;
      if (ok) {
        double bc = 0.0;  // bhattacharyya, tracking.hpp:114-119 (in bin order)
        for (int i = 0; i < K; ++i) bc = xadd(bc, bct[i]);
        lost = !(bc > 0.0);
      }
      sm.iscal[0] = lost;
    }
    __syncthreads();
    TRB_PHASE(6, sm.grp.rank_, sm.grp.size_);
    if (sm.iscal[0]) {
      status = TRB_TRACK_LOST;
      return;
    }
    // the window is the same (same cx, cy); its bins are cached in scr.bins
    const Win r = clip_window(fw, fh, cx, cy, w, h);
    CentroidSrc cs{scr.bins, sm.wsq, r.x0, r.y0, r.x1 - r.x0, reinterpret_cast<uint32_t*>(osum_stage(*sm.os))};
    osum_run<3, false>(sm.grp, (r.x1 - r.x0) * (r.y1 - r.y0), 0, cs, *sm.os, g_trb_stats);
    const double sw = sm.os->result[0], sx = sm.os->result[1], sy = sm.os->result[2];
    __syncthreads();
    if (sw <= 0.0) {
      status = TRB_TRACK_LOST;
      return;
    }
    const double nx = xdiv(sx, sw), ny = xdiv(sy, sw);
    const double shift = glibc_hypot(xsub(nx, cx), xsub(ny, cy));
    cx = nx;
    cy = ny;
    TRB_PHASE(30, sm.grp.rank_, sm.grp.size_);
#ifdef TRB_DIAG
    if (g_itlog && threadIdx.x == 0 && sm.grp.block_rank() == 0) {
      const unsigned long long k = atomicAdd(&g_itlog_n, 1ull);
      if (k < (1u << 16))
        g_itlog[2 * k] = (static_cast<long long>(sm.iscal[9]) << 32) |
                         (static_cast<long long>(sm.grp.size_) << 24) | ((r.x1 - r.x0) * (r.y1 - r.y0)),
        g_itlog[2 * k + 1] = clock64() - t_it0;
    }
#endif
    if (shift < eps) break;
  }
}

// Staged bin words (written by HistSrc2 in the histogram's phase A): word i
// of cluster thread gt at words[i * GT + gt], streamed through a ring of
// kRing 4-byte cp.async slots per thread in shared memory (no register
// read-ahead: a register a pending load targets stalls every instruction
// that touches it).
struct WordStream {
  static constexpr int kRing = 8;
  const uint32_t* words;
  uint32_t* stage;  // [kRing][blockDim.x]
  int GT, gt;
  struct Cursor {
    const uint32_t* p;
    uint32_t* stage;
    int GT, w, k;
    uint32_t cur;
    __device__ __forceinline__ void start(const WordStream& ws) {
      stage = ws.stage, GT = ws.GT, w = 0, k = 0, cur = 0;
      p = ws.words + ws.gt;
      cp_async_wait<0>();  // nothing of an earlier walk is still landing
#pragma unroll
      for (int r = 0; r < kRing - 1; ++r, p += GT) {
        cp_async4(stage + r * blockDim.x + threadIdx.x, p);
        cp_async_commit();
      }
    }
    __device__ __forceinline__ int next_bin() {
      if (k == 0) {
        cp_async_wait<kRing - 2>();  // word w has landed
        cur = stage[(w & (kRing - 1)) * blockDim.x + threadIdx.x];
        cp_async4(stage + ((w + kRing - 1) & (kRing - 1)) * blockDim.x + threadIdx.x, p);
        cp_async_commit();
        p += GT, ++w;
      }
      const int b = (cur >> (8 * k)) & 0xff;
      k = (k + 1) & 3;
      return b;
    }
  };
};

// ------------------------------------------------------ mean-shift, v2
// The same meanshift_step / histogram_opt (tracking.hpp:79-157) on the
// chunk-classified engine (trb_xsum.cuh): the K+1 histogram sums run straight
// from raster order (no partition, no HBM scratch), the centroid's 3 sums
// likewise.  Gray frames with the per-track gray->bin table (the tracker's
// case) and K + 1 <= xs::kMaxL; everything else runs the v1 path above.
struct V2Smem {
  xs::Shared* xs;
  Grp grp;
  double* buf;    // [(K+1) * NT] scan / integer totals / gathered records
  int all_cap;    // gathered records that fit in buf
  float* ftot;    // [(K+1) * NT]
  double* wsum;   // [(K+1) * 32]
  double* ux2;    // [W]      (global, this CTA's slice: L1-resident; keeps shared memory for the engine)
  double* uy2;    // [H + 1]
  double* cen;    // [K*3]
  double* q;      // [K]
  double* p;      // [K]
  double* wsq;    // [K]
  double* bct;    // [K]
  int* iscal;     // [16]
  uint8_t* lut;   // [256]
  uint32_t* ring; // [WordStream::kRing][NT] cp.async staging of bin words
  uint32_t* words;  // global: this group's staged bin words
  static size_t bytes(int K, int W, int H) {
    const int L = K + 1;
    (void)W, (void)H;
    return sizeof(xs::Shared) + 16 + sizeof(double) * (static_cast<size_t>(L) * NT + L * 32 + 7 * K) +
           sizeof(float) * L * NT + sizeof(int) * 16 + 256 + sizeof(uint32_t) * WordStream::kRing * NT + 17 * 16;
  }
  // bin-word scratch per cluster: the window (<= frame) in 4-element words,
  // plus read-ahead slack of the rings; split mode: 1/G of it per CTA
  static __host__ __device__ size_t words_per_cluster(int64_t frame_px, int G) {
    return static_cast<size_t>(frame_px / 4 + 4 * G * NT) + static_cast<size_t>(WordStream::kRing + 2) * G * NT;
  }
  static __host__ __device__ size_t u2_doubles(int W, int H) { return static_cast<size_t>(W) + H + 1; }  // per CTA
  __device__ void carve(void* base, int K, int W, int H, double* u2_base) {
    char* p_ = static_cast<char*>(base);
    auto take = [&](size_t n) {
      char* r = p_;
      p_ += (n + 15) & ~size_t(15);
      return r;
    };
    const int L = K + 1;
    xs = reinterpret_cast<xs::Shared*>(take(sizeof(xs::Shared)));
    grp = Grp::cluster();
    buf = reinterpret_cast<double*>(take(sizeof(double) * L * NT));
    all_cap = static_cast<int>(sizeof(double) * L * NT / sizeof(xs::Rec2));
    ftot = reinterpret_cast<float*>(take(sizeof(float) * L * NT));
    wsum = reinterpret_cast<double*>(take(sizeof(double) * L * 32));
    ux2 = u2_base + static_cast<size_t>(blockIdx.x) * u2_doubles(W, H);
    uy2 = ux2 + W;
    cen = reinterpret_cast<double*>(take(sizeof(double) * 3 * K));
    q = reinterpret_cast<double*>(take(sizeof(double) * K));
    p = reinterpret_cast<double*>(take(sizeof(double) * K));
    wsq = reinterpret_cast<double*>(take(sizeof(double) * K));
    bct = reinterpret_cast<double*>(take(sizeof(double) * K));
    iscal = reinterpret_cast<int*>(take(sizeof(int) * 16));
    lut = reinterpret_cast<uint8_t*>(take(256));
    ring = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * WordStream::kRing * NT));
    words = nullptr;
  }
};

// histogram elements: raster order over the window, value = the
// Epanechnikov weight (tracking.hpp:86-91; uniform: 1), lane = the bin
struct HistSrc2 {
  const uint8_t* frame;
  int fw, x0, y0, ww;
  const double* ux2;
  const double* uy2;
  const uint8_t* lut;
  int epan;
  __device__ __forceinline__ double weight(int xx, double uy) const {
    if (!epan) return 1.0;
    const double t = xsub(1.0, xadd(ux2[xx], uy));
    return (0.0 < t) ? t : 0.0;  // std::max(0.0, t)
  }
  struct Cursor {
    const HistSrc2* s;
    const uint8_t* row;
    int xx, yy;
    double uy;
    __device__ __forceinline__ void next(bool& has, int& sel, double* v) {
      sel = s->lut[row[xx]];
      const double w = s->weight(xx, uy);
      has = w > 0.0;  // if (wgt <= 0.0) continue;
      v[0] = w;
      if (s->words) {  // stage the bin for the later walks (4-element words, chunk-interleaved)
        wacc |= static_cast<uint32_t>(sel) << (8 * k);
        if (++k == 4) *wp = wacc, wp += s->GT, wacc = 0, k = 0;
      }
      if (++xx == s->ww) xx = 0, ++yy, row += s->fw, uy = s->uy2[yy];
    }
    __device__ __forceinline__ void finish() {
      if (s->words && k) *wp = wacc;
    }
    uint32_t* wp;
    uint32_t wacc;
    int k;
  };
  uint32_t* words;  // when set: bin words of the thread's chunk are staged here
  int GT, gt;
  __device__ Cursor begin(int j0) const {
    Cursor c;
    c.s = this;
    c.yy = j0 / ww;
    c.xx = j0 - c.yy * ww;
    c.row = frame + static_cast<int64_t>(y0 + c.yy) * fw + x0;
    c.uy = uy2[c.yy];
    c.wp = words ? words + gt : nullptr;
    c.wacc = 0, c.k = 0;
    return c;
  }
  __device__ void get(int j, bool& has, int& sel, double* v) const {
    const int yy = j / ww, xx = j - yy * ww;
    sel = lut[frame[static_cast<int64_t>(y0 + yy) * fw + x0 + xx]];
    const double w = weight(xx, uy2[yy]);
    has = w > 0.0;
    v[0] = w;
  }
};

// centroid elements: every window pixel whose bin has p > 0, values
// (w, w*x, w*y) with w = sqrt(q/p) of its bin (tracking.hpp:137-145)
struct CentSrc2 {
  const uint8_t* frame;
  int fw, x0, y0, ww;
  const uint8_t* lut;
  const double* wsq;  // < 0 when p[b] <= 0
  struct Cursor {
    const CentSrc2* s;
    const uint8_t* row;
    int xx;
    double xd, yd;
    __device__ __forceinline__ void next(bool& has, int& sel, double* v) {
      const double w = s->wsq[s->lut[row[xx]]];
      sel = 0;
      has = w >= 0.0;
      v[0] = w;
      v[1] = xmul(w, xd);
      v[2] = xmul(w, yd);
      xd = xadd(xd, 1.0);
      if (++xx == s->ww) xx = 0, xd = static_cast<double>(s->x0), yd = xadd(yd, 1.0), row += s->fw;
    }
    __device__ __forceinline__ void finish() {}
  };
  __device__ Cursor begin(int j0) const {
    Cursor c;
    c.s = this;
    const int yy = j0 / ww;
    c.xx = j0 - yy * ww;
    c.row = frame + static_cast<int64_t>(y0 + yy) * fw + x0;
    c.xd = static_cast<double>(x0 + c.xx);
    c.yd = static_cast<double>(y0 + yy);
    return c;
  }
  __device__ void get(int j, bool& has, int& sel, double* v) const {
    const int yy = j / ww, xx = j - yy * ww;
    const double w = wsq[lut[frame[static_cast<int64_t>(y0 + yy) * fw + x0 + xx]]];
    sel = 0;
    has = w >= 0.0;
    v[0] = w;
    v[1] = xmul(w, static_cast<double>(x0 + xx));
    v[2] = xmul(w, static_cast<double>(y0 + yy));
  }
};

// histogram phase B from the staged bins (same elements as HistSrc2)
struct HistSrcW {
  WordStream ws;
  int ww;
  const double* ux2;
  const double* uy2;
  int epan;
  struct Cursor {
    const HistSrcW* s;
    WordStream::Cursor wc;
    int xx, yy;
    double uy;
    __device__ __forceinline__ void next(bool& has, int& sel, double* v) {
      sel = wc.next_bin();
      double w = 1.0;
      if (s->epan) {
        const double t = xsub(1.0, xadd(s->ux2[xx], uy));
        w = (0.0 < t) ? t : 0.0;
      }
      has = w > 0.0;
      v[0] = w;
      if (++xx == s->ww) xx = 0, ++yy, uy = s->uy2[yy];
    }
    __device__ __forceinline__ void finish() {}
  };
  __device__ Cursor begin(int j0) const {
    Cursor c;
    c.s = this;
    c.yy = j0 / ww;
    c.xx = j0 - c.yy * ww;
    c.uy = uy2[c.yy];
    c.wc.start(ws);
    return c;
  }
};

// centroid elements from the staged bins (same elements as CentSrc2, which
// serves the serial fallback's random access)
struct CentSrcW {
  WordStream ws;
  int x0, y0, ww;
  const double* wsq;
  CentSrc2 direct;
  __device__ void get(int j, bool& has, int& sel, double* v) const { direct.get(j, has, sel, v); }
  struct Cursor {
    const CentSrcW* s;
    WordStream::Cursor wc;
    int xx;
    double xd, yd;
    __device__ __forceinline__ void next(bool& has, int& sel, double* v) {
      const double w = s->wsq[wc.next_bin()];
      sel = 0;
      has = w >= 0.0;
      v[0] = w;
      v[1] = xmul(w, xd);
      v[2] = xmul(w, yd);
      xd = xadd(xd, 1.0);
      if (++xx == s->ww) xx = 0, xd = static_cast<double>(s->x0), yd = xadd(yd, 1.0);
    }
    __device__ __forceinline__ void finish() {}
  };
  __device__ Cursor begin(int j0) const {
    Cursor c;
    c.s = this;
    const int yy = j0 / ww;
    c.xx = j0 - yy * ww;
    c.xd = static_cast<double>(x0 + c.xx);
    c.yd = static_cast<double>(y0 + yy);
    c.wc.start(ws);
    return c;
  }
};

__device__ void fill_u2_v2(V2Smem& sm, const Win& r, double cx, double cy, int w, int h) {
  const double hx = static_cast<double>(w) / 2.0, hy = static_cast<double>(h) / 2.0;
  for (int i = threadIdx.x; i < r.x1 - r.x0; i += blockDim.x) {
    const double ux = xdiv(xsub(static_cast<double>(r.x0 + i), cx), hx);
    sm.ux2[i] = xmul(ux, ux);
  }
  for (int i = threadIdx.x; i <= r.y1 - r.y0; i += blockDim.x) {
    const double uy = xdiv(xsub(static_cast<double>(r.y0 + i), cy), hy);
    sm.uy2[i] = i < r.y1 - r.y0 ? xmul(uy, uy) : 0.0;
  }
}

// histogram_opt on the v2 engine; the normalised histogram to out[K].
__device__ bool window_histogram2(const uint8_t* frame, int fw, int fh, double cx, double cy, int w, int h, int K,
                                  int epan, V2Smem& sm, double* out) {
  const Win r = clip_window(fw, fh, cx, cy, w, h);
  if (r.empty()) return false;
  fill_u2_v2(sm, r, cx, cy, w, h);
  __syncthreads();
  const int ww = r.x1 - r.x0, N = ww * (r.y1 - r.y0);
  const int GT = sm.grp.size_ * static_cast<int>(blockDim.x), gt = sm.grp.rank_ * static_cast<int>(blockDim.x) + threadIdx.x;
  HistSrc2 hs{frame, fw, r.x0, r.y0, ww, sm.ux2, sm.uy2, sm.lut, epan, sm.words, GT, gt};
  HistSrcW hw{WordStream{sm.words, sm.ring, GT, gt}, ww, sm.ux2, sm.uy2, epan};
  xs::xsum_run<1, true>(sm.grp, N, K, hs, hw, *sm.xs, sm.buf, sm.ftot, sm.wsum, sm.all_cap, g_trb_stats);
  const double total = sm.xs->res[0];
  if (!(total > 0.0)) {
    __syncthreads();
    return false;
  }
  for (int b = threadIdx.x; b < K; b += blockDim.x) out[b] = xdiv(sm.xs->res[1 + b], total);
  __syncthreads();
  return true;
}

// meanshift_step (tracking.hpp:125-157) on the v2 engine; the track's model
// sits in sm.cen / sm.q / sm.lut.  cx, cy, status updated in place.
__device__ void meanshift_device2(const uint8_t* frame, int fw, int fh, double& cx, double& cy, int w, int h,
                                  int& status, int K, int max_iters, double eps, V2Smem& sm) {
  if (threadIdx.x == 0) sm.iscal[10] = 0;
  if (status != TRB_TRACK_ACTIVE) return;
  if (threadIdx.x == 0) atomicAdd(&g_trb_stats[9], 1ull);
  for (int it = 0; it < max_iters; ++it) {
    if (threadIdx.x == 0) {
      sm.iscal[10] = it + 1;
      if (sm.grp.rank_ == 0) {
        const Win rw = clip_window(fw, fh, cx, cy, w, h);
        atomicAdd(&g_trb_stats[5], 1ull);
        atomicAdd(&g_trb_stats[11], static_cast<unsigned long long>(rw.empty() ? 0 : (rw.x1 - rw.x0) * (rw.y1 - rw.y0)));
      }
    }
#ifdef TRB_DIAG
    {
      const Win rw = clip_window(fw, fh, cx, cy, w, h);
      TRB_PHASE_BEGIN(rw.empty() ? 0 : (rw.x1 - rw.x0) * (rw.y1 - rw.y0), sm.grp.rank_);
    }
#endif
    const bool ok = window_histogram2(frame, fw, fh, cx, cy, w, h, K, 1, sm, sm.p);
    if (ok)
      for (int b = threadIdx.x; b < K; b += blockDim.x) {
        sm.bct[b] = xsqrt(xmul(sm.p[b], sm.q[b]));
        sm.wsq[b] = sm.p[b] <= 0.0 ? -1.0 : xsqrt(xdiv(sm.q[b], sm.p[b]));
      }
    __syncthreads();
    if (threadIdx.x == 0) {
      int lost = !ok;
      if (ok) {
        double bc = 0.0;  // bhattacharyya, tracking.hpp:114-119 (in bin order)
        for (int i = 0; i < K; ++i) bc = xadd(bc, sm.bct[i]);
        lost = !(bc > 0.0);
      }
      sm.iscal[0] = lost;
    }
    __syncthreads();
    if (sm.iscal[0]) {
      status = TRB_TRACK_LOST;
      return;
    }
    const Win r = clip_window(fw, fh, cx, cy, w, h);
    const int ww = r.x1 - r.x0;
    CentSrc2 cs{frame, fw, r.x0, r.y0, ww, sm.lut, sm.wsq};
    const int GT = sm.grp.size_ * static_cast<int>(blockDim.x);
    const int gt = sm.grp.rank_ * static_cast<int>(blockDim.x) + threadIdx.x;
    CentSrcW cw{WordStream{sm.words, sm.ring, GT, gt}, r.x0, r.y0, ww, sm.wsq, cs};
    // the window is the histogram's (same cx, cy): its staged bins serve both centroid walks
    xs::xsum_run<3, false>(sm.grp, ww * (r.y1 - r.y0), 0, cw, cw, *sm.xs, sm.buf, sm.ftot, sm.wsum, sm.all_cap,
                           g_trb_stats);
    const double sw = sm.xs->res[0], sx = sm.xs->res[1], sy = sm.xs->res[2];
    __syncthreads();
    if (sw <= 0.0) {
      status = TRB_TRACK_LOST;
      return;
    }
    const double nx = xdiv(sx, sw), ny = xdiv(sy, sw);
    const double shift = glibc_hypot(xsub(nx, cx), xsub(ny, cy));
    cx = nx;
    cy = ny;
    TRB_PHASE(16, sm.grp.rank_, sm.grp.size_);
    if (shift < eps) break;
  }
}

// ------------------------------------------------------------- k-means
// Integer-valued RGB samples; the window of a frame or an explicit list.
struct FrameWindowSrc {
  const uint8_t* frame;
  int fw, ch, x0, y0, ww;
  UDiv32 dv;
  __device__ __forceinline__ void get(int i, int& r, int& g, int& b) const {
    const int yy = static_cast<int>(dv.div(static_cast<uint32_t>(i)));
    const int x = x0 + (i - yy * ww), y = y0 + yy;
    if (ch == 1) {
      r = g = b = frame[static_cast<int64_t>(y) * fw + x];
    } else {
      const uint8_t* p = frame + (static_cast<int64_t>(y) * fw + x) * 3;
      r = p[0], g = p[1], b = p[2];
    }
  }
};

struct ListSrc {
  const int* px;  // n*3 ints
  __device__ __forceinline__ void get(int i, int& r, int& g, int& b) const {
    r = px[3 * i], g = px[3 * i + 1], b = px[3 * i + 2];
  }
};

__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (t < o) red[t] += red[t + o];
    __syncthreads();
  }
  const long long r = red[0];
  __syncthreads();
  return r;
}

// exclusive scan of one int64 per thread (Hillis-Steele in shared memory)
__device__ __forceinline__ long long block_exscan_ll(long long v, long long* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int o = 1; o < blockDim.x; o <<= 1) {
    const long long y = t >= o ? red[t - o] : 0;
    __syncthreads();
    red[t] += y;
    __syncthreads();
  }
  const long long r = red[t] - v;
  __syncthreads();
  return r;
}

// quantize_colors (quantize.hpp:43-118).  Samples are integer-valued, so
// the k-means++ D^2 weights, their total and prefix sums are exact
// integers (no ordering issue); Lloyd sums are exact integers; the
// assignment distances use non-contracted fp64 like the reference.
// Result centres in sm.cen.  mt19937_64 draws happen on thread 0.
template <class Src>
__device__ void kmeans_device(const Src& src, int n, int K, int iters, uint64_t seed, TrackSmem& sm, Mt64* rng) {
  const int t = threadIdx.x;
  const int C = (n + NT - 1) / NT;
  const int j0 = min(n, t * C), j1 = min(n, j0 + C);
  double* cen = sm.cen;
  if (t == 0) {
    rng->seed(seed);
    const int64_t first = rng->uniform_int(0, static_cast<int64_t>(n) - 1);
    int r, g, b;
    src.get(static_cast<int>(first), r, g, b);
    cen[0] = r, cen[1] = g, cen[2] = b;
  }
  __syncthreads();
  for (int nc = 1; nc < K; ++nc) {
    // D^2 of every sample to its nearest seed (exact integers)
    long long local = 0;
    for (int i = j0; i < j1; ++i) {
      int r, g, b;
      src.get(i, r, g, b);
      int best = INT_MAX;
      for (int c = 0; c < nc; ++c) {
        const int dr = r - static_cast<int>(cen[3 * c]), dg = g - static_cast<int>(cen[3 * c + 1]),
                  db = b - static_cast<int>(cen[3 * c + 2]);
        best = min(best, dr * dr + dg * dg + db * db);
      }
      local += best;
    }
    const long long pre = block_exscan_ll(local, sm.red);
    const long long total = block_sum_ll(local, sm.red);
    if (t == 0) {
      sm.iscal[1] = n - 1;  // pick when no prefix exceeds r
      if (total > 0) sm.scal[0] = xmul(rng->uniform(), static_cast<double>(total));
      else sm.iscal[1] = 0;
    }
    __syncthreads();
    if (total > 0) {
      const double r = sm.scal[0];
      // the chunk holding the first prefix > r
      if (static_cast<double>(pre + local) > r && (t == 0 || !(static_cast<double>(pre) > r))) {
        long long acc = pre;
        for (int i = j0; i < j1; ++i) {
          int rr, g, b;
          src.get(i, rr, g, b);
          int best = INT_MAX;
          for (int c = 0; c < nc; ++c) {
            const int dr = rr - static_cast<int>(cen[3 * c]), dg = g - static_cast<int>(cen[3 * c + 1]),
                      db = b - static_cast<int>(cen[3 * c + 2]);
            best = min(best, dr * dr + dg * dg + db * db);
          }
          acc += best;
          if (static_cast<double>(acc) > r) {
            sm.iscal[1] = i;
            break;
          }
        }
      }
    }
    __syncthreads();
    if (t == 0) {
      int r, g, b;
      src.get(sm.iscal[1], r, g, b);
      cen[3 * nc] = r, cen[3 * nc + 1] = g, cen[3 * nc + 2] = b;
    }
    __syncthreads();
  }
  // Lloyd iterations
  long long* cnt = sm.red;           // [K]
  long long* sum = sm.red + K;       // [3K]  (needs 4K <= 2*NT)
  double* old = sm.old;
  if (t == 0) atomicAdd(&g_trb_stats[6], 1ull);
  for (int it = 0; it < iters; ++it) {
    if (t == 0) atomicAdd(&g_trb_stats[7], 1ull);
    for (int i = t; i < 3 * K; i += NT) old[i] = cen[i];
    for (int i = t; i < 4 * K; i += NT) sm.red[i] = 0;
    __syncthreads();
    for (int i = j0; i < j1; ++i) {
      int r, g, b;
      src.get(i, r, g, b);
      const int a = q_assign(old, K, r, g, b);
      atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[a]), 1ull);
      atomicAdd(reinterpret_cast<unsigned long long*>(&sum[3 * a]), static_cast<unsigned long long>(r));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sum[3 * a + 1]), static_cast<unsigned long long>(g));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sum[3 * a + 2]), static_cast<unsigned long long>(b));
    }
    __syncthreads();
    if (t == 0) sm.iscal[2] = 0;  // moved
    __syncthreads();
    for (int c = 0; c < K; ++c) {
      double nc3[3];
      if (cnt[c] == 0) {
        if (t == 0) atomicAdd(&g_trb_stats[8], 1ull);
        // farthest sample from its (old-assignment) centre, current centres,
        // lowest index on ties (quantize.hpp:99-107)
        double bd = -1.0;
        int bi = 0;
        for (int i = j0; i < j1; ++i) {
          int r, g, b;
          src.get(i, r, g, b);
          const int a = q_assign(old, K, r, g, b);
          const double dr = xsub(r, cen[3 * a]), dg = xsub(g, cen[3 * a + 1]), db = xsub(b, cen[3 * a + 2]);
          const double d = xadd(xadd(xmul(dr, dr), xmul(dg, dg)), xmul(db, db));
          if (d > bd) bd = d, bi = i;
        }
        // block argmax (max d, then min index); chunks are in index order
        __shared__ double w_d[NT];
        __shared__ int w_i[NT];
        w_d[t] = (j0 < j1) ? bd : -2.0;
        w_i[t] = bi;
        __syncthreads();
        for (int o = NT / 2; o > 0; o >>= 1) {
          if (t < o) {
            const double d2 = w_d[t + o];
            const int i2 = w_i[t + o];
            if (d2 > w_d[t] || (d2 == w_d[t] && i2 < w_i[t])) w_d[t] = d2, w_i[t] = i2;
          }
          __syncthreads();
        }
        int r, g, b;
        src.get(w_i[0], r, g, b);
        nc3[0] = r, nc3[1] = g, nc3[2] = b;
        __syncthreads();
      } else {
        const double m = static_cast<double>(cnt[c]);
        nc3[0] = xdiv(static_cast<double>(sum[3 * c]), m);
        nc3[1] = xdiv(static_cast<double>(sum[3 * c + 1]), m);
        nc3[2] = xdiv(static_cast<double>(sum[3 * c + 2]), m);
      }
      if (t == 0) {
        if (nc3[0] != cen[3 * c] || nc3[1] != cen[3 * c + 1] || nc3[2] != cen[3 * c + 2]) sm.iscal[2] = 1;
        cen[3 * c] = nc3[0], cen[3 * c + 1] = nc3[1], cen[3 * c + 2] = nc3[2];
      }
      __syncthreads();
    }
    if (!sm.iscal[2]) break;
    __syncthreads();
  }
  __syncthreads();
}

// quantize_colors for a GRAY window (r = g = b): every per-sample quantity
// of kmeans_device depends on the sample's gray value only, so after one
// pass that builds the window's 256-bin histogram and the first raster
// index of every value, the Lloyd sums, the assignments and the
// empty-cluster farthest point are O(256) per pass instead of O(n).  The
// k-means++ prefix search still walks the samples in raster order (with a
// 256-entry D^2 table).  Same integers, same fp64 operations, same RNG
// draws as kmeans_device: identical centres.  Needs 1024 ints of sm.cnt.
__device__ void kmeans_gray_device(const FrameWindowSrc& src, int n, int K, int iters, uint64_t seed, TrackSmem& sm,
                                   Mt64* rng) {
  const int t = threadIdx.x;
  const int C = (n + NT - 1) / NT;
  const int j0 = min(n, t * C), j1 = min(n, j0 + C);
  double* cen = sm.cen;
  int* hist = sm.cnt;          // [256] samples per gray value
  int* firsti = sm.cnt + 256;  // [256] first raster index of the value
  int* dtab = sm.cnt + 512;    // [256] D^2 to the nearest seed
  int* asg = sm.cnt + 768;     // [256] Lloyd assignment
  const int ww = src.ww;
  // walk samples j0..j1-1 of the window in raster order: f(i, gray)
  auto walk = [&](auto&& f) {
    if (j0 >= j1) return;
    int xx = j0 % ww;
    const uint8_t* row = src.frame + static_cast<int64_t>(src.y0 + j0 / ww) * src.fw + src.x0;
    for (int i = j0; i < j1; ++i) {
      if (!f(i, static_cast<int>(row[xx]))) return;
      if (++xx == ww) xx = 0, row += src.fw;
    }
  };
  for (int v = t; v < 256; v += NT) hist[v] = 0, firsti[v] = INT_MAX;
  __syncthreads();
  {
    int cur = -1, run = 0;
    walk([&](int i, int v) {
      if (v != cur) {
        if (run) atomicAdd(&hist[cur], run);
        cur = v, run = 0;
        atomicMin(&firsti[v], i);
      }
      ++run;
      return true;
    });
    if (run) atomicAdd(&hist[cur], run);
  }
  if (t == 0) {
    rng->seed(seed);
    const int64_t first = rng->uniform_int(0, static_cast<int64_t>(n) - 1);
    int r, g, b;
    src.get(static_cast<int>(first), r, g, b);
    cen[0] = r, cen[1] = g, cen[2] = b;
  }
  __syncthreads();
  for (int nc = 1; nc < K; ++nc) {
    for (int v = t; v < 256; v += NT) {
      int best = INT_MAX;
      for (int c = 0; c < nc; ++c) {
        const int dr = v - static_cast<int>(cen[3 * c]), dg = v - static_cast<int>(cen[3 * c + 1]),
                  db = v - static_cast<int>(cen[3 * c + 2]);
        best = min(best, dr * dr + dg * dg + db * db);
      }
      dtab[v] = best;
    }
    __syncthreads();
    long long local = 0;
    walk([&](int, int v) {
      local += dtab[v];
      return true;
    });
    const long long pre = block_exscan_ll(local, sm.red);
    const long long total = block_sum_ll(local, sm.red);
    if (t == 0) {
      sm.iscal[1] = n - 1;
      if (total > 0) sm.scal[0] = xmul(rng->uniform(), static_cast<double>(total));
      else sm.iscal[1] = 0;
    }
    __syncthreads();
    if (total > 0) {
      const double r = sm.scal[0];
      if (static_cast<double>(pre + local) > r && (t == 0 || !(static_cast<double>(pre) > r))) {
        long long acc = pre;
        walk([&](int i, int v) {
          acc += dtab[v];
          if (static_cast<double>(acc) > r) {
            sm.iscal[1] = i;
            return false;
          }
          return true;
        });
      }
    }
    __syncthreads();
    if (t == 0) {
      int r, g, b;
      src.get(sm.iscal[1], r, g, b);
      cen[3 * nc] = r, cen[3 * nc + 1] = g, cen[3 * nc + 2] = b;
    }
    __syncthreads();
  }
  long long* cnt = sm.red;      // [K]
  long long* sum = sm.red + K;  // [3K]
  double* old = sm.old;
  __shared__ double w_d[NT];
  __shared__ int w_i[NT];
  if (t == 0) atomicAdd(&g_trb_stats[6], 1ull);
  for (int it = 0; it < iters; ++it) {
    if (t == 0) atomicAdd(&g_trb_stats[7], 1ull);
    for (int i = t; i < 3 * K; i += NT) old[i] = cen[i];
    for (int i = t; i < 4 * K; i += NT) sm.red[i] = 0;
    __syncthreads();
    for (int v = t; v < 256; v += NT) {
      const int a = q_assign(old, K, v, v, v);
      asg[v] = a;
      if (hist[v]) {
        const unsigned long long hv = static_cast<unsigned long long>(hist[v]);
        atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[a]), hv);
        atomicAdd(reinterpret_cast<unsigned long long*>(&sum[3 * a]), hv * v);
        atomicAdd(reinterpret_cast<unsigned long long*>(&sum[3 * a + 1]), hv * v);
        atomicAdd(reinterpret_cast<unsigned long long*>(&sum[3 * a + 2]), hv * v);
      }
    }
    __syncthreads();
    if (t == 0) sm.iscal[2] = 0;
    __syncthreads();
    for (int c = 0; c < K; ++c) {
      double nc3[3];
      if (cnt[c] == 0) {
        if (t == 0) atomicAdd(&g_trb_stats[8], 1ull);
        // farthest sample (old assignment, current centres; first index on ties)
        double bd = -2.0;
        int bi = INT_MAX;
        for (int v = t; v < 256; v += NT)
          if (hist[v]) {
            const int a = asg[v];
            const double dr = xsub(v, cen[3 * a]), dg = xsub(v, cen[3 * a + 1]), db = xsub(v, cen[3 * a + 2]);
            const double dd = xadd(xadd(xmul(dr, dr), xmul(dg, dg)), xmul(db, db));
            if (dd > bd || (dd == bd && firsti[v] < bi)) bd = dd, bi = firsti[v];
          }
        w_d[t] = bd;
        w_i[t] = bi;
        __syncthreads();
        for (int o = NT / 2; o > 0; o >>= 1) {
          if (t < o) {
            const double d2 = w_d[t + o];
            const int i2 = w_i[t + o];
            if (d2 > w_d[t] || (d2 == w_d[t] && i2 < w_i[t])) w_d[t] = d2, w_i[t] = i2;
          }
          __syncthreads();
        }
        int r, g, b;
        src.get(w_i[0], r, g, b);
        nc3[0] = r, nc3[1] = g, nc3[2] = b;
        __syncthreads();
      } else {
        const double m = static_cast<double>(cnt[c]);
        nc3[0] = xdiv(static_cast<double>(sum[3 * c]), m);
        nc3[1] = xdiv(static_cast<double>(sum[3 * c + 1]), m);
        nc3[2] = xdiv(static_cast<double>(sum[3 * c + 2]), m);
      }
      if (t == 0) {
        if (nc3[0] != cen[3 * c] || nc3[1] != cen[3 * c + 1] || nc3[2] != cen[3 * c + 2]) sm.iscal[2] = 1;
        cen[3 * c] = nc3[0], cen[3 * c + 1] = nc3[1], cen[3 * c + 2] = nc3[2];
      }
      __syncthreads();
    }
    if (!sm.iscal[2]) break;
    __syncthreads();
  }
  __syncthreads();
}

__device__ void build_lut(TrackSmem& sm, int K) {
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    const double d = v;
    sm.lut[v] = static_cast<uint8_t>(q_assign(sm.cen, K, d, d, d));
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t slot_index(const TrackDev& d, int s, int slot) {
  return static_cast<int64_t>(s) * d.T + slot;
}

}  // namespace

// ------------------------------------------------------------ meanshift
// Persistent grid of thread-block clusters over (stream, list position)
// items; one CLUSTER per track, its window split across the cluster's CTAs.
__device__ __forceinline__ TrackScratch cluster_scratch(unsigned char* base, size_t stride, int64_t maxN) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = static_cast<int>(cl.num_blocks());
  const int cid = blockIdx.x / G;
  unsigned char* p = base + static_cast<size_t>(cid) * stride;
  TrackScratch s;
  s.vals = reinterpret_cast<double*>(p);
  s.bins = reinterpret_cast<uint8_t*>(s.vals + 2 * maxN + kValsSlack);
  return s;
}

// Iteration-count hint for the next frame's queue order: this frame's
// count, or (iter_decay > 0) a decaying maximum over the recent frames, so a
// track whose count oscillates is scheduled as its expensive frames need.
__device__ __forceinline__ int iter_hint(int now, int prev, int decay) {
  return decay > 0 ? max(now, prev - (prev * decay >> 3)) : now;
}

// Tracks cheap enough to run on one CTA (estimated from the last frame's
// iteration count: iters x (30 us + 14.1 us per kpx)) whose window fits the
// CTA's 1/G share of the cluster scratch.
__device__ __forceinline__ bool split_class(const TrackDev& d, int64_t g) {
  const int64_t area = static_cast<int64_t>(d.w[g]) * d.h[g];
  const double est = max(1, d.iters[g]) * (d.split_fix + d.split_perpx * static_cast<double>(area));
  return d.G > 1 && est < d.split_us && area <= ((d.maxN / d.G) & ~15LL);
}

// Work list of the active tracks, largest window first (longest processing
// time first keeps the persistent clusters balanced).  One CTA.
__global__ void __launch_bounds__(1024) track_schedule_kernel(TrackDev d) {
  // buckets: [split class][stream group][cost]: all cluster-class tracks come
  // before every split-class one (a cluster that turns to split mode never
  // turns back); inside a class, stream group g's tracks before group g+1's
  // (fewer frames are being read at a time: better L2 locality), costliest
  // first inside a group
  constexpr int kMaxGroups = 4;
  __shared__ int cnt[256 * kMaxGroups], off[256 * kMaxGroups];
  const int NG = max(1, min(kMaxGroups, d.stream_groups));
  const int NB = 256 * NG;
  const int t = threadIdx.x;
  for (int i = t; i < NB; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  auto bucket = [&](int item) -> int {
    const int s = item / d.T, i = item - s * d.T;
    if (i >= d.n_list[s]) return -1;
    const int64_t g = slot_index(d, s, d.list[static_cast<int64_t>(s) * d.T + i]);
    if (d.status[g] != TRB_TRACK_ACTIVE) return -1;
    // estimated cost: previous frame's iteration count x (fixed overhead
    // ~30k px + window area); 4 buckets per octave, small index = costly.
    const unsigned cost =
        static_cast<unsigned>(max(d.iter_floor, d.iters[g])) * static_cast<unsigned>(d.order_fix + max(1, d.w[g] * d.h[g]));
    const int lz = __clz(cost);
    const int sub = lz <= 29 ? static_cast<int>((cost >> (29 - lz)) & 3u) : 0;
    const int grp = static_cast<int>(static_cast<int64_t>(s) * NG / d.S);
    return (split_class(d, g) ? 128 * NG : 0) + 128 * grp + 4 * lz + (3 - sub);
  };
  // only the listed tracks: one warp per stream, lanes over its list
  const int lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  for (int s = wid; s < d.S; s += nw) {
    const int nl = d.n_list[s];
    for (int i = lane; i < nl; i += 32) {
      const int b = bucket(s * d.T + i);
      if (b >= 0) atomicAdd(&cnt[b], 1);
    }
  }
  __syncthreads();
  if (wid == 0) {  // exclusive scan of the bucket counts (NB / 32 per lane)
    const int per = NB / 32;
    int sum = 0;
    for (int k = 0; k < per; ++k) sum += cnt[lane * per + k];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int o = incl - sum;
    for (int k = 0; k < per; ++k) {
      const int v = cnt[lane * per + k];
      off[lane * per + k] = o, o += v;
    }
    if (lane == 31) {
      *d.work_n = incl;
      d.host_mirror[0] = incl;  // the host's active-track hint (cluster size)
      *d.work_head = 0;
      *d.spawn_n = 0;  // this frame's spawn list (track_gate_kernel appends)
      *d.spawn_head = 0;
    }
  }
  __syncthreads();
  for (int s = wid; s < d.S; s += nw) {
    const int nl = d.n_list[s];
    for (int i = lane; i < nl; i += 32) {
      const int b = bucket(s * d.T + i);
      if (b >= 0) d.work[atomicAdd(&off[b], 1)] = s * d.T + i;
    }
  }
}

__device__ void meanshift_item(const TrackDev& d, int q, TrackSmem& sm, const TrackScratch& scr, bool lead) {
  const int K = d.K;
  const bool gray = d.CH == 1;
  const int item = d.work[q];
  const int s = item / d.T, i = item - s * d.T;
  TRB_PROGRESS(blockIdx.x, 1, item, -1, 0);
  const int slot = d.list[static_cast<int64_t>(s) * d.T + i];
  const int64_t g = slot_index(d, s, slot);
  int status = d.status[g];
  if (status != TRB_TRACK_ACTIVE) return;
  if (threadIdx.x == 0) sm.iscal[9] = item;  // (diagnostics: iteration log)
  for (int k = threadIdx.x; k < 3 * K; k += NT) sm.cen[k] = d.centers[g * 3 * K + k];
  for (int k = threadIdx.x; k < K; k += NT) sm.q[k] = d.hist[g * K + k];
  if (gray)
    for (int k = threadIdx.x; k < 256; k += NT) sm.lut[k] = d.lut[g * 256 + k];
  __syncthreads();
  double cx = d.cx[g], cy = d.cy[g];
  meanshift_device(d.frames[s], d.W, d.H, d.CH, cx, cy, d.w[g], d.h[g], status, K, d.max_iters, d.eps, gray, sm, scr);
  sm.grp.sync();  // every CTA has read the track before the leader updates it
  if (lead) {
    d.cx[g] = cx;
    d.cy[g] = cy;
    d.status[g] = status;
    d.iters[g] = iter_hint(sm.iscal[10], d.iters[g], d.iter_decay);  // scheduling hint for the next frame
  }
}

// Persistent clusters over the costliest-first queue.  A cluster works on
// one track with all its CTAs while the tracks are expensive; once it draws
// a track whose estimated single-CTA time is below d.split_us (and whose
// window fits 1/G of the scratch) it switches to split mode, where every CTA
// claims and runs small tracks on its own (single-CTA barriers, no DSMEM).
#ifndef TRB_MS_MINBLOCKS
#define TRB_MS_MINBLOCKS 2
#endif
__global__ void __launch_bounds__(NT, TRB_MS_MINBLOCKS) track_meanshift_kernel(TrackDev d) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results first
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  TrackSmem sm;
  sm.carve(smem_raw, nullptr, d.K, d.W, d.H);
  const TrackScratch scr = cluster_scratch(d.scratch, d.scratch_stride, d.maxN);
  const int G = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
  const int n_work = *d.work_n;
  // One work loop (one inlined copy of the mean-shift code): cluster mode
  // until the first split-class track, then split mode — this CTA alone,
  // with its 1/G share of the cluster scratch.
  bool split = false;
  TrackScratch cur_scr = scr;
  for (;;) {
    if (!split) {
      if (rank == 0 && threadIdx.x == 0) {
        const int q = atomicAdd(d.work_head, 1);
        sm.iscal[8] = q < n_work ? q : -1;
      }
      cl.sync();
      sm.iscal[11] = *cl.map_shared_rank(&sm.iscal[8], 0);
      cl.sync();  // the leader may overwrite iscal[8] only after everyone read it
    } else {
      if (threadIdx.x == 0) {
        const int q = atomicAdd(d.work_head, 1);
        sm.iscal[11] = q < n_work ? q : -1;
      }
      __syncthreads();
    }
    const int q = sm.iscal[11];
    __syncthreads();
    if (q < 0) break;
#ifdef TRB_DIAG
    if (g_phase_on && threadIdx.x == 0) {  // per-CTA busy time and finish time (globaltimer ns)
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      s_item_t0 = t0;
    }
#endif
    bool to_split = false;
    if (!split) {
      const int item = d.work[q];
      const int s = item / d.T, i = item - s * d.T;
      const int64_t g = slot_index(d, s, d.list[static_cast<int64_t>(s) * d.T + i]);
      to_split = split_class(d, g);  // read before the leader updates iters
    }
    meanshift_item(d, q, sm, cur_scr, (split || rank == 0) && threadIdx.x == 0);
#ifdef TRB_DIAG
    if (g_phase_on && threadIdx.x == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      atomicAdd(&g_cta_time[2 * blockIdx.x], t1 - s_item_t0);
      atomicMax(&g_cta_time[2 * blockIdx.x + 1], t1);
    }
#endif
    if (to_split) {  // every later item is split-class too
      split = true;
      sm.grp = Grp::single();
      cur_scr.vals = scr.vals + static_cast<int64_t>(rank) * (((2 * d.maxN + kValsSlack) / G) & ~31LL);
      cur_scr.bins = scr.bins + static_cast<int64_t>(rank) * (((d.maxN + kBinsSlack) / G) & ~15LL);
    }
  }
}

// v2 mean-shift kernel: the same persistent queue (costliest first, split
// mode for cheap tracks) over meanshift_device2; no HBM scratch.
__device__ void meanshift_item2(const TrackDev& d, int q, V2Smem& sm, bool lead) {
  const int K = d.K;
  const int item = d.work[q];
  const int s = item / d.T, i = item - s * d.T;
  const int slot = d.list[static_cast<int64_t>(s) * d.T + i];
  const int64_t g = slot_index(d, s, slot);
  int status = d.status[g];
  if (status != TRB_TRACK_ACTIVE) return;
  for (int k = threadIdx.x; k < 3 * K; k += NT) sm.cen[k] = d.centers[g * 3 * K + k];
  for (int k = threadIdx.x; k < K; k += NT) sm.q[k] = d.hist[g * K + k];
  for (int k = threadIdx.x; k < 256; k += NT) sm.lut[k] = d.lut[g * 256 + k];
  __syncthreads();
  double cx = d.cx[g], cy = d.cy[g];
  meanshift_device2(d.frames[s], d.W, d.H, cx, cy, d.w[g], d.h[g], status, K, d.max_iters, d.eps, sm);
  sm.grp.sync();  // every CTA has read the track before the leader updates it
  if (lead) {
    d.cx[g] = cx;
    d.cy[g] = cy;
    d.status[g] = status;
    d.iters[g] = iter_hint(sm.iscal[10], d.iters[g], d.iter_decay);
  }
}

__global__ void __launch_bounds__(NT, TRB_MS_MINBLOCKS) track_meanshift2_kernel(TrackDev d) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results first
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  V2Smem sm;
  sm.carve(smem_raw, d.K, d.W, d.H, d.u2);
  const int rank = static_cast<int>(cl.block_rank());
  const int G = static_cast<int>(cl.num_blocks());
  const size_t wpc = V2Smem::words_per_cluster(static_cast<int64_t>(d.W) * d.H, G);
  uint32_t* const cl_words = d.words2 + static_cast<size_t>(blockIdx.x / G) * wpc;
  sm.words = cl_words;
  const int n_work = *d.work_n;
  bool split = false;
  for (;;) {
    if (!split) {
      if (rank == 0 && threadIdx.x == 0) {
        const int q = atomicAdd(d.work_head, 1);
        sm.iscal[8] = q < n_work ? q : -1;
      }
      cl.sync();
      sm.iscal[11] = *cl.map_shared_rank(&sm.iscal[8], 0);
      cl.sync();
    } else {
      if (threadIdx.x == 0) {
        const int q = atomicAdd(d.work_head, 1);
        sm.iscal[11] = q < n_work ? q : -1;
      }
      __syncthreads();
    }
    const int q = sm.iscal[11];
    __syncthreads();
    if (q < 0) break;
    bool to_split = false;
    if (!split) {
      const int item = d.work[q];
      const int s = item / d.T, i = item - s * d.T;
      const int64_t g = slot_index(d, s, d.list[static_cast<int64_t>(s) * d.T + i]);
      to_split = split_class(d, g);
    }
    meanshift_item2(d, q, sm, (split || rank == 0) && threadIdx.x == 0);
    if (to_split) {  // this CTA alone from now on, with its 1/G of the cluster's bin words
      split = true;
      sm.grp = Grp::single();
      sm.words = cl_words + static_cast<size_t>(rank) * (wpc / G);
    }
  }
}

// ---------------------------------------------------------------- gate
// One CTA per stream: spawn gating (tracking.hpp:185-195), spawn_track's
// geometry and success conditions (:208-234), lost counting and retirement
// (:197-201) and the log (:203-204).
__global__ void __launch_bounds__(NT) track_gate_kernel(TrackDev d) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results first
  __shared__ int sh_n, sh_ncur, sh_next_id, sh_ok;
  __shared__ double sh_min[2][NT / 32];
  const int s = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  int32_t* list = d.list + static_cast<int64_t>(s) * d.T;
  const trb_blob* blobs = d.blobs + static_cast<int64_t>(s) * d.blob_stride;
  uint8_t* matched = d.matched + static_cast<int64_t>(s) * d.blob_stride;
  const int nb = d.nblobs[s];
  const int n = d.n_list[s];
  auto gate = [&](const trb_blob& b, int slot) {
    const int64_t g = slot_index(d, s, slot);
    const double dist = glibc_hypot(xsub(b.cx, d.cx[g]), xsub(b.cy, d.cy[g]));
    const double w = d.w[g], h = d.h[g];
    const double diag = xsqrt(xadd(xmul(w, w), xmul(h, h)));  // Track::window_diagonal, :49
    return dist <= xmul(1.5, diag);
  };
  // 1. blobs against the tracks that existed before this frame's spawns
  for (int i = t; i < nb; i += NT) {
    int m = 0;
    for (int k = 0; k < n && !m; ++k) m = gate(blobs[i], list[k]);
    matched[i] = static_cast<uint8_t>(m);
  }
  if (t == 0) sh_n = n, sh_ncur = n, sh_next_id = d.next_id[s];
  __syncthreads();
  // 2. unmatched blobs in label order: this frame's earlier spawns count too
  for (int i = 0; i < nb; ++i) {
    if (matched[i]) continue;  // uniform
    const trb_blob b = blobs[i];
    // any of this frame's earlier spawns gates the blob: one barrier that
    // also publishes the vote (no shared flag that a fast thread could reset
    // for the next blob while slower warps still read it)
    int hit = 0;
    for (int k = sh_n + t; k < sh_ncur && !hit; k += NT) hit = gate(b, list[k]);
    if (__syncthreads_or(hit)) continue;
    // spawn_track: the id is consumed even when the spawn fails (:210)
    const int id = sh_next_id;
    int tw = max(3, b.x_max - b.x_min + 1), th = max(3, b.y_max - b.y_min + 1);
    while (tw * th < d.K) {
      if (tw <= th) ++tw;
      else ++th;
    }
    const Win r = clip_window(d.W, d.H, b.cx, b.cy, tw, th);
    bool ok = !r.empty() && static_cast<int64_t>(r.x1 - r.x0) * (r.y1 - r.y0) >= d.K;
    if (ok) {
      // histogram_opt is nullopt iff no window pixel has a positive
      // Epanechnikov weight; fl(a+b) is monotone, so test the minima.
      const double hx = tw / 2.0, hy = th / 2.0;
      double mx = __longlong_as_double(0x7ff0000000000000LL), my = mx;
      for (int x = r.x0 + t; x < r.x1; x += NT) {
        const double u = xdiv(xsub(static_cast<double>(x), b.cx), hx);
        mx = fmin(mx, xmul(u, u));
      }
      for (int y = r.y0 + t; y < r.y1; y += NT) {
        const double u = xdiv(xsub(static_cast<double>(y), b.cy), hy);
        my = fmin(my, xmul(u, u));
      }
      for (int o = 16; o > 0; o >>= 1) {
        mx = fmin(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        my = fmin(my, __shfl_xor_sync(0xffffffffu, my, o));
      }
      if (lane == 0) sh_min[0][wid] = mx, sh_min[1][wid] = my;
      __syncthreads();
      if (t == 0) {
        double a = sh_min[0][0], c = sh_min[1][0];
        for (int k = 1; k < NT / 32; ++k) a = fmin(a, sh_min[0][k]), c = fmin(c, sh_min[1][k]);
        sh_ok = xsub(1.0, xadd(a, c)) > 0.0;
      }
      __syncthreads();
      ok = sh_ok;
    }
    if (t == 0) {
      sh_next_id = id + 1;
      if (ok) {
        int slot = -1;
        for (int k = 0; k < d.T; ++k)
          if (!d.used[slot_index(d, s, k)]) {
            slot = k;
            break;
          }
        if (slot < 0 || sh_ncur >= d.T) {
          // the reference would append a track here; this handle cannot:
          // the step fails (sticky error, raised by the host at the next call)
          d.err[s] |= 1;
          atomicOr(d.err_any, 1);
          d.host_mirror[1] = 1;
        } else {
          const int64_t g = slot_index(d, s, slot);
          d.used[g] = 1;
          d.pending[g] = 1;
          d.spawn_list[atomicAdd(d.spawn_n, 1)] = static_cast<int32_t>(g);
          d.id[g] = id;
          d.cx[g] = b.cx;
          d.cy[g] = b.cy;
          d.w[g] = tw;
          d.h[g] = th;
          d.status[g] = TRB_TRACK_ACTIVE;
          d.lost[g] = 0;
          list[sh_ncur] = slot;
          sh_ncur = sh_ncur + 1;
        }
      }
    }
    __syncthreads();
  }
  // 3. lost counting, retirement (order preserving), log
  if (t == 0) {
    const int ncur = sh_ncur;
    int j = 0;
    for (int k = 0; k < ncur; ++k) {
      const int slot = list[k];
      const int64_t g = slot_index(d, s, slot);
      if (d.status[g] == TRB_TRACK_LOST) d.lost[g] += 1;
      if (d.status[g] == TRB_TRACK_LOST && d.lost[g] >= 5) {
        d.used[g] = 0;
        continue;
      }
      list[j++] = slot;
    }
    d.n_list[s] = j;
    d.next_id[s] = sh_next_id;
    sh_ncur = j;
  }
  __syncthreads();
  const int nl = sh_ncur;
  const int64_t base = d.n_log[s];
  const int frame = d.frame_no[s];
  // the log is a ring of log_cap entries per stream: entries [tail, head)
  // are held until the host drains them (trb_streams_drain_log); a step
  // whose entries do not fit fails (sticky error) instead of overwriting
  const bool fits = base + nl - d.log_tail[s] <= d.log_cap;
  if (!fits && t == 0) {
    atomicOr(&d.err[s], 2);
    atomicOr(d.err_any, 2);
    d.host_mirror[2] = 1;
  }
  trb_track_log_entry* log = d.log + static_cast<int64_t>(s) * d.log_cap;
  if (t == 0) d.step_log_base[s] = base;
  for (int k = t; k < nl && fits; k += NT) {
    const int64_t pos = (base + k) % d.log_cap;
    const int64_t g = slot_index(d, s, list[k]);
    trb_track_log_entry e;
    e.frame = frame;
    e.track_id = d.id[g];
    e.x = d.cx[g];
    e.y = d.cy[g];
    e.w = d.w[g];
    e.h = d.h[g];
    e.status = d.status[g];
    e._pad = 0;
    log[pos] = e;
  }
  __syncthreads();
  if (t == 0) {
    d.n_log[s] = base + (fits ? nl : 0);  // a step that does not fit logs nothing (and fails)
    d.frame_no[s] = frame + 1;
  }
}

// ---------------------------------------------------------------- spawn
// One cluster per pending track: quantize_colors on the window pixels with
// seed mix_seed(cfg.seed, id) (tracking.hpp:221-229) on the leader CTA, the
// centres broadcast through DSMEM, then the cluster-parallel target
// histogram (:230-232) and the gray->bin table.
__global__ void __launch_bounds__(NT) track_spawn_kernel(TrackDev d) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results first
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Mt64 rng;

  cg::cluster_group cl = cg::this_cluster();
  TrackSmem sm;
  sm.carve(smem_raw, nullptr, d.K, d.W, d.H);
  const int K = d.K;
  const TrackScratch scr = cluster_scratch(d.scratch, d.scratch_stride, d.maxN);
  const int G = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  const bool gray = d.CH == 1;
  // clusters claim this frame's spawns from the gate kernel's list (no scan
  // of every slot: with few or no spawns the kernel is a few microseconds)
  for (;;) {
    if (rank == 0 && threadIdx.x == 0) {
      const int q = atomicAdd(d.spawn_head, 1);
      sm.iscal[8] = q < *d.spawn_n ? d.spawn_list[q] : -1;
    }
    cl.sync();
    const int claimed = *cl.map_shared_rank(&sm.iscal[8], 0);
    cl.sync();  // the leader may overwrite iscal[8] only after everyone read it
    if (claimed < 0) break;
    const int64_t g = claimed;
    const int s = static_cast<int>(g / d.T);
    TRB_PROGRESS(blockIdx.x, 2, claimed, -1, 0);
    const double cx = d.cx[g], cy = d.cy[g];
    const int w = d.w[g], h = d.h[g];
    if (rank == 0) {
      const Win r = clip_window(d.W, d.H, cx, cy, w, h);
      FrameWindowSrc src{d.frames[s], d.W, d.CH, r.x0, r.y0, r.x1 - r.x0, UDiv32::make(r.x1 - r.x0)};
      const int n = (r.x1 - r.x0) * (r.y1 - r.y0);
      const uint64_t seed = mix_seed(d.seed, static_cast<uint64_t>(d.id[g]));
      if (gray && (K + 1) * NT >= 1024)
        kmeans_gray_device(src, n, K, d.kmeans_iters, seed, sm, &rng);
      else
        kmeans_device(src, n, K, d.kmeans_iters, seed, sm, &rng);
      for (int rr = 1; rr < G; ++rr)
        for (int k = threadIdx.x; k < 3 * K; k += NT) *cl.map_shared_rank(&sm.cen[k], rr) = sm.cen[k];
    }
    cl.sync();
    if (gray) build_lut(sm, K);
    window_histogram(d.frames[s], d.W, d.H, d.CH, cx, cy, w, h, K, 1, gray, sm, scr, sm.q);
    if (rank == 0) {
      for (int k = threadIdx.x; k < 3 * K; k += NT) d.centers[g * 3 * K + k] = sm.cen[k];
      for (int k = threadIdx.x; k < K; k += NT) d.hist[g * K + k] = sm.q[k];
      if (gray)
        for (int k = threadIdx.x; k < 256; k += NT) d.lut[g * 256 + k] = sm.lut[k];
    }
    cl.sync();  // all CTAs have read `pending` and the slot before it is cleared
    if (rank == 0 && threadIdx.x == 0) d.pending[g] = 0;
  }
}

// ----------------------------------------------------- standalone ops
struct OneArgs {
  const uint8_t* frame;
  int W, H, CH;
  double cx, cy;
  int w, h, status, K, max_iters, epan, mode;  // mode 0 meanshift, 1 histogram
  double eps;
  const double* centers;  // device K*3
  const double* target;   // device K
  double* out;            // device: [cx, cy, status, ok] or hist[K] + ok
  unsigned char* scratch;
  size_t scratch_stride;
  int64_t maxN;
  double* u2;  // v2: per-CTA ux2/uy2 slices
  uint32_t* words;  // v2: staged bin words
};

// One cluster: meanshift_step or histogram_opt on a single explicit track,
// on the v2 engine (gray frames, K + 1 <= xs::kMaxL).
__global__ void __launch_bounds__(NT) track_one2_kernel(OneArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  V2Smem sm;
  sm.carve(smem_raw, a.K, a.W, a.H, a.u2);
  sm.words = a.words;
  for (int k = threadIdx.x; k < 3 * a.K; k += NT) sm.cen[k] = a.centers[k];
  if (a.target)
    for (int k = threadIdx.x; k < a.K; k += NT) sm.q[k] = a.target[k];
  __syncthreads();  // the gray -> bin table reads every centre
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    const double dv = v;
    sm.lut[v] = static_cast<uint8_t>(q_assign(sm.cen, a.K, dv, dv, dv));
  }
  __syncthreads();
  const bool lead = cl.block_rank() == 0;
  if (a.mode == 0) {
    double cx = a.cx, cy = a.cy;
    int status = a.status;
    meanshift_device2(a.frame, a.W, a.H, cx, cy, a.w, a.h, status, a.K, a.max_iters, a.eps, sm);
    if (lead && threadIdx.x == 0) a.out[0] = cx, a.out[1] = cy, a.out[2] = status;
  } else {
    const bool ok = window_histogram2(a.frame, a.W, a.H, a.cx, a.cy, a.w, a.h, a.K, a.epan, sm, sm.p);
    if (lead) {
      for (int k = threadIdx.x; k < a.K; k += NT) a.out[k] = sm.p[k];
      if (threadIdx.x == 0) a.out[a.K] = ok ? 1.0 : 0.0;
    }
  }
}

// One cluster: meanshift_step or histogram_opt on a single explicit track.
__global__ void __launch_bounds__(NT) track_one_kernel(OneArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();

  TrackSmem sm;
  sm.carve(smem_raw, nullptr, a.K, a.W, a.H);
  const TrackScratch scr = cluster_scratch(a.scratch, a.scratch_stride, a.maxN);
  for (int k = threadIdx.x; k < 3 * a.K; k += NT) sm.cen[k] = a.centers[k];
  if (a.target)
    for (int k = threadIdx.x; k < a.K; k += NT) sm.q[k] = a.target[k];
  __syncthreads();
  const bool gray = a.CH == 1;
  if (gray) build_lut(sm, a.K);
  const bool lead = cl.block_rank() == 0;
  if (a.mode == 0) {
    double cx = a.cx, cy = a.cy;
    int status = a.status;
    meanshift_device(a.frame, a.W, a.H, a.CH, cx, cy, a.w, a.h, status, a.K, a.max_iters, a.eps, gray, sm, scr);
    if (lead && threadIdx.x == 0) a.out[0] = cx, a.out[1] = cy, a.out[2] = status;
  } else {
    const bool ok = window_histogram(a.frame, a.W, a.H, a.CH, a.cx, a.cy, a.w, a.h, a.K, a.epan, gray, sm, scr, sm.p);
    if (lead) {
      for (int k = threadIdx.x; k < a.K; k += NT) a.out[k] = sm.p[k];
      if (threadIdx.x == 0) a.out[a.K] = ok ? 1.0 : 0.0;
    }
  }
}

__global__ void __launch_bounds__(NT) quantize_kernel(const int* px, int n, int K, int iters, uint64_t seed,
                                                      double* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Mt64 rng;

  TrackSmem sm;
  sm.carve(smem_raw, nullptr, K, 1, 1);
  kmeans_device(ListSrc{px}, n, K, iters, seed, sm, &rng);
  for (int k = threadIdx.x; k < 3 * K; k += NT) out[k] = sm.cen[k];
}

// quantize_colors (quantize.hpp:43-118) for arbitrary real-valued samples:
// the general case has no integer structure to parallelise exactly (the D^2
// total and the Lloyd sums are order-dependent fp64 sums), so one device
// thread runs the reference's sequential algorithm with non-contracted
// __d*_rn arithmetic and the device mt19937_64.  Used by the public free
// function only; the tracker's samples are pixels (integers: quantize_kernel).
__global__ void __launch_bounds__(1024) quantize_serial_kernel(const double* __restrict__ px, int64_t n, int k,
                                                              int iters, uint64_t seed, double* __restrict__ centers,
                                                              double* __restrict__ d2, int* __restrict__ assign,
                                                              double* __restrict__ sum, int64_t* __restrict__ count,
                                                              Mt64* rng) {
  // One CTA.  Everything order-independent runs on all threads (distances,
  // the running D^2 minimum, assignments, counts, the farthest point with the
  // lowest index on ties); the order-dependent fp64 sums — the D^2 total, the
  // pick's running prefix, each cluster's coordinate sums — stay sequential in
  // point order, one thread per chain (quantize.hpp:52-114's order exactly).
  __shared__ long long s_pick;
  __shared__ double s_far[32];
  __shared__ long long s_fari[32];
  __shared__ int s_moved;
  const int t = threadIdx.x, NTq = blockDim.x;
  auto sq_dist3 = [](const double* a, const double* b) {
    const double dr = xsub(a[0], b[0]), dg = xsub(a[1], b[1]), db = xsub(a[2], b[2]);
    return xadd(xadd(xmul(dr, dr), xmul(dg, dg)), xmul(db, db));
  };
  if (t == 0) {
    rng->seed(seed);
    const int64_t first = rng->uniform_int(0, n - 1);  // k-means++: uniform first centre
    for (int c = 0; c < 3; ++c) centers[c] = px[3 * first + c];
  }
  __syncthreads();
  for (int64_t i = t; i < n; i += NTq) d2[i] = __longlong_as_double(0x7ff0000000000000LL);
  __syncthreads();
  double* pre = d2 + n;  // running D^2 prefix of the current pass (the pick's acc values)
  constexpr int kChunk = 4096;
  __shared__ double s_chunk[kChunk];
  __shared__ double s_total;
  __shared__ unsigned long long s_first;
  for (int nc = 1; nc < k; ++nc) {  // D^2-weighted picks
    double total = 0.0;  // thread 0's chain
    for (int64_t base = 0; base < n; base += kChunk) {
      const int m = n - base < kChunk ? static_cast<int>(n - base) : kChunk;
      for (int u = t; u < m; u += NTq) {  // min over the centres so far (order-free: the newest one only)
        const int64_t i = base + u;
        const double d = sq_dist3(&px[3 * i], &centers[3 * (nc - 1)]);
        const double b = d < d2[i] ? d : d2[i];
        d2[i] = b;
        s_chunk[u] = b;
      }
      __syncthreads();
      if (t == 0)  // the sequential total; its partials are exactly the pick loop's acc
        for (int u = 0; u < m; ++u) s_chunk[u] = total = xadd(total, s_chunk[u]);
      __syncthreads();
      for (int u = t; u < m; u += NTq) pre[base + u] = s_chunk[u];
      __syncthreads();
    }
    if (t == 0) {
      s_total = total;
      s_first = static_cast<unsigned long long>(n - 1);
    }
    __syncthreads();
    int64_t pick = 0;
    if (s_total > 0.0) {
      if (t == 0) s_chunk[0] = xmul(rng->uniform(), s_total);
      __syncthreads();
      const double r = s_chunk[0];
      for (int64_t i = t; i < n; i += NTq)  // first i whose prefix exceeds r (else n - 1)
        if (pre[i] > r) {
          atomicMin(&s_first, static_cast<unsigned long long>(i));
          break;
        }
      __syncthreads();
      pick = static_cast<int64_t>(s_first);
    }
    if (t < 3) centers[3 * nc + t] = px[3 * pick + t];
    __syncthreads();
  }
  for (int it = 0; it < iters; ++it) {  // Lloyd
    for (int64_t i = t; i < n; i += NTq) assign[i] = q_assign(centers, k, px[3 * i], px[3 * i + 1], px[3 * i + 2]);
    for (int c = t; c < k; c += NTq) count[c] = 0;
    __syncthreads();
    for (int64_t i = t; i < n; i += NTq)
      atomicAdd(reinterpret_cast<unsigned long long*>(&count[assign[i]]), 1ull);
    for (int j = t; j < 3 * k; j += NTq) {  // one register chain per (cluster, coordinate), point order
      const int c = j / 3, q = j - 3 * c;
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i)  // assign[i] is a warp-wide broadcast load
        if (assign[i] == c) acc = xadd(acc, px[3 * i + q]);
      sum[j] = acc;
    }
    if (t == 0) s_moved = 0;
    __syncthreads();
    for (int c = 0; c < k; ++c) {  // centres update in order (an empty one sees the partial update)
      if (count[c] == 0) {  // farthest point (first index on ties) from its current centre
        __syncthreads();  // earlier centres' updates visible
        double fd = -1.0;
        long long fi = 0;
        for (int64_t i = t; i < n; i += NTq) {
          const double d = sq_dist3(&px[3 * i], &centers[3 * assign[i]]);
          if (d > fd) fd = d, fi = i;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_down_sync(0xffffffffu, fd, o);
          const long long oi = __shfl_down_sync(0xffffffffu, fi, o);
          if (od > fd || (od == fd && oi < fi)) fd = od, fi = oi;
        }
        if ((t & 31) == 0) s_far[t >> 5] = fd, s_fari[t >> 5] = fi;
        __syncthreads();
        if (t == 0) {
          double bd = s_far[0];
          long long bi = s_fari[0];
          for (int w = 1; w < NTq / 32; ++w)
            if (s_far[w] > bd || (s_far[w] == bd && s_fari[w] < bi)) bd = s_far[w], bi = s_fari[w];
          s_pick = bi;
        }
        __syncthreads();
        if (t == 0) {
          double nc3[3];
          for (int q = 0; q < 3; ++q) nc3[q] = px[3 * s_pick + q];
          if (nc3[0] != centers[3 * c] || nc3[1] != centers[3 * c + 1] || nc3[2] != centers[3 * c + 2]) s_moved = 1;
          for (int q = 0; q < 3; ++q) centers[3 * c + q] = nc3[q];
        }
        __syncthreads();
      } else if (t == 0) {
        const double m = static_cast<double>(count[c]);
        double nc3[3];
        for (int q = 0; q < 3; ++q) nc3[q] = xdiv(sum[3 * c + q], m);
        if (nc3[0] != centers[3 * c] || nc3[1] != centers[3 * c + 1] || nc3[2] != centers[3 * c + 2]) s_moved = 1;
        for (int q = 0; q < 3; ++q) centers[3 * c + q] = nc3[q];
      }
    }
    __syncthreads();
    if (!s_moved) break;
    __syncthreads();
  }
}

// ------------------------------------------------------------- host side
// Per-iteration timing log (diagnostics): enable with a device buffer of
// 2^16 pairs; read back with read_itlog().
void enable_itlog(bool on) {
  static long long* buf = nullptr;
  if (on && !buf) TRB_CUDA(cudaMalloc(&buf, sizeof(long long) * 2 * (1 << 16)));
  long long* p = on ? buf : nullptr;
  TRB_CUDA(cudaMemcpyToSymbol(g_itlog, &p, sizeof(p)));
  unsigned long long z = 0;
  TRB_CUDA(cudaMemcpyToSymbol(g_itlog_n, &z, sizeof(z)));
  const int ph = on ? 1 : 0;
  TRB_CUDA(cudaMemcpyToSymbol(g_phase_on, &ph, sizeof(ph)));
  unsigned long long zz[256] = {};
  if (on) TRB_CUDA(cudaMemcpyToSymbol(g_phase, zz, sizeof(zz)));
}

void read_cta_times(unsigned long long* out2048, bool reset) {
  TRB_CUDA(cudaMemcpyFromSymbol(out2048, g_cta_time, 2048 * sizeof(*out2048)));
  if (reset) {
    std::vector<unsigned long long> z(2048, 0);
    TRB_CUDA(cudaMemcpyToSymbol(g_cta_time, z.data(), 2048 * sizeof(unsigned long long)));
  }
}

void read_phases(unsigned long long* out128) {
  TRB_CUDA(cudaMemcpyFromSymbol(out128, g_phase, 256 * sizeof(*out128)));
}

void read_warpwalk(unsigned long long* out128, bool reset) {
  TRB_CUDA(cudaMemcpyFromSymbol(out128, g_warpwalk, 128 * sizeof(*out128)));
  if (reset) {
    unsigned long long z[128] = {};
    TRB_CUDA(cudaMemcpyToSymbol(g_warpwalk, z, sizeof(z)));
  }
}

int64_t read_itlog(long long* out, int64_t cap) {
  long long* p = nullptr;
  unsigned long long n = 0;
  TRB_CUDA(cudaMemcpyFromSymbol(&p, g_itlog, sizeof(p)));
  TRB_CUDA(cudaMemcpyFromSymbol(&n, g_itlog_n, sizeof(n)));
  n = std::min<unsigned long long>(n, 1u << 16);
  n = std::min<unsigned long long>(n, static_cast<unsigned long long>(cap));
  if (p && n) TRB_CUDA(cudaMemcpy(out, p, sizeof(long long) * 2 * n, cudaMemcpyDeviceToHost));
  return static_cast<int64_t>(n);
}

// Hang diagnostics: progress records of every CTA in host-mapped memory.
int* enable_progress(int n_ctas) {
  static int* host = nullptr;
  static int cap = 0;
  if (n_ctas > cap) {
    if (host) cudaFreeHost(host);
    TRB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host), sizeof(int) * 4 * n_ctas, cudaHostAllocMapped));
    cap = n_ctas;
  }
  for (int i = 0; i < 4 * cap; ++i) host[i] = -7;
  int* dev = nullptr;
  TRB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
  TRB_CUDA(cudaMemcpyToSymbol(g_progress, &dev, sizeof(dev)));
  return host;
}

void read_debug_stats(unsigned long long* out, bool reset) {
  TRB_CUDA(cudaMemcpyFromSymbol(out, g_trb_stats, sizeof(unsigned long long) * 32));
  if (reset) {
    unsigned long long z[32] = {};
    TRB_CUDA(cudaMemcpyToSymbol(g_trb_stats, z, sizeof(z)));
  }
}

static void set_smem(const void* fn, size_t bytes) {
  TRB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

static size_t check_smem(int K, int W, int H) {
  const size_t b = TrackSmem::bytes(K, W, H);
  if (b > 200 * 1024)
    throw Error(TRB_CONFIG_ERROR, "tracker k_clusters / frame size exceed the device shared-memory budget");
  if (4 * K > 2 * NT) throw Error(TRB_CONFIG_ERROR, "tracker k_clusters too large for the device k-means");
  // partition_window packs (chunk g, offset i) as g << 20 | i: a window
  // chunk (window px / threads of the group, >= 1 CTA) must stay below 2^20
  if (static_cast<int64_t>(W) * H >= (int64_t(1) << 20) * NT)
    throw Error(TRB_CONFIG_ERROR, "tracker: frame too large (" + std::to_string(W) + "x" + std::to_string(H) + ")");
  return b;
}
// ... and the chunk index g < G x NT must fit the 12 bits above bit 20
static_assert(kMaxCluster * NT <= 4096, "partition_window's packed (chunk, offset) cursors need G x NT <= 4096");

// Engine choice.  v2 (trb_xsum.cuh: chunk-classified, no partition) has the
// lower fixed cost per iteration and wins on small windows (frames up to
// 640x480: C1 +25 %, C2 +7 % frames/s); v1 (trb_osum.cuh: staged element
// streams) has the cheaper element walks and wins on 1080p / 4K windows
// (C3 -20 %, C4 -30 %, C5 -25 % with v2).  Both are bit-exact.  v2 needs
// gray frames and K + 1 <= xs::kMaxL.  TRB_ENGINE=1 / 2 forces one (A/B).
static bool engine_v2(int K, int CH, int64_t frame_px) {
  static const int sel = [] {
    const char* e = getenv("TRB_ENGINE");
    return e ? atoi(e) : 0;
  }();
  const bool ok = CH == 1 && K + 1 <= xs::kMaxL;
  if (sel == 1) return false;
  if (sel == 2) return ok;
  return ok && frame_px <= 640 * 480;
}

static size_t check_smem_v2(int K, int W, int H) {
  const size_t b = V2Smem::bytes(K, W, H);
  if (b > 220 * 1024) throw Error(TRB_CONFIG_ERROR, "tracker frame size exceeds the device shared-memory budget");
  return b;
}

// Cluster size of the tracker kernels (CTAs per track).  TRB_CLUSTER
// overrides; sizes above 8 use the non-portable cluster attribute.
static int cluster_size() {
  static int g = [] {
    const char* e = getenv("TRB_CLUSTER");
    int v = e ? atoi(e) : 8;
    return std::max(1, std::min(v, kMaxCluster));
  }();
  return g;
}

template <typename Kern>
static void prepare_cluster_kernel(Kern kern, size_t smem, int G) {
  set_smem(reinterpret_cast<const void*>(kern), smem);
  if (G > 8)
    TRB_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

// Number of G-CTA clusters that can be co-resident for `kern`.
template <typename Kern>
static int max_clusters(Kern kern, size_t smem, int G) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G * 64);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  TRB_CUDA(cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(kern), &cfg));
  return std::max(1, n);
}

template <typename... KArgs, typename... Args>
static void launch_cluster_ex(bool pdl, void (*kern)(KArgs...), int n_clusters, int G, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_clusters * G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  TRB_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

// pdl: programmatic dependent launch (the kernel must pdl_wait() first)
template <typename... KArgs, typename... Args>
static void launch_cluster(void (*kern)(KArgs...), int n_clusters, int G, size_t smem, cudaStream_t st,
                           Args... args) {
  launch_cluster_ex(false, kern, n_clusters, G, smem, st, args...);
}


TrackerState::TrackerState(const trb_tracker_config& cfg, int S, int track_cap, int64_t log_cap)
    : cfg_(cfg), S_(S), T_(track_cap), K_(cfg.k_clusters), log_cap_(log_cap) {
  validate_tracker(cfg);
  const int64_t n = static_cast<int64_t>(S) * T_;
  // int32 block: n_list,next_id,frame_no,err (4*S) + list, id,w,h,status,lost,used,pending (8*n)
  if (track_cap < 1 || track_cap > (1 << 20)) throw Error(TRB_INVALID_ARGUMENT, "track capacity must be in [1, 2^20]");
  if (log_cap < 1) throw Error(TRB_INVALID_ARGUMENT, "track-log capacity must be >= 1");
  i32_.alloc(sizeof(int32_t) * (4 * S + 9 * n + 1));
  f64_.alloc(sizeof(double) * n * (2 + 4 * K_));
  lut_.alloc(static_cast<size_t>(n) * 256);
  log_.alloc(sizeof(trb_track_log_entry) * log_cap_ * S, false);
  nlog_.alloc(sizeof(int64_t) * 3 * S);  // head, tail, last frame's base
  // the cluster grid and breakpoint scratch are sized at the first process()
  // call, once the frame geometry (shared-memory need) is known
  int32_t* p = i32_.as<int32_t>();
  d_.S = S, d_.T = T_, d_.K = K_;
  d_.max_iters = cfg.max_iters, d_.kmeans_iters = cfg.kmeans_iters, d_.eps = cfg.eps, d_.seed = cfg.seed;
  d_.n_list = p, d_.next_id = p + S, d_.frame_no = p + 2 * S, d_.err = p + 3 * S;
  p += 4 * S;
  d_.list = p, d_.id = p + n, d_.w = p + 2 * n, d_.h = p + 3 * n, d_.status = p + 4 * n, d_.lost = p + 5 * n;
  d_.used = p + 6 * n, d_.pending = p + 7 * n, d_.iters = p + 8 * n;
  d_.err_any = p + 9 * n;
  mirror_.alloc_mapped(4 * sizeof(int32_t));
  {
    volatile int32_t* m = static_cast<volatile int32_t*>(mirror_.p);
    m[0] = -1, m[1] = 0, m[2] = 0;
  }
  d_.host_mirror = static_cast<volatile int32_t*>(mirror_.device_ptr());
  double* f = f64_.as<double>();
  d_.cx = f, d_.cy = f + n, d_.centers = f + 2 * n, d_.hist = f + 2 * n + 3 * K_ * n;
  d_.lut = lut_.as<uint8_t>();
  d_.log = log_.as<trb_track_log_entry>();
  d_.log_cap = log_cap_;
  d_.n_log = nlog_.as<int64_t>();
  d_.log_tail = d_.n_log + S;
  d_.step_log_base = d_.n_log + 2 * S;
  work_.alloc(sizeof(int32_t) * (2 * n + 4));
  d_.work = work_.as<int32_t>();
  d_.work_n = d_.work + n;
  d_.work_head = d_.work + n + 1;
  d_.spawn_list = d_.work + n + 2;
  d_.spawn_n = d_.spawn_list + n;
  d_.spawn_head = d_.spawn_n + 1;
  // next_id starts at 1 (tracking.hpp:239)
  std::vector<int32_t> ones(S, 1);
  TRB_CUDA(cudaMemcpy(d_.next_id, ones.data(), sizeof(int32_t) * S, cudaMemcpyHostToDevice));
}

TrackerState::~TrackerState() = default;

void TrackerState::process(const uint8_t* const* frames_dev, int w, int h, int ch, const trb_blob* blobs,
                           int64_t blob_stride, const int32_t* nblobs, cudaStream_t st, int* launches, cudaEvent_t after_meanshift,
                           cudaEvent_t blobs_ready) {
  if (matched_cap_ < blob_stride) {
    matched_.alloc(static_cast<size_t>(blob_stride) * S_);
    matched_cap_ = blob_stride;
  }
  d_.W = w, d_.H = h, d_.CH = ch;
  d_.frames = frames_dev;
  d_.blobs = blobs;
  d_.blob_stride = blob_stride;
  d_.nblobs = nblobs;
  d_.matched = matched_.as<uint8_t>();
  const size_t smem = check_smem(K_, w, h);
  const int G = cluster_size();
  if (smem != smem_set_) {
    prepare_cluster_kernel(track_meanshift_kernel, smem, G);
    prepare_cluster_kernel(track_spawn_kernel, smem, G);
    const int64_t items = static_cast<int64_t>(S_) * T_;
    grid_ = static_cast<int>(std::min<int64_t>(items, max_clusters(track_meanshift_kernel, smem, G)));
    if (const char* eg = getenv("TRB_TRACK_CLUSTERS")) grid_ = std::max(1, std::min(grid_, atoi(eg)));  // (A/B)
    d_.maxN = static_cast<int64_t>(w) * h;
    // cheap tracks run on single CTAs (split mode); a CTA then owns 1/G of
    // its cluster's scratch
    const char* es = getenv("TRB_SPLIT_US");
    d_.split_us = es ? atof(es) : 200.0;  // A/B after the graded chunks: 150-200 ahead of 100, 300, 400
    auto envf = [](const char* k, double dflt) {
      const char* e = getenv(k);
      return e ? atof(e) : dflt;
    };
    d_.split_fix = envf("TRB_SPLIT_FIX", 30.0);
    d_.split_perpx = envf("TRB_SPLIT_PERKPX", 14.1) * 1e-3;
    d_.order_fix = static_cast<int>(envf("TRB_ORDER_FIX", 5000.0));  // A/B (4 x 4 runs): 5k px ahead of 10k, 20k, 30k
    const char* eg2 = getenv("TRB_STREAM_GROUPS");
    d_.stream_groups = eg2 ? atoi(eg2) : 1;
    const char* ef = getenv("TRB_ITER_FLOOR");
    d_.iter_floor = ef ? std::max(1, atoi(ef)) : 6;  // iteration history is noisy: order mostly by area
    d_.iter_decay = static_cast<int>(envf("TRB_ITER_DECAY", 2.0));  // hint = max(now, prev - prev*decay/8); A/B: 2 ahead of 0, 1, 4 (C5 +1.2 %)
    d_.G = G;
    if (getenv("TRB_VERBOSE"))
      fprintf(stderr, "[trb] tracker: %d clusters of %d CTAs, split below %.0f us, %zu B dynamic smem per CTA\n",
              grid_, G, d_.split_us, smem);
    d_.scratch_stride = (TrackScratch::bytes(G, d_.maxN) + 255) & ~size_t(255);
    bp_.alloc(d_.scratch_stride * static_cast<size_t>(grid_), false);
    d_.scratch = bp_.as<unsigned char>();
    smem_set_ = smem;
  }
  const bool v2 = engine_v2(K_, ch, static_cast<int64_t>(w) * h);
  if (v2 && smem2_ == 0) {
    smem2_ = check_smem_v2(K_, w, h);
    prepare_cluster_kernel(track_meanshift2_kernel, smem2_, G);
    const int64_t items = static_cast<int64_t>(S_) * T_;
    grid2_ = static_cast<int>(std::min<int64_t>(items, max_clusters(track_meanshift2_kernel, smem2_, G)));
    if (const char* eg = getenv("TRB_TRACK_CLUSTERS")) grid2_ = std::max(1, std::min(grid2_, atoi(eg)));
    u2_.alloc(sizeof(double) * V2Smem::u2_doubles(w, h) * static_cast<size_t>(grid2_) * G, false);
    d_.u2 = u2_.as<double>();
    words2_.alloc(sizeof(uint32_t) * V2Smem::words_per_cluster(static_cast<int64_t>(w) * h, G) * grid2_, false);
    d_.words2 = words2_.as<uint32_t>();
    if (getenv("TRB_VERBOSE"))
      fprintf(stderr, "[trb] tracker v2: %d clusters of %d CTAs, %zu B dynamic smem per CTA\n", grid2_, G, smem2_);
  }
  // Mean-shift cluster size (v1 engine, frames above 640x480, TRB_CLUSTER
  // unset): when the active tracks are few (the previous frame's queue length,
  // stored into mapped host memory by the schedule kernel; a frame or two stale) a track gets a 16-CTA
  // (or 12-CTA) cluster, which shortens every iteration's walks — the
  // sequential iterations of the biggest windows are the step's critical path
  // (C3 +25 %, C4 +57 %, 8 C5 streams +21 %, 16 streams +13 %); with many
  // tracks, more 8-CTA clusters keep the GPU full (64 C5 streams at 16: -26 %).
  int Gm = G;
  int gridm = grid_;
  if (!v2 && !getenv("TRB_CLUSTER") && static_cast<int64_t>(w) * h > 640 * 480) {
    if (!grid_big_[0]) {
      for (int k = 0; k < 2; ++k) {
        const int g = k == 0 ? 16 : 12;
        prepare_cluster_kernel(track_meanshift_kernel, smem, g);
        grid_big_[k] = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(S_) * T_,
                                                          std::min(grid_, max_clusters(track_meanshift_kernel, smem, g))));
      }
    }
    // measured crossovers (C5 streams, ~5 tracks each, and C4): 16 wins up to
    // ~40 active tracks (S = 4, 8; C4), 12 around 80 (S = 16), 8 from ~160 (S = 32, 64)
    const int a = static_cast<const volatile int32_t*>(mirror_.p)[0];  // written by a recent schedule kernel
    if (a >= 0 && a <= 48) Gm = 16, gridm = grid_big_[0];
    else if (a >= 0 && a <= 100) Gm = 12, gridm = grid_big_[1];
  }
  // the schedule orders the queue with the same G as the mean-shift launch
  // (its split-mode class depends on G: a CTA alone gets 1/G of the scratch)
  TrackDev dm = d_;
  dm.G = Gm;
  track_schedule_kernel<<<1, 1024, 0, st>>>(dm);
  TRB_LAUNCH_CHECK("track_schedule_kernel");
  const bool pdl = !after_meanshift;  // (profiling records an event between the kernels)
  if (v2)
    launch_cluster_ex(pdl, track_meanshift2_kernel, grid2_, G, smem2_, st, d_);
  else
    launch_cluster_ex(pdl, track_meanshift_kernel, gridm, Gm, smem, st, dm);
  if (after_meanshift) TRB_CUDA(cudaEventRecord(after_meanshift, st));
  if (blobs_ready) TRB_CUDA(cudaStreamWaitEvent(st, blobs_ready, 0));
  if (pdl && !blobs_ready) launch_pdl(track_gate_kernel, dim3(S_), dim3(NT), 0, st, d_);
  else track_gate_kernel<<<S_, NT, 0, st>>>(d_);
  TRB_LAUNCH_CHECK("track_gate_kernel");
  launch_cluster_ex(pdl, track_spawn_kernel, grid_, G, smem, st, d_);
  *launches += 4;
}

void TrackerState::check_errors(cudaStream_t st, bool log_too) {
  std::vector<int32_t> e(S_);
  TRB_CUDA(cudaMemcpyAsync(e.data(), d_.err, sizeof(int32_t) * S_, cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  for (int s = 0; s < S_; ++s) {
    if (e[s] & 1) throw Error(TRB_CAPACITY, "tracker: track capacity exceeded on stream " + std::to_string(s));
    if ((e[s] & 2) && log_too)
      throw Error(TRB_CAPACITY, "tracker: track-log ring full on stream " + std::to_string(s) +
                                    " (drain it with trb_streams_drain_log or raise trb_streams_options.log_cap)");
  }
}

int TrackerState::num_tracks(int s, cudaStream_t st) {
  int32_t n = 0;
  TRB_CUDA(cudaMemcpyAsync(&n, d_.n_list + s, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  return n;
}

void TrackerState::tracks(int s, trb_track* out, int cap, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(S_) * T_;
  std::vector<int32_t> i32(4 * S_ + 8 * n);
  std::vector<double> f(2 * n);
  TRB_CUDA(cudaMemcpyAsync(i32.data(), i32_.p, sizeof(int32_t) * i32.size(), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaMemcpyAsync(f.data(), f64_.p, sizeof(double) * f.size(), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  const int32_t* p = i32.data() + 4 * S_;
  const int nl = i32[s];
  for (int i = 0; i < nl && i < cap; ++i) {
    const int slot = p[static_cast<int64_t>(s) * T_ + i];
    const int64_t g = static_cast<int64_t>(s) * T_ + slot;
    trb_track& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.track_id = p[n + g];
    o.w = p[2 * n + g];
    o.h = p[3 * n + g];
    o.status = p[4 * n + g];
    o.lost_frames = p[5 * n + g];
    o.k = K_;
    o.cx = f[g];
    o.cy = f[n + g];
  }
}

void TrackerState::track_model(int s, int i, double* centers, double* hist, cudaStream_t st) {
  int32_t slot = 0;
  TRB_CUDA(cudaMemcpyAsync(&slot, d_.list + static_cast<int64_t>(s) * T_ + i, sizeof(int32_t), cudaMemcpyDeviceToHost,
                           st));
  TRB_CUDA(cudaStreamSynchronize(st));
  const int64_t g = static_cast<int64_t>(s) * T_ + slot;
  if (centers)
    TRB_CUDA(cudaMemcpyAsync(centers, d_.centers + g * 3 * K_, sizeof(double) * 3 * K_, cudaMemcpyDeviceToHost, st));
  if (hist) TRB_CUDA(cudaMemcpyAsync(hist, d_.hist + g * K_, sizeof(double) * K_, cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
}

int64_t TrackerState::log_size(int s, cudaStream_t st) {
  int64_t ht[2] = {0, 0};
  TRB_CUDA(cudaMemcpyAsync(&ht[0], d_.n_log + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaMemcpyAsync(&ht[1], d_.log_tail + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  return std::min(ht[0] - ht[1], log_cap_);
}

// entries [tail, tail + n) of the ring of stream s, oldest first
static int64_t copy_log_ring(const TrackDev& d, int s, int64_t cap, trb_track_log_entry* out, int64_t* tail_out,
                             cudaStream_t st) {
  int64_t ht[2] = {0, 0};
  TRB_CUDA(cudaMemcpyAsync(&ht[0], d.n_log + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaMemcpyAsync(&ht[1], d.log_tail + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  const int64_t tail = ht[1], n = std::min(std::min(ht[0] - tail, d.log_cap), cap);
  const trb_track_log_entry* ring = d.log + static_cast<int64_t>(s) * d.log_cap;
  const int64_t p0 = tail % d.log_cap, n0 = std::min(n, d.log_cap - p0);
  if (n0 > 0)
    TRB_CUDA(cudaMemcpyAsync(out, ring + p0, sizeof(trb_track_log_entry) * n0, cudaMemcpyDeviceToHost, st));
  if (n > n0)
    TRB_CUDA(cudaMemcpyAsync(out + n0, ring, sizeof(trb_track_log_entry) * (n - n0), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  *tail_out = tail;
  return n;
}

void TrackerState::log(int s, trb_track_log_entry* out, int64_t cap, cudaStream_t st) {
  int64_t tail = 0;
  copy_log_ring(d_, s, cap, out, &tail, st);
}

int64_t TrackerState::drain_log(int s, trb_track_log_entry* out, int64_t cap, cudaStream_t st) {
  int64_t tail = 0;
  const int64_t n = copy_log_ring(d_, s, cap, out, &tail, st);
  tail += n;
  TRB_CUDA(cudaMemcpyAsync(d_.log_tail + s, &tail, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  return n;
}

namespace {
// One CTA per stream: the step's blob table and log entries, packed
__global__ void __launch_bounds__(128) pack_step_kernel(TrackDev d, const trb_blob* blobs, int64_t blob_stride,
                                                        const int32_t* nblobs, int32_t* n_blobs_out,
                                                        trb_blob* blobs_out, int bcap, int32_t* n_log_out,
                                                        trb_track_log_entry* log_out, int lcap) {
  const int s = blockIdx.x;
  const int nb = nblobs[s];
  const int64_t base = d.step_log_base[s];
  const int nl = static_cast<int>(d.n_log[s] - base);
  if (threadIdx.x == 0) n_blobs_out[s] = nb, n_log_out[s] = nl;
  const trb_blob* src = blobs + static_cast<int64_t>(s) * blob_stride;
  trb_blob* dst = blobs_out + static_cast<int64_t>(s) * bcap;
  for (int i = threadIdx.x; i < min(nb, bcap); i += blockDim.x) dst[i] = src[i];
  const trb_track_log_entry* ring = d.log + static_cast<int64_t>(s) * d.log_cap;
  trb_track_log_entry* ldst = log_out + static_cast<int64_t>(s) * lcap;
  for (int i = threadIdx.x; i < min(nl, lcap); i += blockDim.x) ldst[i] = ring[(base + i) % d.log_cap];
}
}  // namespace

void TrackerState::pack_step(const trb_blob* blobs, int64_t blob_stride, const int32_t* nblobs, int32_t* n_blobs_out,
                             trb_blob* blobs_out, int bcap, int32_t* n_log_out, trb_track_log_entry* log_out, int lcap,
                             cudaStream_t st) {
  pack_step_kernel<<<S_, 128, 0, st>>>(d_, blobs, blob_stride, nblobs, n_blobs_out, blobs_out, bcap, n_log_out,
                                       log_out, lcap);
  TRB_LAUNCH_CHECK("pack_step_kernel");
}

int TrackerState::frames_processed(int s, cudaStream_t st) {
  int32_t n = 0;
  TRB_CUDA(cudaMemcpyAsync(&n, d_.frame_no + s, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  return n;
}

// ---- standalone ops ----
static DevBuf& scratch_bp() {
  thread_local DevBuf b;
  return b;
}

static void scratch_for(OneArgs& a) {
  DevBuf& b = scratch_bp();
  a.maxN = static_cast<int64_t>(a.W) * a.H;
  a.scratch_stride = (TrackScratch::bytes(cluster_size(), a.maxN) + 255) & ~size_t(255);
  b.alloc(a.scratch_stride, false);
  a.scratch = b.as<unsigned char>();
}

static void launch_one(const OneArgs& a, size_t smem, cudaStream_t st) {
  const int G = cluster_size();
  if (engine_v2(a.K, a.CH, static_cast<int64_t>(a.W) * a.H)) {
    const size_t s2 = check_smem_v2(a.K, a.W, a.H);
    thread_local DevBuf u2, words;
    u2.alloc(sizeof(double) * V2Smem::u2_doubles(a.W, a.H) * G, false);
    words.alloc(sizeof(uint32_t) * V2Smem::words_per_cluster(static_cast<int64_t>(a.W) * a.H, G), false);
    OneArgs b = a;
    b.u2 = u2.as<double>();
    b.words = words.as<uint32_t>();
    prepare_cluster_kernel(track_one2_kernel, s2, G);
    launch_cluster(track_one2_kernel, 1, G, s2, st, b);
    return;
  }
  prepare_cluster_kernel(track_one_kernel, smem, G);
  launch_cluster(track_one_kernel, 1, G, smem, st, a);
}

void device_meanshift_step(const uint8_t* frame_dev, int w, int h, int ch, double* cx, double* cy, int tw, int th,
                           const double* centers, const double* target, int k, int max_iters, double eps,
                           int* status, cudaStream_t st) {
  DevBuf buf;
  buf.alloc(sizeof(double) * (4 * k + 8), false);
  double* dc = buf.as<double>();
  TRB_CUDA(cudaMemcpyAsync(dc, centers, sizeof(double) * 3 * k, cudaMemcpyHostToDevice, st));
  TRB_CUDA(cudaMemcpyAsync(dc + 3 * k, target, sizeof(double) * k, cudaMemcpyHostToDevice, st));
  OneArgs a{};
  a.frame = frame_dev;
  a.W = w, a.H = h, a.CH = ch;
  a.cx = *cx, a.cy = *cy, a.w = tw, a.h = th, a.status = *status, a.K = k, a.max_iters = max_iters, a.eps = eps;
  a.mode = 0;
  a.centers = dc;
  a.target = dc + 3 * k;
  a.out = dc + 4 * k;
  scratch_for(a);
  const size_t smem = check_smem(k, w, h);
  launch_one(a, smem, st);
  double out[3];
  TRB_CUDA(cudaMemcpyAsync(out, a.out, sizeof(out), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  *cx = out[0], *cy = out[1], *status = static_cast<int>(out[2]);
}

bool device_histogram(const uint8_t* frame_dev, int w, int h, int ch, double cx, double cy, int tw, int th,
                      const double* centers, int k, int epanechnikov, double* hist, cudaStream_t st) {
  DevBuf buf;
  buf.alloc(sizeof(double) * (4 * k + 8), false);
  double* dc = buf.as<double>();
  TRB_CUDA(cudaMemcpyAsync(dc, centers, sizeof(double) * 3 * k, cudaMemcpyHostToDevice, st));
  OneArgs a{};
  a.frame = frame_dev;
  a.W = w, a.H = h, a.CH = ch;
  a.cx = cx, a.cy = cy, a.w = tw, a.h = th, a.K = k, a.epan = epanechnikov, a.mode = 1;
  a.centers = dc;
  a.out = dc + 3 * k;
  scratch_for(a);
  const size_t smem = check_smem(k, w, h);
  launch_one(a, smem, st);
  std::vector<double> out(k + 1);
  TRB_CUDA(cudaMemcpyAsync(out.data(), a.out, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
  if (out[k] == 0.0) return false;
  std::memcpy(hist, out.data(), sizeof(double) * k);
  return true;
}

void device_quantize_colors(const double* pixels, int64_t n, int k, int iters, uint64_t seed, double* centers,
                            cudaStream_t st) {
  if (k < 2) throw Error(TRB_INVALID_ARGUMENT, "quantize_colors needs k >= 2");
  if (iters < 1) throw Error(TRB_INVALID_ARGUMENT, "quantize_colors needs iters >= 1");
  if (n < k)
    throw Error(TRB_INVALID_ARGUMENT,
                "quantize_colors: " + std::to_string(n) + " pixels < k=" + std::to_string(k));
  std::vector<int> ip(static_cast<size_t>(n) * 3);
  bool integral = true;
  for (int64_t i = 0; i < 3 * n && integral; ++i) {
    const double v = pixels[i];
    integral = v >= 0.0 && v <= 65535.0 && v == static_cast<double>(static_cast<int>(v));
    if (integral) ip[i] = static_cast<int>(v);
  }
  if (!integral) {  // general real-valued samples: the sequential device kernel
    DevBuf dpx, dc, dd2, das, dsum, dcnt, drng;
    dpx.alloc(sizeof(double) * 3 * n, false);
    dc.alloc(sizeof(double) * 3 * k, false);
    dd2.alloc(sizeof(double) * 2 * n, false);  // D^2 + its running prefix
    das.alloc(sizeof(int) * n, false);
    dsum.alloc(sizeof(double) * 3 * k, false);
    dcnt.alloc(sizeof(int64_t) * k, false);
    drng.alloc(sizeof(Mt64), false);
    TRB_CUDA(cudaMemcpyAsync(dpx.p, pixels, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    quantize_serial_kernel<<<1, 1024, 0, st>>>(dpx.as<double>(), n, k, iters, seed, dc.as<double>(), dd2.as<double>(),
                                            das.as<int>(), dsum.as<double>(), dcnt.as<int64_t>(), drng.as<Mt64>());
    TRB_LAUNCH_CHECK("quantize_serial_kernel");
    TRB_CUDA(cudaMemcpyAsync(centers, dc.p, sizeof(double) * 3 * k, cudaMemcpyDeviceToHost, st));
    TRB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DevBuf dpx, dout;
  dpx.alloc(sizeof(int) * ip.size(), false);
  dout.alloc(sizeof(double) * 3 * k, false);
  TRB_CUDA(cudaMemcpyAsync(dpx.p, ip.data(), sizeof(int) * ip.size(), cudaMemcpyHostToDevice, st));
  const size_t smem = check_smem(k, 1, 1);
  set_smem(reinterpret_cast<const void*>(quantize_kernel), smem);
  quantize_kernel<<<1, NT, smem, st>>>(dpx.as<int>(), static_cast<int>(n), k, iters, seed, dout.as<double>());
  TRB_LAUNCH_CHECK("quantize_kernel");
  TRB_CUDA(cudaMemcpyAsync(centers, dout.p, sizeof(double) * 3 * k, cudaMemcpyDeviceToHost, st));
  TRB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace trb
