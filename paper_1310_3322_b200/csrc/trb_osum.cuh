// trb_osum.cuh — cluster-parallel, bit-exact reproduction of SEQUENTIAL
// fp64 summations  S_j = fl(S_{j-1} + a_j), S_{-1} = +0, a_j >= 0.
//
// Why: the reference tracker accumulates its Epanechnikov histogram
// (tracking.hpp:86-98) and its mean-shift centroid (tracking.hpp:135-146) as
// plain sequential double sums in raster order; the track log is printed
// with %.17g, so a tree reduction (different rounding) would break parity.
//
// Idea.  While the running sum S stays inside one binade [2^e, 2^(e+1)) it
// is X*u with u = 2^(e-52) and X an integer in [2^52, 2^53).  For a step
// with a >= 0 that keeps S in the binade, fl(S + a) = (X + RN(a/u))*u where
// the rounding of a/u to an integer depends on a alone — except when a/u is
// exactly k + 1/2, where round-half-even gives E(X + k) with
// E(y) = y + (y & 1) ("up to even").  Both step kinds are integer maps
//         add(r):  X -> X + r          tie(k):  X -> E(X + k)
// and the set {X -> X + B} U {X -> E(X + A) + B} is closed under
// composition (E(X+A) is even, so E(E(X+A) + y) = E(X+A) + E(y)).  A run of
// steps inside one binade is therefore a "piece" (tie?, A, B) of exact int64
// numbers, and pieces compose associatively — a parallel scan.  The only
// steps left for a serial replay are "breakpoints": the first element and
// binade crossings (~log2 of the dynamic range per sum).  Which binade a step
// sees is predicted from an approximate parallel prefix P (relative error
// <= delta); a step whose interval [P(1-delta), P_next(1+delta)] is not inside
// one binade becomes a breakpoint, and the replay re-verifies every
// prediction, falling back to a full serial sum (exact by construction) if
// one ever fails.
//
// Shape: one thread-block CLUSTER of G CTAs x NT threads; cluster thread g
// owns the contiguous element chunk [g*C, (g+1)*C).  Up to 3 lanes (sums fed
// by the same elements) and optional segments (independent sums laid end to
// end; used for the histogram bins after a stable partition by bin).  All
// per-thread state lives in registers.
//   phase A  chunk totals -> segmented cluster scan (warp shuffles, smem,
//            DSMEM carry) -> approximate prefix at every chunk start
//   phase B  walk the chunk: safe/tie steps compose into the thread's piece,
//            breakpoints are recorded (piece-before, value, index)
//   phase C  segmented cluster scan of the thread pieces (reset at
//            breakpoints); the carried-in piece is folded into each thread's
//            first breakpoint; breakpoints ranked into one cluster list
//   phase D  every CTA replays each lane / segment serially from its copy
//            of the gathered list (no barrier after it).
#pragma once

#include <cooperative_groups.h>
#include <limits.h>

#include "trb_exact.cuh"

#ifndef TRB_OSUM_WALK_BEGIN
#define TRB_OSUM_WALK_BEGIN()
#define TRB_OSUM_WALK_END()
#define TRB_OSUM_COUNT(v)
#define TRB_OSUM_WALK_FIRST(cond, dep)
#define TRB_OSUM_ELEM_TRACE(k, dep)
#endif
#ifndef TRB_OSUM_MARK
#define TRB_OSUM_MARK(stage) ((void)0)
#endif

namespace trb {

namespace cg = cooperative_groups;

#ifndef TRB_NT
#define TRB_NT 256
#endif
constexpr int kOsumThreads = TRB_NT;
constexpr int kOsumBpRecs = 240;  // breakpoint records per CTA (all lanes)
constexpr int kMaxCluster = 16;
constexpr int kMaxSegs = 256;     // segments (histogram bins) per run
constexpr int kOsumGather = 480;  // cluster-wide breakpoints gathered in CTA 0 (all lanes)
constexpr int kEmptyE = INT_MIN;

// ----------------------------------------------------------- piece algebra
struct Piece {
  long long A, B;
  int e;    // binade of every step in the piece, kEmptyE = identity
  int tie;  // 0: X -> X + B ; 1: X -> E(X + A) + B
};

__device__ __forceinline__ Piece piece_identity() { return Piece{0, 0, kEmptyE, 0}; }
__device__ __forceinline__ long long up_even(long long y) { return y + (y & 1); }

// p then q; *bad is set when two non-empty pieces disagree on the binade
__device__ __forceinline__ Piece compose(const Piece& p, const Piece& q, int* bad) {
  if (q.e == kEmptyE) return p;
  if (p.e == kEmptyE) return q;
  if (p.e != q.e) *bad = 1;
  Piece r;
  r.e = p.e;
  if (!q.tie) {
    r.tie = p.tie, r.A = p.A, r.B = p.B + q.B;
  } else if (!p.tie) {
    r.tie = 1, r.A = p.B + q.A, r.B = q.B;
  } else {
    r.tie = 1, r.A = p.A, r.B = up_even(p.B + q.A) + q.B;
  }
  return r;
}

__device__ __forceinline__ long long apply(const Piece& p, long long X) {
  return p.tie ? up_even(X + p.A) + p.B : X + p.B;
}

__device__ __forceinline__ int osum_exp(double x) {  // binade of a positive normal double, else kEmptyE
  const long long b = __double_as_longlong(x);
  const int be = static_cast<int>((b >> 52) & 0x7ff);
  return (be == 0 || be == 0x7ff || b < 0) ? kEmptyE : be - 1023;
}

// 2^k as a double for -1022 <= k <= 1023 (exact, no libm call)
__device__ __forceinline__ double osum_pow2(int k) {
  return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
}

// ------------------------------------------------------------- records
struct OsumBp {
  Piece p;      // piece before this step (after the fold: since the previous breakpoint)
  double v;     // the element value
  int j;        // element index
  short t;      // owning thread (CTA-local)
  char first;   // first breakpoint of this lane in the thread's chunk
  char start;   // the element starts a segment
  int seg;      // segment id (SEG runs)
  int pad;
};

// Shared memory of the engine (static size).
struct OsumShared {
  OsumBp bp[kOsumBpRecs];
  double warp_d[32][4];       // phase A warp aggregates: [warp][f, P0..P2]
  double cta_d[2][4];         // phase A CTA aggregate (double-buffered)
  Piece warp_p[32][3];
  int warp_pf[32][3];
  Piece wpre_p[32][3];  // phase C: exclusive prefix of the warps before w (inside the CTA)
  int wpre_f[32][3];
  int warp_pbad[32];
  Piece cta_p[2][3];
  int cta_pf[2][3];
  int nbp[3];
  int bp_base[3];
  int nbp_total[3];
  Piece carry_p[3];
  Piece fin_p[3];
  int bad[4];
  int segpos[kMaxSegs + 1];
  double result[kMaxSegs];
  int phase;
  // parallel DSMEM gathers of the other CTAs' aggregates
  double gath_d[kMaxCluster][4];
  Piece gath_p[kMaxCluster][3];
  int gath_pf[kMaxCluster][3];
  int gath_n[kMaxCluster][3];
  // cluster-wide ranked breakpoint list, gathered into CTA 0 (DSMEM stores).
  // Free while phases A/B walk the elements: the element sources use it as
  // their cp.async staging ring (osum_stage()).
  alignas(16) OsumBp gbp[kOsumGather];
};
constexpr int kOsumStageBytes = kOsumGather * static_cast<int>(sizeof(OsumBp));
__device__ __forceinline__ uint4* osum_stage(OsumShared& s) { return reinterpret_cast<uint4*>(&s.gbp[0]); }

// cp.async (global -> shared, 16 bytes, bypassing registers): the element
// sources stage read-ahead data in shared memory, because a register that a
// pending load targets stalls every instruction that touches it (including
// the compiler's own moves), which defeats register read-ahead.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The CTA group one engine run spans: the whole thread-block cluster, or a
// single CTA acting alone ("split mode": each CTA of a cluster runs its own
// small track; barriers degrade to __syncthreads, DSMEM maps to itself).
struct Grp {
  int rank_, size_;
  __device__ static Grp cluster() {
    cg::cluster_group c = cg::this_cluster();
    return Grp{static_cast<int>(c.block_rank()), static_cast<int>(c.num_blocks())};
  }
  __device__ static Grp single() { return Grp{0, 1}; }
  __device__ unsigned block_rank() const { return static_cast<unsigned>(rank_); }
  __device__ unsigned num_blocks() const { return static_cast<unsigned>(size_); }
  __device__ void sync() const {
    if (size_ > 1) cg::this_cluster().sync();
    else __syncthreads();
  }
  template <class T>
  __device__ T* map_shared_rank(T* p, int r) const {
    return size_ > 1 ? cg::this_cluster().map_shared_rank(p, r) : p;
  }
};

// A safe step a of binade e (M = 2^e) appended to the thread's piece.  The
// identity piece is {B = 0, A = 0, tie = 0}, so a plain step needs no test of
// emptiness: B += r and the binade is (re)stated.
__device__ __forceinline__ void osum_step_safe(Piece& pc, double a, double M, int e, int& tbad) {
  const double y = xadd(M, a);
  const double d = xsub(a, xsub(y, M));
  const long long r = __double_as_longlong(y) - __double_as_longlong(M);
  const double hu = __longlong_as_double(__double_as_longlong(M) - (53LL << 52));  // u/2
  if (fabs(d) == hu) {  // a/u = k + 1/2
    Piece q;
    q.e = e, q.tie = 1, q.A = d > 0.0 ? r : r - 1, q.B = 0;
    pc = compose(pc, q, &tbad);
  } else {
    pc.B += r;
    pc.e = e;
  }
}

// warp-shuffle helpers for the scan payloads
__device__ __forceinline__ Piece shfl_up_piece(const Piece& p, int o) {
  Piece r;
  r.A = __shfl_up_sync(0xffffffffu, p.A, o);
  r.B = __shfl_up_sync(0xffffffffu, p.B, o);
  r.e = __shfl_up_sync(0xffffffffu, p.e, o);
  r.tie = __shfl_up_sync(0xffffffffu, p.tie, o);
  return r;
}

// Exact serial fallback (one thread): the sums in element order with real
// IEEE adds.  Out of line — it is cold, and keeping it out of the hot
// function keeps the per-iteration instruction footprint small.
template <int L, bool SEG, class Src>
__device__ __noinline__ void osum_serial(int N, int nseg, int C, int GT, const Src& src, OsumShared& s) {
  double S[L];
#pragma unroll
  for (int l = 0; l < L; ++l) S[l] = 0.0;
  int cs = -1;
  for (int g = 0; g < GT; ++g) {  // chunk by chunk, in order
    int a0, a1;
    Src::bounds(N, GT, g, a0, a1);
    if (a0 >= a1) continue;
    auto cur = src.begin(a0, g, C, GT);
    for (int jb = a0; jb < a1; jb += Src::kUnroll)
#pragma unroll
      for (int k = 0; k < Src::kUnroll; ++k) {
        if (jb + k >= a1) break;
        bool start, has;
        int seg;
        double v[L];
        cur.next(k, start, seg, has, v);
        if (SEG && start) {
          if (cs >= 0) s.result[cs] = S[0];
          cs = seg;
          S[0] = 0.0;
        }
        if (!has) continue;
#pragma unroll
        for (int l = 0; l < L; ++l) S[l] = xadd(S[l], v[l]);
      }
  }
  if (SEG) {
    for (int k = 0; k < nseg; ++k)
      if (s.segpos[k] < 0) s.result[k] = 0.0;
    if (cs >= 0) s.result[cs] = S[0];
  } else {
#pragma unroll
    for (int l = 0; l < L; ++l) s.result[l] = S[l];
  }
}

// One run of the engine.
//   Src::bounds(N, GT, gt, j0, j1): thread gt's chunk [j0, j1) (contiguous,
//   in thread order; Src::max_chunk bounds its length);
//   Src::Cursor cur = src.begin(j0, gt, C, GT);  cur.next(k, start, seg, has, v)
//   walks elements j0, j0+1, ... of thread gt's chunk, k = (j - j0) %
//   Src::kUnroll (the loops unroll by kUnroll so k is static) (the source may
//   store chunks interleaved: element gt*C + i at i*GT + gt); `start` marks a segment start (SEG only), `has`
//   whether the element contributes, v[L] its values (>= 0).
//   results: SEG -> s.result[seg] for seg < nseg (0 for empty segments);
//            else s.result[lane].  Visible in every CTA on return.
// stats (optional, global): [0] runs, [1] lanes/segments, [2] fallbacks,
// [3] breakpoints, [4] elements, [16+bit] failure reasons.
template <int L, bool SEG, class Src>
__device__ void osum_run(const Grp& cl, int N, int nseg, const Src& src, OsumShared& s,
                         unsigned long long* stats = nullptr) {
  const int NT = blockDim.x, t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  const int rank = static_cast<int>(cl.block_rank()), G = static_cast<int>(cl.num_blocks());
  const int GT = G * NT, gt = rank * NT + t;
  const int C = Src::max_chunk(N, GT);  // longest chunk (error budget below)
  int j0, j1;
  Src::bounds(N, GT, gt, j0, j1);
  // relative error bound of every approximate prefix P:
  //   delta = (N + 2C + 96 + G) * 2^-52
  // mantissa bounds (units of 2^-52 of the binade) equivalent to a relative
  // margin of >= 2*delta on each side: 2*delta*2^52 = 2*(N + 2C + 96 + G)
  // (integer arithmetic, so it stays cheap wherever the compiler re-derives it)
  constexpr long long kMant = (1LL << 52) - 1;
  const long long marg = 2LL * (N + 2 * C + 96 + G) + 4;
  const long long lowm = marg, highm = kMant - 2 * marg;
  const int cap_lane = kOsumBpRecs / L;
  const int buf = s.phase;  // double-buffer index for the CTA aggregates
  // NB: s.result is NOT touched before the barriers below — callers read the
  // previous run's results right up to this call (CTA 0 rewrites every
  // result, including empty segments, in phase D).
  // (no barrier: nbp / bad are first used after phase A's barriers, and the
  // previous run's readers finished before its closing barrier)
  if (t < 3) s.nbp[t] = 0;
  if (t < 4) s.bad[t] = 0;

  // ---------------- phase A: approximate (segmented) prefix at chunk starts
  int af = 0;
  double aP[L];
#pragma unroll
  for (int l = 0; l < L; ++l) aP[l] = 0.0;
  {
    auto cur = src.begin(j0, gt, C, GT);
    // unrolled so the cursor's read-ahead slots are static registers
    for (int jb = j0; jb < j1; jb += Src::kUnroll)
#pragma unroll
    for (int k = 0; k < Src::kUnroll; ++k) {
      const int j = jb + k;
      if (j >= j1) break;
      bool start, has;
      int seg;
      double v[L];
      cur.next(k, start, seg, has, v);
      if (SEG && start) {
        af = 1;
#pragma unroll
        for (int l = 0; l < L; ++l) aP[l] = 0.0;
      }
      if (has)
#pragma unroll
        for (int l = 0; l < L; ++l) aP[l] = xadd(aP[l], v[l]);
    }
  }
  // warp inclusive segmented scan
  int sf = af;
  double sP[L];
#pragma unroll
  for (int l = 0; l < L; ++l) sP[l] = aP[l];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int pf = __shfl_up_sync(0xffffffffu, sf, o);
    double pP[L];
#pragma unroll
    for (int l = 0; l < L; ++l) pP[l] = __shfl_up_sync(0xffffffffu, sP[l], o);
    if (lane >= o && !sf) {
      sf = pf;
#pragma unroll
      for (int l = 0; l < L; ++l) sP[l] = xadd(pP[l], sP[l]);
    }
  }
  if (lane == 31) {
    s.warp_d[wid][0] = sf;
#pragma unroll
    for (int l = 0; l < L; ++l) s.warp_d[wid][1 + l] = sP[l];
  }
  __syncthreads();
  if (t == 0) {  // CTA aggregate
    int f = 0;
    double P[L];
#pragma unroll
    for (int l = 0; l < L; ++l) P[l] = 0.0;
    for (int w = 0; w < nw; ++w) {
      if (s.warp_d[w][0] != 0.0) {
        f = 1;
#pragma unroll
        for (int l = 0; l < L; ++l) P[l] = s.warp_d[w][1 + l];
      } else {
#pragma unroll
        for (int l = 0; l < L; ++l) P[l] = xadd(P[l], s.warp_d[w][1 + l]);
      }
    }
    s.cta_d[buf][0] = f;
#pragma unroll
    for (int l = 0; l < L; ++l) s.cta_d[buf][1 + l] = P[l];
  }
  TRB_OSUM_MARK(1);
  cl.sync();
  TRB_OSUM_MARK(2);
  // gather the lower CTAs' aggregates once (parallel DSMEM loads), then
  // exclusive prefix for this thread: carry(CTAs < rank) . warps < wid . lanes < lane
  if (t < rank) {
    const double* d = cl.map_shared_rank(&s.cta_d[buf][0], t);
#pragma unroll
    for (int q = 0; q < 4; ++q) s.gath_d[t][q] = d[q];
  }
  __syncthreads();
  double xP[L];
  {
    int f = 0;
#pragma unroll
    for (int l = 0; l < L; ++l) xP[l] = 0.0;
    for (int r = 0; r < rank; ++r) {
      const double* d = s.gath_d[r];
      if (d[0] != 0.0) {
        f = 1;
#pragma unroll
        for (int l = 0; l < L; ++l) xP[l] = d[1 + l];
      } else {
#pragma unroll
        for (int l = 0; l < L; ++l) xP[l] = xadd(xP[l], d[1 + l]);
      }
    }
    for (int w = 0; w < wid; ++w) {
      if (s.warp_d[w][0] != 0.0) {
#pragma unroll
        for (int l = 0; l < L; ++l) xP[l] = s.warp_d[w][1 + l];
      } else {
#pragma unroll
        for (int l = 0; l < L; ++l) xP[l] = xadd(xP[l], s.warp_d[w][1 + l]);
      }
    }
    // lanes before me inside the warp: exclusive = inclusive of lane-1
    const int lf = __shfl_up_sync(0xffffffffu, sf, 1);
    double lP[L];
#pragma unroll
    for (int l = 0; l < L; ++l) lP[l] = __shfl_up_sync(0xffffffffu, sP[l], 1);
    if (lane > 0) {
      if (lf) {
#pragma unroll
        for (int l = 0; l < L; ++l) xP[l] = lP[l];
      } else {
#pragma unroll
        for (int l = 0; l < L; ++l) xP[l] = xadd(xP[l], lP[l]);
      }
    }
    (void)f;
  }

  TRB_OSUM_MARK(3);
  TRB_OSUM_WALK_BEGIN();
  // ---------------- phase B: classify every step
  // A lane is "armed" for binade e once a step has been verified safe there:
  // P only grows inside a segment, so later steps stay safe while P_next <=
  // hi (= the highm bound of binade e) and only that one compare is needed.
  // The rounding of a step a to the grid u = 2^(e-52) is read off
  // y = fl(2^e + a) (exact for 0 <= a < 2^e, round-half-even like the sum);
  // a tie shows as |a - (y - 2^e)| == u/2.
  Piece pc[L];
  int hadbp[L], firstbp[L];
  double hi[L], M[L];
  int ea[L];
  int tbad = 0, tover = 0;
#pragma unroll
  for (int l = 0; l < L; ++l)
    pc[l] = piece_identity(), hadbp[l] = 0, firstbp[l] = -1, hi[l] = -1.0, M[l] = 1.0, ea[l] = 0;
  // Segment heads.  The state at a segment start (element 0 of a plain run)
  // is exactly +0, so the thread owning that element sums from there to the
  // next start / its chunk end with real IEEE adds — the exact sequential
  // prefix — and records it as ONE breakpoint (value = that sum, piece =
  // its steps before the start).  The replay's S = +0 + sum reproduces the
  // state; no step of a head is classified (a young sum crosses a binade
  // every few elements, which made the owning thread the cluster's slowest).
  bool inhead = false;
  int hj = 0, hseg = 0;
  double Sh[L];
#pragma unroll
  for (int l = 0; l < L; ++l) Sh[l] = 0.0;
  auto emit_head = [&]() {
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const int idx = atomicAdd(&s.nbp[l], 1);
      if (idx < cap_lane) {
        OsumBp& b = s.bp[l * cap_lane + idx];
        b.p = pc[l];
        b.v = Sh[l];
        b.j = hj;
        b.t = static_cast<short>(t);
        b.first = static_cast<char>(!hadbp[l]);
        b.start = static_cast<char>(SEG);
        b.seg = hseg;
        if (!hadbp[l]) firstbp[l] = idx;
      } else {
        tover = 1;
      }
      hadbp[l] = 1;
      pc[l] = piece_identity();
      hi[l] = -1.0;
    }
  };
  {
    double P[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
      P[l] = xP[l];
      // pre-armed from the prefix before the first step (lower margin met):
      // the first step is then safe iff P_next <= hi, as for any armed step
      const long long bp_ = __double_as_longlong(xP[l]);
      const int eb = static_cast<int>(bp_ >> 52);
      if (xP[l] > 0.0 && eb > 64 && eb < 1982 && (bp_ & kMant) >= lowm) {
        hi[l] = __longlong_as_double((static_cast<long long>(eb) << 52) | highm);
        M[l] = osum_pow2(eb - 1023);
        ea[l] = eb - 1023;
      }
    }
    auto cur = src.begin(j0, gt, C, GT);
    static_assert(Src::kUnroll == 1, "phase B walks one element per iteration");
    for (int j = j0; j < j1; ++j) {
      bool start, has;
      int seg;
      double v[L];
      cur.next(0, start, seg, has, v);
      TRB_OSUM_WALK_FIRST(j == j0, v[0]);
      TRB_OSUM_ELEM_TRACE(j - j0, v[0]);
      const bool hs = SEG ? start : j == 0;
      if (!hs && !inhead) {
        // the common step, kept lean (no branch per lane, no state merges):
        // every lane armed with P_next <= hi and no tie -> X += RN(a/u).
        // Anything else (arming, binade crossing, tie, head) falls through
        // to the general code below for this element.
        if (!has) continue;
        bool ok = true;
        double Pn[L];
        long long r[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
          Pn[l] = xadd(P[l], v[l]);
          const double y = xadd(M[l], v[l]);
          const double d = xsub(v[l], xsub(y, M[l]));
          const double hu = __longlong_as_double(__double_as_longlong(M[l]) - (53LL << 52));  // u/2
          ok = ok & (Pn[l] <= hi[l]) & (fabs(d) != hu);
          r[l] = __double_as_longlong(y) - __double_as_longlong(M[l]);
        }
        if (ok) {
#pragma unroll
          for (int l = 0; l < L; ++l) pc[l].B += r[l], pc[l].e = ea[l], P[l] = Pn[l];
          continue;
        }
      }
      if (hs) {  // a segment head begins (S = +0 exactly)
        if (inhead) emit_head();
        inhead = true, hj = j, hseg = seg;
#pragma unroll
        for (int l = 0; l < L; ++l) Sh[l] = 0.0;
      }
      if (inhead) {
        if (has)
#pragma unroll
          for (int l = 0; l < L; ++l) Sh[l] = xadd(Sh[l], v[l]);
        continue;
      }
      if (SEG && start)
#pragma unroll
        for (int l = 0; l < L; ++l) P[l] = 0.0;
      if (!has) continue;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const double vl = v[l];
        const double Pp = P[l];
        const double Pn = xadd(Pp, vl);
        P[l] = Pn;
        if (!(SEG && start) && Pn <= hi[l]) {  // armed: a safe step of binade ea
          osum_step_safe(pc[l], vl, M[l], ea[l], tbad);
          continue;
        }
        TRB_OSUM_COUNT(nslow_);
        // a zero step never changes S — except at a segment start, where it
        // must still open the segment (S = +0 + 0)
        if (vl == 0.0 && !(SEG && start)) continue;
        bool safe = false;
        if (Pp > 0.0 && !(SEG && start)) {
          // P and P_next in one binade with relative margin delta on both
          // sides, checked on the raw bits: P(1-delta) >= 2^e and
          // P_next(1+delta) < 2^(e+1)  <=  mantissa(P) >= lowm, mantissa(P_next) <= highm
          const long long bp_ = __double_as_longlong(Pp), bn_ = __double_as_longlong(Pn);
          const int eb = static_cast<int>(bp_ >> 52);
          if (eb == static_cast<int>(bn_ >> 52) && eb > 64 && eb < 1982 && (bp_ & kMant) >= lowm &&
              (bn_ & kMant) <= highm) {
            hi[l] = __longlong_as_double((static_cast<long long>(eb) << 52) | highm);
            M[l] = osum_pow2(eb - 1023);
            ea[l] = eb - 1023;
            safe = true;
          }
        }
        if (safe) {
          osum_step_safe(pc[l], vl, M[l], ea[l], tbad);
        } else {
          TRB_OSUM_COUNT(nbp_);
          const int idx = atomicAdd(&s.nbp[l], 1);
          if (idx < cap_lane) {
            OsumBp& b = s.bp[l * cap_lane + idx];
            b.p = pc[l];
            b.v = vl;
            b.j = j;
            b.t = static_cast<short>(t);
            b.first = static_cast<char>(!hadbp[l]);
            b.start = static_cast<char>(SEG && start);
            b.seg = seg;
            if (!hadbp[l]) firstbp[l] = idx;
          } else {
            tover = 1;
          }
          hadbp[l] = 1;
          pc[l] = piece_identity();
          hi[l] = -1.0;
          // re-arm at once from the prefix after this (replayed) step when it
          // clears the lower margin of its binade (as the pre-arming from xP):
          // a crossing then costs one slow step, not two or three
          const long long bn_ = __double_as_longlong(Pn);
          const int en = static_cast<int>(bn_ >> 52);
          if (!(SEG && start) && Pn > 0.0 && en > 64 && en < 1982 && (bn_ & kMant) >= lowm) {
            hi[l] = __longlong_as_double((static_cast<long long>(en) << 52) | highm);
            M[l] = osum_pow2(en - 1023);
            ea[l] = en - 1023;
          }
        }
      }
    }
    if (inhead) emit_head();
  }
  TRB_OSUM_WALK_END();
  TRB_OSUM_MARK(4);
  if (tbad) atomicOr(&s.bad[0], 2);
  if (tover) atomicOr(&s.bad[0], 4);

  // ---------------- phase C: segmented scan of the pieces (per lane)
  Piece xp[L];  // exclusive piece before this thread (since the last breakpoint)
  {
    int wbad = 0;
    Piece sp[L];
    int spf[L];
#pragma unroll
    for (int l = 0; l < L; ++l) sp[l] = pc[l], spf[l] = hadbp[l];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const Piece pp = shfl_up_piece(sp[l], o);
        const int pf = __shfl_up_sync(0xffffffffu, spf[l], o);
        if (lane >= o && !spf[l]) {
          sp[l] = compose(pp, sp[l], &wbad);
          spf[l] = pf;
        }
      }
    }
    if (lane == 31) {
#pragma unroll
      for (int l = 0; l < L; ++l) s.warp_p[wid][l] = sp[l], s.warp_pf[wid][l] = spf[l];
      s.warp_pbad[wid] = wbad;
    }
    TRB_OSUM_MARK(20);
    __syncthreads();
    TRB_OSUM_MARK(21);
    if (t == 0) {
      int bad = 0;
      for (int l = 0; l < L; ++l) {
        Piece a = piece_identity();
        int f = 0;
        for (int w = 0; w < nw; ++w) {
          s.wpre_p[w][l] = a, s.wpre_f[w][l] = f;
          bad |= s.warp_pbad[w];
          if (s.warp_pf[w][l]) a = s.warp_p[w][l], f = 1;
          else a = compose(a, s.warp_p[w][l], &bad);
        }
        s.cta_p[buf][l] = a;
        s.cta_pf[buf][l] = f;
      }
      if (bad) atomicOr(&s.bad[0], 8);
    }
    TRB_OSUM_MARK(5);
    cl.sync();
    TRB_OSUM_MARK(6);
    // carry from lower CTAs, breakpoint bases, cluster-final piece: gather
    // every CTA's aggregate with parallel DSMEM loads, then combine locally
    if (t < G * L) {
      const int r = t / L, l = t - r * L;
      s.gath_p[r][l] = *cl.map_shared_rank(&s.cta_p[buf][l], r);
      s.gath_pf[r][l] = *cl.map_shared_rank(&s.cta_pf[buf][l], r);
      s.gath_n[r][l] = *cl.map_shared_rank(&s.nbp[l], r);
    }
    __syncthreads();
    if (t < L) {
      const int l = t;
      Piece a = piece_identity();
      int base = 0, bad = 0;
      for (int r = 0; r < G; ++r) {
        if (r == rank) s.carry_p[l] = a, s.bp_base[l] = base;
        const Piece rp = s.gath_p[r][l];
        base += min(s.gath_n[r][l], cap_lane);
        if (s.gath_pf[r][l]) a = rp;
        else a = compose(a, rp, &bad);
      }
      s.fin_p[l] = a;
      s.nbp_total[l] = base;
      if (bad) atomicOr(&s.bad[0], 8);
    }
    __syncthreads();
    // exclusive piece of this thread = carry . warps < wid . lanes < lane
#pragma unroll
    for (int l = 0; l < L; ++l) {
      Piece a = s.carry_p[l];
      int bad = 0;
      if (s.wpre_f[wid][l]) a = s.wpre_p[wid][l];
      else a = compose(a, s.wpre_p[wid][l], &bad);
      const Piece lp = shfl_up_piece(sp[l], 1);
      const int lf = __shfl_up_sync(0xffffffffu, spf[l], 1);
      if (lane > 0) {
        if (lf) a = lp;
        else a = compose(a, lp, &bad);
      }
      xp[l] = a;
      if (bad) atomicOr(&s.bad[0], 8);
    }
  }
  // fold the carried-in piece into each thread's first breakpoint (its own
  // record: no barrier needed before, one after — the ranking reads all)
#pragma unroll
  for (int l = 0; l < L; ++l) {
    if (firstbp[l] >= 0) {
      OsumBp& b = s.bp[l * cap_lane + firstbp[l]];
      int bad = 0;
      b.p = compose(xp[l], b.p, &bad);
      if (bad) atomicOr(&s.bad[0], 16);
    }
  }
  __syncthreads();
  TRB_OSUM_MARK(7);
  // rank each CTA list by element index into the cluster list, stored
  // (DSMEM) into EVERY CTA's gathered list: each CTA then replays locally and
  // no barrier is needed after the replay
  const int cap_g = kOsumGather / L;
  for (int l = 0; l < L; ++l) {
    const int n = min(s.nbp[l], cap_lane);
    for (int i = t; i < n; i += NT) {
      const int ji = s.bp[l * cap_lane + i].j;
      int rk = 0;
      for (int q = 0; q < n; ++q) rk += s.bp[l * cap_lane + q].j < ji;
      const int pos = s.bp_base[l] + rk;
      if (pos < cap_g) {
        const OsumBp rec = s.bp[l * cap_lane + i];
        for (int dst = 0; dst < G; ++dst) cl.map_shared_rank(&s.gbp[0], dst)[l * cap_g + pos] = rec;
      } else {
        atomicOr(&s.bad[0], 4);
      }
    }
  }
  __syncthreads();
  if (t == 0 && s.bad[0])
    for (int dst = 0; dst < G; ++dst)
      if (dst != rank) atomicOr(cl.map_shared_rank(&s.bad[0], dst), s.bad[0]);
  TRB_OSUM_MARK(8);
  cl.sync();
  TRB_OSUM_MARK(9);

  // ---------------- phase D: replay (every CTA, identical inputs)
  {
    const int why = s.bad[0];
    if (why && t == 0) s.bad[1] = 1;
    const int nlanes = SEG ? nseg : L;
    if (SEG) {  // segment -> first breakpoint position
      for (int k = t; k <= nseg; k += NT) s.segpos[k] = -1;
      __syncthreads();
      const OsumBp* list = s.gbp;
      const int n0 = min(s.nbp_total[0], cap_g);
      for (int q = t; q < n0; q += NT)
        if (list[q].start) {
          TRB_CHECK(list[q].seg >= 0 && list[q].seg < nseg, "segment id", list[q].seg, q);
          s.segpos[list[q].seg] = q;
        }
      __syncthreads();
    }
    for (int k = t; k < nlanes; k += NT) {
      const int l = SEG ? 0 : k;
      const OsumBp* list = s.gbp + l * cap_g;
      const int n = min(s.nbp_total[l], cap_g);
      int q0 = 0, q1 = n;
      if (SEG) {
        q0 = s.segpos[k];
        if (q0 < 0) {  // empty segment
          s.result[k] = 0.0;
          continue;
        }
        q1 = q0 + 1;
        while (q1 < n && !list[q1].start) ++q1;
      }
      bool ok = !why;
      double S = 0.0;
      // no early exit: the loads of the list do not depend on S, so the loop
      // pipelines; a failed check only clears `ok` (the result is then
      // recomputed by the serial fallback)
      auto run_piece = [&](const Piece& p) {
        if (p.e == kEmptyE) return;
        const int pe = (p.e > -1000 && p.e < 1000) ? p.e : 0;
        ok &= osum_exp(S) == pe;
        // S = X * 2^(pe-52) with X its 53-bit significand: integer ops only
        const long long X = (__double_as_longlong(S) & kMant) | (1LL << 52);
        const long long X2 = apply(p, X);
        ok &= X2 >= (1LL << 52) && X2 < (1LL << 53);
        S = __longlong_as_double((static_cast<long long>(pe + 1023) << 52) | (X2 & kMant));
      };
      for (int q = q0; q < q1; ++q) {
        TRB_CHECK(q >= 0 && q < cap_g, "replay read", q, n);
        const OsumBp b = list[q];
        if (q > q0 || !SEG) run_piece(b.p);  // a segment start's piece belongs to the previous segment
        S = xadd(S, b.v);
      }
      if (ok) run_piece((SEG && q1 < n) ? list[q1].p : s.fin_p[l]);
      s.result[k] = S;
      if (!ok) atomicOr(&s.bad[1], 1);
    }
    __syncthreads();
    if (stats && t == 0 && rank == 0) {
      atomicAdd(&stats[0], 1ull);
      atomicAdd(&stats[1], static_cast<unsigned long long>(nlanes));
      unsigned long long nb = 0;
      for (int l = 0; l < L; ++l) nb += s.nbp_total[l];
      atomicAdd(&stats[3], nb);
      atomicAdd(&stats[4], static_cast<unsigned long long>(N));
      for (int bit = 0; bit < 8; ++bit)
        if (why & (1 << bit)) atomicAdd(&stats[16 + bit], 1ull);
      if (s.bad[1]) atomicAdd(&stats[2], 1ull);
    }
    // exact serial fallback (all lanes / segments) if anything failed
    if (s.bad[1]) {
      if (t == 0) osum_serial<L, SEG>(N, nseg, C, GT, src, s);
      __syncthreads();
    }
  }
  if (t == 0) s.phase = buf ^ 1;
  TRB_OSUM_MARK(10);
  // No cluster barrier: the results are local.  A CTA that runs ahead
  // cannot touch another CTA's shared memory or the element data before that
  // CTA reaches the next run's barriers, and every remote read of this run
  // happened before the barrier above.
  __syncthreads();
  TRB_OSUM_MARK(11);
}

}  // namespace trb
