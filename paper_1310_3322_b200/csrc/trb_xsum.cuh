// trb_xsum.cuh — chunk-classified, bit-exact reproduction of SEQUENTIAL fp64
// sums S_j = fl(S_{j-1} + a_j), S_{-1} = +0, a_j >= 0 (the tracker's
// histogram and centroid sums, tracking.hpp:86-98 and :135-146).
//
// Same arithmetic fact as trb_osum.cuh: while S stays in one binade
// [2^e, 2^(e+1)) it is X*u (u = 2^(e-52), X an integer) and a step that keeps
// it there is X -> X + RN(a/u), an integer that depends on a alone unless
// a/u is exactly k + 1/2 (a tie: round-half-even on X).  The sum of a run of
// such steps is therefore an integer sum, which can be formed in any order.
//
// What this engine does differently (fewer instructions per element, fewer
// barriers per sum):
//  * Whole chunks are classified, not elements.  Every thread owns a
//    contiguous chunk of elements.  One pass forms approximate chunk totals,
//    a CTA/cluster scan gives every chunk its approximate start prefix P0 and
//    end prefix P1 (relative error <= delta).  If [P0(1-delta), P1(1+delta)]
//    lies inside one binade, every step of the chunk is a plain integer step
//    of that binade: the walk is y = fl(2^e + a), r = bits(y) - bits(2^e),
//    B += r, plus a tie test.  Only chunks that straddle a binade boundary
//    ("general" chunks, ~log2(range) per sum) classify element by element.
//  * Many lanes per run, dense or selected: the histogram runs K+1 sums at
//    once (the total, and one per bin: an element feeds the total and the
//    lane of its bin) straight from raster order — no stable partition by
//    bin, no scratch in HBM.  A thread keeps up to kQ bin lanes in registers
//    per pass over its chunk (a chunk rarely holds more than 2-3 bins).
//  * Breakpoints are the only serial work: the first element of a sum
//    ("head": the owning thread sums its elements of that lane with real
//    IEEE adds from +0 — exact), steps of general chunks that cannot be
//    classified, and ties.  Each record carries the lane's integer prefix;
//    a replay per lane walks the records in element order with
//    S <- S + (ip_k - ip_{k-1}) * u  (integer add on the significand) then
//    S <- fl(S + a_k), and finally adds the tail.
//  * Two cluster barriers per run (after the approximate scan; after the
//    records are ranked), every CTA replays the gathered records itself.
// Any failed check (record overflow, an integer run leaving its binade) falls
// back to a serial sum per lane, exact by construction (debug stats count
// it; never observed).
#pragma once

#include "trb_osum.cuh"

#ifndef TRB_XS_MARK
#define TRB_XS_MARK(k) ((void)0)
#endif

namespace trb {
namespace xs {

constexpr int kQ = 3;         // selected lanes held in registers per pass
constexpr int kMaxL = 20;     // lanes per run (NF + K): K <= 16 bins + total
constexpr int kRecCta = 768;   // breakpoint records per CTA per run (a single-CTA group holds them all)
constexpr long long kMant = (1LL << 52) - 1;
// lean loop for all-safe chunks (measured slower: register pressure, warp
// divergence against the young-sum warps; kept for experiments)
#ifndef TRB_XS_FAST
#define TRB_XS_FAST 0
#endif
constexpr bool kFastWalk = TRB_XS_FAST != 0;

enum { kNone = 0, kSafe = 1, kGeneral = 2, kHead = 3 };
enum { kRecStep = 0, kRecHead = 1, kRecTie = 2 };

struct Rec {
  double v;       // step: the element value; head: the exact head sum; tie piece: the bits of A
  long long ip;   // lane integer prefix at the record (thread-local, then CTA, then cluster)
  long long b;    // tie piece: B
  int key;        // 4*j + sub: the order of a lane's records (sub 0 piece flush, 1 step, 2 chunk-end flush)
  uint8_t lane;
  uint8_t kind;
  uint16_t lrank; // rank among this CTA's records of the lane
};
static_assert(sizeof(Rec) == 32, "Rec layout");
// a gathered record (cluster order), placed in the free scan buffer
struct Rec2 {
  double v;
  long long ip, b;
  int kind, pad;
};
static_assert(sizeof(Rec2) == 32, "Rec2 layout");

// Static shared memory of the engine (the per-thread x per-lane scan buffers
// are dynamic).
struct Shared {
  double cta_tot[kMaxL];        // phase A: this CTA's approximate lane totals (read remotely)
  long long cta_ip[kMaxL];      // phase C: this CTA's lane integer totals (read remotely)
  int cta_cnt[kMaxL];           // phase C: records per lane in this CTA (read remotely)
  int cta_flag;                 // failure bits of this CTA (read remotely)
  int nrec;
  double carry[kMaxL];          // approximate prefix of the lower CTAs, per lane
  double gtot[kMaxCluster][kMaxL];
  long long gip[kMaxCluster][kMaxL];
  int gcnt[kMaxCluster][kMaxL];
  int gflag[kMaxCluster];
  unsigned wmask[32];           // phase A: lanes present per warp
  int gbase[kMaxCluster][kMaxL];   // phase C pull: destination base per (source CTA, lane)
  long long gipc[kMaxCluster][kMaxL];  // integer prefix of the lower CTAs per (source CTA, lane)
  int goff[kMaxCluster + 1];       // record offsets per source CTA
  int lane_base[kMaxL + 1];
  double res[kMaxL];
  int fail;
  Rec rec[kRecCta];
};

struct LaneSt {
  long long B;       // integer steps since the chunk start, outside tie pieces (units of the binade at the time)
  long long pA, pB;  // the open tie piece X -> E(X + pA) + pB (pt = 1)
  double M;          // 2^e of the binade the integer steps use
  double hi;         // general: arm bound (largest prefix still safe in binade e), -1 disarmed
  double P;          // general: running approximate prefix; head: exact running sum
  int mode;
  int bin;           // selected lanes: the bin (-1 = empty slot)
  int pt;            // a tie piece is open
};

struct Ctx {
  Shared* s;
  long long lowm, highm, highm_end;  // highm_end: upper margin for the chunk-end prefix (float chunk totals)
  int t;
};

__device__ __forceinline__ double pow2(int eb) {  // eb = biased exponent
  return __longlong_as_double(static_cast<long long>(eb) << 52);
}
__device__ __forceinline__ long long up_even(long long y) { return y + (y & 1); }

__device__ __forceinline__ void emit(const Ctx& c, int lane, int kind, double v, long long ip, long long b, int key) {
  const int idx = atomicAdd(&c.s->nrec, 1);
  if (idx < kRecCta) {
    Rec& r = c.s->rec[idx];
    r.v = v, r.ip = ip, r.b = b, r.key = key, r.lane = static_cast<uint8_t>(lane), r.kind = static_cast<uint8_t>(kind);
    r.lrank = 0;
  } else {
    c.s->fail = 1;  // overflow: every CTA learns it through cta_flag
  }
}

// A step of binade M = 2^e that stays in the binade: X -> X + RN(a/u), or on
// a tie (a/u = k + 1/2) X -> E(X + k), E = round up to even.  Plain steps add
// to B; from the first tie on, the steps compose into a tie piece
// (E(X + A) + B composed with +r or with tie(k) keeps that form, because
// E(X + A) is even: E(E(X + A) + y) = E(X + A) + E(y)) — one record per
// piece instead of one per tie (a lane summing one repeated value can tie on
// every element of a binade).
__device__ __forceinline__ void int_step(LaneSt& L, double a) {
  const double y = xadd(L.M, a);
  const double d = xsub(a, xsub(y, L.M));
  const double hu = __longlong_as_double(__double_as_longlong(L.M) - (53LL << 52));  // u/2
  const long long r = __double_as_longlong(y) - __double_as_longlong(L.M);
  if (fabs(d) == hu) {
    const long long k = d > 0.0 ? r : r - 1;
    if (!L.pt) L.pt = 1, L.pA = k, L.pB = 0;
    else L.pB = up_even(L.pB + k);
  } else if (L.pt) {
    L.pB += r;
  } else {
    L.B += r;
  }
}

__device__ __forceinline__ void flush_piece(LaneSt& L, int lane, int key, const Ctx& c) {
  if (!L.pt) return;
  emit(c, lane, kRecTie, __longlong_as_double(L.pA), L.B, L.pB, key);
  L.pt = 0;
}

// Chunk classification from its approximate start / end prefixes.
__device__ __forceinline__ void classify(LaneSt& L, bool present, double p0, double p1, const Ctx& c) {
  L.B = 0, L.hi = -1.0, L.M = 1.0, L.P = 0.0, L.pt = 0, L.pA = 0, L.pB = 0;
  if (!present) {
    L.mode = kNone;
    return;
  }
  if (p0 == 0.0) {  // no earlier element: the exact state is +0 — sum the chunk with IEEE adds
    L.mode = kHead;
    return;
  }
  const long long b0 = __double_as_longlong(p0), b1 = __double_as_longlong(p1);
  const int e0 = static_cast<int>(b0 >> 52);
  if (p0 > 0.0 && e0 == static_cast<int>(b1 >> 52) && e0 > 64 && e0 < 1982 && (b0 & kMant) >= c.lowm &&
      (b1 & kMant) <= c.highm_end) {
    L.mode = kSafe;
    L.M = pow2(e0);
    return;
  }
  L.mode = kGeneral;
  L.P = p0;
  if (p0 > 0.0 && e0 > 64 && e0 < 1982 && (b0 & kMant) >= c.lowm) {  // pre-armed from the start prefix
    L.hi = __longlong_as_double((static_cast<long long>(e0) << 52) | c.highm);
    L.M = pow2(e0);
  }
}

// One element of a general chunk (per-element classification, as trb_osum).
__device__ __forceinline__ void general_step(LaneSt& L, double a, int j, int lane, const Ctx& c) {
  const double Pp = L.P, Pn = xadd(Pp, a);
  L.P = Pn;
  if (Pn <= L.hi) {
    int_step(L, a);
    return;
  }
  if (a == 0.0) return;  // a zero step never changes S
  const long long bp = __double_as_longlong(Pp), bn = __double_as_longlong(Pn);
  const int eb = static_cast<int>(bp >> 52);
  if (Pp > 0.0 && eb == static_cast<int>(bn >> 52) && eb > 64 && eb < 1982 && (bp & kMant) >= c.lowm &&
      (bn & kMant) <= c.highm) {
    if (L.pt && pow2(eb) != L.M) flush_piece(L, lane, 4 * j, c);  // a piece never spans two binades
    L.hi = __longlong_as_double((static_cast<long long>(eb) << 52) | c.highm);
    L.M = pow2(eb);
    int_step(L, a);
    return;
  }
  flush_piece(L, lane, 4 * j, c);
  emit(c, lane, kRecStep, a, L.B, 0, 4 * j + 1);
  L.hi = -1.0;
  const int en = static_cast<int>(bn >> 52);
  if (Pn > 0.0 && en > 64 && en < 1982 && (bn & kMant) >= c.lowm) {  // re-arm from the replayed step's prefix
    L.hi = __longlong_as_double((static_cast<long long>(en) << 52) | c.highm);
    L.M = pow2(en);
  }
}

__device__ __forceinline__ void step(LaneSt& L, double a, int j, int lane, const Ctx& c) {
  if (L.mode == kSafe) {
    int_step(L, a);
  } else if (L.mode == kHead) {
    L.P = xadd(L.P, a);
  } else if (L.mode == kGeneral) {
    general_step(L, a, j, lane, c);
  }
}

// end of a lane's pass over the chunk: close a tie piece, emit a head's sum
__device__ __forceinline__ void finish_lane(LaneSt& L, int lane, int j0, int j1, const Ctx& c) {
  if (L.mode == kHead) emit(c, lane, kRecHead, L.P, 0, 0, 4 * j0);
  flush_piece(L, lane, 4 * (j1 - 1) + 2, c);
}

__device__ __forceinline__ void swap_lane(LaneSt& a, LaneSt& b) {
  const LaneSt t = a;
  a = b;
  b = t;
}

// In-place exclusive scan over the CTA's threads of buf[l * NT + t] for
// l < L (per warp: shuffle scan of its 32 threads; then warp offsets).
// tot[l] receives the CTA total.  T = double (approximate prefixes) or
// long long (integer prefixes, exact).
template <typename T>
__device__ void cta_exscan(T* buf, int L, unsigned lmask, T* tot, T* wsum /* [L][32] scratch */) {
  // only the lanes present in this CTA (lmask): every other lane's entries
  // are 0 already and stay so, its CTA total is 0
  const int NT = blockDim.x, t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  for (int l = t; l < L; l += NT)
    if (!((lmask >> l) & 1u)) tot[l] = T(0);
  for (unsigned m = lmask; m; m &= m - 1) {
    const int l = __ffs(m) - 1;
    const T v = buf[l * NT + t];
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    buf[l * NT + t] = incl - v;  // exclusive within the warp (exact for integers; for doubles
                                 // the difference only needs the approximate prefix bound,
                                 // and it is exactly 0 when every earlier value is 0)
    if (lane == 31) wsum[l * 32 + wid] = incl;
  }
  __syncthreads();
  int idx = 0;
  for (unsigned m = lmask; m; m &= m - 1, ++idx) {  // warp offsets: the idx-th present lane on warp idx % nw
    if (idx % nw != wid) continue;
    const int l = __ffs(m) - 1;
    const T v = lane < nw ? wsum[l * 32 + lane] : T(0);
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < nw) wsum[l * 32 + lane] = incl - v;
    if (lane == 31) tot[l] = incl;
  }
  __syncthreads();
  for (unsigned m = lmask; m; m &= m - 1) {
    const int l = __ffs(m) - 1;
    buf[l * NT + t] += wsum[l * 32 + wid];
  }
  __syncthreads();
}

// S (exact, a positive normal double) advanced by n integer steps of its own
// binade; ok cleared when the significand leaves [2^52, 2^53).
__device__ __forceinline__ double add_units(double S, long long n, bool& ok) {
  if (n == 0) return S;
  const long long b = __double_as_longlong(S);
  const long long e = b >> 52;
  ok &= S > 0.0 && e > 0 && e < 2047 && n > 0;
  const long long X = (b & kMant) | (1LL << 52);
  const long long X2 = X + n;
  ok &= X2 >= (1LL << 52) && X2 < (1LL << 53);
  return __longlong_as_double((e << 52) | (X2 & kMant));
}

// S (exact, positive normal) through a tie piece of its own binade:
// X -> E(X + A) + B.
__device__ __forceinline__ double apply_tie(double S, long long A, long long B, bool& ok) {
  const long long b = __double_as_longlong(S);
  const long long e = b >> 52;
  ok &= S > 0.0 && e > 0 && e < 2047;
  const long long X = (b & kMant) | (1LL << 52);
  const long long X2 = up_even(X + A) + B;
  ok &= X2 >= (1LL << 52) && X2 < (1LL << 53);
  return __longlong_as_double((e << 52) | (X2 & kMant));
}

// One run.  Src supplies the elements of thread chunk [j0, j1):
//   typename Src::Cursor cur = src.begin(j0);  cur.next(has, sel, v)  (v[NF]);
//   cur.finish() after the last element of phase A
//   src.get(j, has, sel, v)  (random access, serial fallback only)
// srcA feeds phase A (and the fallback), srcB phase B (e.g. srcA computes
// each element's bin and stages it, srcB reads the staged words).
// Lanes: 0..NF-1 fixed (every element with `has` feeds lane l with v[l]);
// if SEL, NF + b for bins b < K (an element feeds lane NF + sel with v[0]).
// buf: dynamic shared scratch of L * blockDim.x 8-byte words, ftot: L *
// blockDim.x floats, wsum: L * 32 8-byte words.
// Results: s.res[l], identical in every CTA of the group, on return.
// all_cap: Rec2 records that fit in buf (its full allocation, which may
// exceed this run's L * blockDim.x words).
template <int NF, bool SEL, class SrcA, class SrcB>
__device__ void xsum_run(const Grp& cl, int N, int K, const SrcA& src, const SrcB& srcB, Shared& s, double* buf,
                         float* ftot, double* wsumd, int all_cap, unsigned long long* stats) {
  const int NT = blockDim.x, t = threadIdx.x;
  const int rank = static_cast<int>(cl.block_rank()), G = static_cast<int>(cl.num_blocks());
  const int GT = G * NT, gt = rank * NT + t;
  const int L = NF + (SEL ? K : 0);
  const int C = ((N + GT - 1) / GT + 3) & ~3;  // a multiple of 4: whole staged 4-element words per thread
  const int j0 = min(N, gt * C), j1 = min(N, j0 + C);
  // relative error of every approximate prefix vs the exact sequential sum:
  // the sequential sum's own drift (N roundings) + the scan's (chunk, warp,
  // CTA, cluster levels) — delta = D * 2^-52 with a factor-2 margin below
  const long long D = 2LL * N + 4LL * C + 256 + 2LL * G;
  Ctx c;
  c.s = &s, c.t = t;
  c.lowm = 2 * D + 4;
  c.highm = kMant - 2 * c.lowm;
  // chunk end = start + the chunk total rounded to float (relative error 2^-24 of the end)
  c.highm_end = c.highm - (1LL << 30);
  // (s.nrec / s.fail are reset after the first cluster barrier: other CTAs may
  // still be pulling this CTA's records of the previous run until then)

  // ---------------- phase A: approximate chunk totals per lane
  for (int l = 0; l < L; ++l) buf[l * NT + t] = 0.0;
  unsigned mask = 0;  // selected lanes present in the chunk
  bool anyf = false;
  {
    double aF[NF];
#pragma unroll
    for (int l = 0; l < NF; ++l) aF[l] = 0.0;
    int cur = -1;
    double acc = 0.0;
    auto cu = src.begin(j0);
    for (int j = j0; j < j1; ++j) {
      bool has;
      int sel;
      double v[NF];
      cu.next(has, sel, v);
      if (!has) continue;
      anyf = true;
#pragma unroll
      for (int l = 0; l < NF; ++l) aF[l] = xadd(aF[l], v[l]);
      if (SEL) {
        if (sel != cur) {
          if (cur >= 0) buf[(NF + cur) * NT + t] += acc;
          cur = sel, acc = 0.0;
          mask |= 1u << sel;
        }
        acc = xadd(acc, v[0]);
      }
    }
    cu.finish();
    if (SEL && cur >= 0) buf[(NF + cur) * NT + t] += acc;
#pragma unroll
    for (int l = 0; l < NF; ++l) buf[l * NT + t] = aF[l];
  }
  TRB_XS_MARK(0);
  // own chunk totals (float: only the chunk-end prefix needs them, with the
  // widened upper margin highm_end)
  for (int l = 0; l < L; ++l) ftot[l * NT + t] = static_cast<float>(buf[l * NT + t]);
  // lanes present in this CTA (fixed lanes: any element; selected: its bin)
  const unsigned tmask = (mask << NF) | (anyf ? ((1u << NF) - 1u) : 0u);
  {
    const unsigned wm = __reduce_or_sync(0xffffffffu, tmask);
    if ((t & 31) == 0) s.wmask[t >> 5] = wm;
  }
  __syncthreads();
  unsigned lmask = 0;
  for (int w = 0; w < (NT >> 5); ++w) lmask |= s.wmask[w];
  cta_exscan<double>(buf, L, lmask, s.cta_tot, wsumd);
  cl.sync();  // every CTA's totals are visible; every CTA finished the previous run's pulls
  if (t == 0) s.nrec = 0, s.fail = 0;
  for (int i = t; i < G * L; i += NT) {
    const int r = i / L, l = i - r * L;
    s.gtot[r][l] = (r == rank) ? s.cta_tot[l] : *cl.map_shared_rank(&s.cta_tot[l], r);
  }
  __syncthreads();
  for (int l = t; l < L; l += NT) {
    double cr = 0.0;
    for (int r = 0; r < rank; ++r) cr = xadd(cr, s.gtot[r][l]);
    s.carry[l] = cr;
  }
  __syncthreads();
  TRB_XS_MARK(1);
  // start / end prefix of this thread's chunk for lane l (own entries only:
  // the integer totals overwrite them lane by lane during phase B)
  auto p0 = [&](int l) { return xadd(s.carry[l], buf[l * NT + t]); };
  auto p1 = [&](int l) { return xadd(p0(l), static_cast<double>(ftot[l * NT + t])); };

  // ---------------- phase B: integer steps, records
  LaneSt F[NF];
#pragma unroll
  for (int l = 0; l < NF; ++l) classify(F[l], anyf, p0(l), p1(l), c), F[l].bin = l;
  // the scan buffer entries of this thread are read at lane setup only; the
  // lane's integer total overwrites them at the end of its pass, absent
  // lanes get 0 now (own column only: no other thread reads it)
  for (int l = 0; l < L; ++l) {
    const bool present = l < NF ? anyf : ((mask >> (l - NF)) & 1u) != 0;
    if (!present) reinterpret_cast<long long*>(buf)[l * NT + t] = 0;
  }
  unsigned rem = mask;
  bool first = true;
  for (;;) {
    LaneSt Q[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      if (SEL && rem) {
        const int b = __ffs(rem) - 1;
        rem &= rem - 1;
        classify(Q[q], true, p0(NF + b), p1(NF + b), c);
        Q[q].bin = b;
      } else {
        Q[q].mode = kNone, Q[q].bin = -1, Q[q].B = 0, Q[q].P = 0.0, Q[q].hi = -1.0, Q[q].M = 1.0;
      }
    }
    if (!first && Q[0].bin < 0) break;
    auto cu = srcB.begin(j0);
    int j = j0;
    // common case: every lane of this pass is a safe chunk (no open piece):
    // a lean loop of integer steps; the first tie (or anything else) hands
    // the element and the rest of the chunk to the general loop below
    bool fast = kFastWalk;
    if (first)
#pragma unroll
      for (int l = 0; l < NF; ++l) fast &= F[l].mode == kSafe || F[l].mode == kNone;
#pragma unroll
    for (int q = 0; q < kQ; ++q) fast &= Q[q].mode == kSafe || Q[q].bin < 0;
    if (fast) {
      long long BF[NF], BQ[kQ];
#pragma unroll
      for (int l = 0; l < NF; ++l) BF[l] = 0;
#pragma unroll
      for (int q = 0; q < kQ; ++q) BQ[q] = 0;
      bool bail = false;
      bool bh;
      int bsel;
      double bv[NF];
      for (; j < j1; ++j) {
        bool has;
        int sel;
        double v[NF];
        cu.next(has, sel, v);
        if (!has) continue;
        bool tie = false;
        long long rF[NF];
        if (first) {
#pragma unroll
          for (int l = 0; l < NF; ++l) {
            const double M = F[l].M;
            const double y = xadd(M, v[l]);
            const double d = xsub(v[l], xsub(y, M));
            tie |= fabs(d) == __longlong_as_double(__double_as_longlong(M) - (53LL << 52));
            rF[l] = F[l].mode == kSafe ? __double_as_longlong(y) - __double_as_longlong(M) : 0;
          }
        }
        long long rQ = 0;
        int qi = -1;
        if (SEL) {
#pragma unroll
          for (int q = 0; q < kQ; ++q)
            if (sel == Q[q].bin) qi = q;
          if (qi >= 0) {
            double M = Q[0].M;
#pragma unroll
            for (int q = 1; q < kQ; ++q)
              if (qi == q) M = Q[q].M;
            const double y = xadd(M, v[0]);
            const double d = xsub(v[0], xsub(y, M));
            tie |= fabs(d) == __longlong_as_double(__double_as_longlong(M) - (53LL << 52));
            rQ = __double_as_longlong(y) - __double_as_longlong(M);
          }
        }
        if (tie) {  // rare: this element and the rest of the chunk take the general path
          bail = true, bh = has, bsel = sel;
#pragma unroll
          for (int l = 0; l < NF; ++l) bv[l] = v[l];
          break;
        }
        if (first)
#pragma unroll
          for (int l = 0; l < NF; ++l) BF[l] += rF[l];
#pragma unroll
        for (int q = 0; q < kQ; ++q)
          if (qi == q) BQ[q] += rQ;
      }
      if (first)
#pragma unroll
        for (int l = 0; l < NF; ++l) F[l].B += BF[l];
#pragma unroll
      for (int q = 0; q < kQ; ++q) Q[q].B += BQ[q];
      if (bail) {  // the interrupted element through the general steps
        if (first) {
#pragma unroll
          for (int l = 0; l < NF; ++l) step(F[l], bv[l], j, l, c);
        }
        if (SEL)
#pragma unroll
          for (int q = 0; q < kQ; ++q)
            if (bsel == Q[q].bin) step(Q[q], bv[0], j, NF + bsel, c);
        (void)bh;
        ++j;
      }
    }
    for (; j < j1; ++j) {
      bool has;
      int sel;
      double v[NF];
      cu.next(has, sel, v);
      if (!has) continue;
      if (first) {
#pragma unroll
        for (int l = 0; l < NF; ++l) step(F[l], v[l], j, l, c);
      }
      if (SEL) {
        if (sel != Q[0].bin) {
#pragma unroll
          for (int q = 1; q < kQ; ++q)
            if (sel == Q[q].bin) swap_lane(Q[0], Q[q]);
        }
        if (sel == Q[0].bin) step(Q[0], v[0], j, NF + sel, c);
      }
    }
    if (first) {
#pragma unroll
      for (int l = 0; l < NF; ++l) {
        finish_lane(F[l], l, j0, j1, c);
        reinterpret_cast<long long*>(buf)[l * NT + t] = F[l].B;
      }
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      if (Q[q].bin < 0) continue;
      const int l = NF + Q[q].bin;
      finish_lane(Q[q], l, j0, j1, c);
      reinterpret_cast<long long*>(buf)[l * NT + t] = Q[q].B;
    }
    first = false;
    if (!SEL || !rem) break;
  }

  // ---------------- phase C: integer prefixes, ranked records, gather, replay
  TRB_XS_MARK(2);
  __syncthreads();
  long long* ibuf = reinterpret_cast<long long*>(buf);
  cta_exscan<long long>(ibuf, L, lmask, s.cta_ip, reinterpret_cast<long long*>(wsumd));
  const int nrec = min(s.nrec, kRecCta);
  for (int l = t; l < L; l += NT) s.cta_cnt[l] = 0;
  __syncthreads();
  for (int i = t; i < nrec; i += NT) {
    Rec& r = s.rec[i];
    // the record's owner thread: chunks are contiguous, owner = (j - CTA start) / C
    const int owner = min(NT - 1, max(0, (r.key >> 2) / max(1, C) - rank * NT));
    r.ip += ibuf[r.lane * NT + owner];
    int rk = 0;
    for (int q = 0; q < nrec; ++q) {
      const Rec& o = s.rec[q];
      rk += (o.lane == r.lane) & (o.key < r.key);
    }
    r.lrank = static_cast<uint16_t>(rk);
    atomicAdd(&s.cta_cnt[r.lane], 1);
    if (stats) atomicAdd(&stats[r.kind == 1 ? 26 : (r.lane < NF ? 24 : 25)], 1ull);
  }
  if (t == 0) s.cta_flag = s.fail | (s.nrec > kRecCta ? 1 : 0);
  __syncthreads();
  TRB_XS_MARK(3);
  cl.sync();  // ranked records, counts and integer totals of every CTA are visible
  TRB_XS_MARK(4);
  for (int i = t; i < G * L; i += NT) {
    const int r = i / L, l = i - r * L;
    const Shared* rs = (r == rank) ? &s : cl.map_shared_rank(&s, r);
    s.gip[r][l] = rs->cta_ip[l];
    s.gcnt[r][l] = rs->cta_cnt[l];
    if (l == 0) s.gflag[r] = rs->cta_flag;
  }
  __syncthreads();
  if (t == 0) {
    int base = 0, fl = 0;
    for (int l = 0; l < L; ++l) {
      s.lane_base[l] = base;
      for (int r = 0; r < G; ++r) base += s.gcnt[r][l];
    }
    s.lane_base[L] = base;
    for (int r = 0; r < G; ++r) fl |= s.gflag[r];
    s.fail = fl | (base > all_cap ? 2 : 0);
  }
  __syncthreads();
  const bool failed = s.fail != 0;
  // the gathered list goes into the scan buffer: free now (the integer
  // prefixes were folded into this CTA's records before the barrier, and no
  // other CTA reads it)
  Rec2* all = reinterpret_cast<Rec2*>(buf);
  if (!failed) {
    // pull every CTA's records into place: lane base + records of the lane in
    // lower CTAs + rank inside the source CTA; integer prefix + lower CTAs' totals
    // (one flattened pass over every CTA's records: the remote loads of all
    // CTAs are in flight together)
    for (int i = t; i < G * L; i += NT) {  // per (source CTA, lane): destination base, carried prefix
      const int r = i / L, l = i - r * L;
      int before = 0;
      long long ipc = 0;
      for (int q = 0; q < r; ++q) before += s.gcnt[q][l], ipc += s.gip[q][l];
      s.gbase[r][l] = s.lane_base[l] + before;
      s.gipc[r][l] = ipc;
    }
    if (t == 0) {
      int o = 0;
      for (int r = 0; r < G; ++r) {
        s.goff[r] = o;
        for (int l = 0; l < L; ++l) o += s.gcnt[r][l];
      }
      s.goff[G] = o;
    }
    __syncthreads();
    const int total = s.goff[G];
    for (int k = t; k < total; k += NT) {
      int r = 0;
      while (k >= s.goff[r + 1]) ++r;
      const Shared* rs = (r == rank) ? &s : cl.map_shared_rank(&s, r);
      const Rec rc = rs->rec[k - s.goff[r]];
      const int l = rc.lane;
      Rec2 g;
      g.v = rc.v, g.ip = rc.ip + s.gipc[r][l], g.b = rc.b, g.kind = rc.kind, g.pad = 0;
      all[s.gbase[r][l] + rc.lrank] = g;
    }
  }
  __syncthreads();
  TRB_XS_MARK(5);
  // replay, one thread per lane
  if (!failed) {
    for (int l = t; l < L; l += NT) {
      long long ip_end = 0;
      for (int r = 0; r < G; ++r) ip_end += s.gip[r][l];
      double S = 0.0;
      long long ipp = 0;
      bool ok = true;
      if (s.lane_base[l] == s.lane_base[l + 1] && ip_end == 0) {  // no element anywhere (or only zeros)
        s.res[l] = 0.0;
        continue;
      }
      for (int q = s.lane_base[l]; q < s.lane_base[l + 1]; ++q) {
        const Rec2 rc = all[q];
        S = add_units(S, rc.ip - ipp, ok);
        if (rc.kind == kRecHead) {  // the exact state is +0 before a head
          ok &= S == 0.0;
          S = rc.v;
        } else if (rc.kind == kRecTie) {
          S = apply_tie(S, __double_as_longlong(rc.v), rc.b, ok);
        } else {
          S = xadd(S, rc.v);
        }
        ipp = rc.ip;
      }
      S = add_units(S, ip_end - ipp, ok);
      s.res[l] = S;
      if (!ok) atomicOr(&s.fail, 4);
    }
  }
  __syncthreads();
  TRB_XS_MARK(6);
  if (stats && t == 0 && rank == 0) {
    atomicAdd(&stats[0], 1ull);
    atomicAdd(&stats[1], static_cast<unsigned long long>(L));
    atomicAdd(&stats[3], static_cast<unsigned long long>(s.lane_base[L]));
    atomicAdd(&stats[4], static_cast<unsigned long long>(N));
    if (s.fail) atomicAdd(&stats[2], 1ull);
    if (s.fail & 1) atomicAdd(&stats[18], 1ull);
    if (s.fail & 2) atomicAdd(&stats[19], 1ull);
    if (s.fail & 4) atomicAdd(&stats[22], 1ull);
    atomicMax(&stats[29], static_cast<unsigned long long>(s.lane_base[L]));
    unsigned long long mx = 0;
    for (int r = 0; r < G; ++r) {
      int n = 0;
      for (int l = 0; l < L; ++l) n += s.gcnt[r][l];
      mx = max(mx, static_cast<unsigned long long>(n));
    }
    atomicMax(&stats[28], mx);
  }
  if (s.fail) {  // exact serial fallback: one thread per lane over every element
    for (int l = t; l < L; l += NT) {
      double S = 0.0;
      for (int j = 0; j < N; ++j) {
        bool has;
        int sel;
        double v[NF];
        src.get(j, has, sel, v);
        if (!has) continue;
        if (l < NF) S = xadd(S, v[l]);
        else if (sel == l - NF) S = xadd(S, v[0]);
      }
      s.res[l] = S;
    }
    __syncthreads();
  }
}

}  // namespace xs
}  // namespace trb
