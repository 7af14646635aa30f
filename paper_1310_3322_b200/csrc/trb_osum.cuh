// trb_osum.cuh — block-parallel, bit-exact reproduction of a SEQUENTIAL
// fp64 summation  S_j = fl(S_{j-1} + a_j), S_{-1} = +0, a_j >= 0.
//
// Why: the reference tracker accumulates its Epanechnikov histogram
// (tracking.hpp:86-98) and its mean-shift centroid (tracking.hpp:135-146) as
// plain sequential double sums in raster order; the track log is printed
// with %.17g, so a tree reduction (different rounding) would break parity.
//
// Idea: while the running sum S stays inside one binade [2^e, 2^(e+1)) it is
// a multiple of u = 2^(e-52), and  fl(S + a) = S + RN_u(a)  exactly, where
// RN_u rounds a to the nearest multiple of u — independent of S — unless
// a sits exactly half-way between two multiples (a tie, resolved by S's
// parity) or S + a leaves the binade.  So every "safe" step contributes an
// exact integer r = RN_u(a)/u, and runs of safe steps are summed with exact
// int64 arithmetic in parallel.  The remaining "breakpoint" steps (binade
// crossings, ties, the first element) are replayed serially with real IEEE
// additions.  Which binade each step sees is predicted from an approximate
// parallel prefix P (error <= delta relative); a step whose interval
// [P_prev(1-delta), P_next(1+delta)] is not inside one binade is made a
// breakpoint, and the serial replay re-checks every prediction, falling back
// to a full serial sum (exact by construction) if one ever fails.
//
// Shape: one CTA of NT threads, thread t owns the contiguous element chunk
// [t*C, (t+1)*C).  M concurrent sums; an element may feed several sums
// (`emit(m, v)` calls, in the reference's per-element order).
//   phase A  chunk totals (approximate)   -> block exclusive scan  -> P at chunk starts
//   phase B  classify steps: safe -> exact int64 pieces, else breakpoint record
//   phase C  block segmented scan of pieces (reset at breakpoints)
//   phase D  per sum, breakpoints ranked by element index, then one thread
//            per sum replays: S += R*u (exact), S = fl(S + a_bp)
#pragma once

#include <limits.h>

#include "trb_exact.cuh"

namespace trb {

constexpr int kOsumThreads = 256;
constexpr int kOsumBpCap = 256;  // breakpoints per sum (~ binades crossed)
constexpr int kEmptyE = INT_MIN;

struct OsumBp {
  long long R;  // safe increments before this step (units 2^(e-52)), after fix-up
  double v;     // the element value
  int j;        // element index
  int e;        // binade of the piece before this step
  int t;        // owning thread
  int first;    // first breakpoint of this sum in thread t's chunk
};

// Shared-memory workspace for M sums at NT threads: 21*M*NT + 40*M bytes.
struct OsumSmem {
  double* run;      // [M][NT]
  long long* R;     // [M][NT]
  int* e;           // [M][NT]
  unsigned char* f; // [M][NT]  has-breakpoint flag
  double* result;   // [M]
  long long* finR;  // [M]
  int* fine;        // [M]
  int* nbp;         // [M]
  int* bad;         // [M]
  static __host__ __device__ size_t bytes(int M, int NT) {
    return static_cast<size_t>(M) * NT * (8 + 8 + 4 + 1) + static_cast<size_t>(M) * (8 + 8 + 4 + 4 + 4) + 64;
  }
  __device__ void carve(void* base, int M, int NT) {
    char* p = static_cast<char*>(base);
    run = reinterpret_cast<double*>(p);
    p += sizeof(double) * M * NT;
    R = reinterpret_cast<long long*>(p);
    p += sizeof(long long) * M * NT;
    result = reinterpret_cast<double*>(p);
    p += sizeof(double) * M;
    finR = reinterpret_cast<long long*>(p);
    p += sizeof(long long) * M;
    e = reinterpret_cast<int*>(p);
    p += sizeof(int) * M * NT;
    fine = reinterpret_cast<int*>(p);
    p += sizeof(int) * M;
    nbp = reinterpret_cast<int*>(p);
    p += sizeof(int) * M;
    bad = reinterpret_cast<int*>(p);
    p += sizeof(int) * M;
    f = reinterpret_cast<unsigned char*>(p);
  }
};

__device__ __forceinline__ int osum_exp(double x) {  // binade of a positive normal double, else kEmptyE
  const long long b = __double_as_longlong(x);
  const int be = static_cast<int>((b >> 52) & 0x7ff);
  return (be == 0 || be == 0x7ff || b < 0) ? kEmptyE : be - 1023;
}

// merge two piece exponents (kEmptyE = piece without safe steps); returns
// false when two non-empty pieces of one segment disagree on the binade
__device__ __forceinline__ bool osum_merge_e(int a_e, int b_e, int* out) {
  if (a_e == kEmptyE) {
    *out = b_e;
    return true;
  }
  *out = a_e;
  return b_e == kEmptyE || a_e == b_e;
}

// Exclusive scan of run[m][*] (doubles) for every m; warp w scans sums
// m = w, w + nwarps, ...  Each lane first reduces NT/32 consecutive entries.
__device__ __forceinline__ void osum_scan_run(OsumSmem& s, int M, int NT) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = NT >> 5;
  const int per = NT >> 5;
  for (int m = wid; m < M; m += nw) {
    double* row = s.run + static_cast<size_t>(m) * NT;
    double acc = 0.0;
    for (int i = 0; i < per; ++i) acc = xadd(acc, row[lane * per + i]);
    double incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = xadd(incl, y);
    }
    double run = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) run = 0.0;
    for (int i = 0; i < per; ++i) {
      const double v = row[lane * per + i];
      row[lane * per + i] = run;
      run = xadd(run, v);
    }
  }
}

// Segmented exclusive scan of the per-thread tail pieces (f, e, R) of every
// sum; afterwards e/R[m][t] hold the piece accumulated since the last
// breakpoint before thread t, and finR/fine[m] the final piece.
__device__ __forceinline__ void osum_scan_pieces(OsumSmem& s, int M, int NT) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = NT >> 5;
  const int per = NT >> 5;
  for (int m = wid; m < M; m += nw) {
    long long* Rr = s.R + static_cast<size_t>(m) * NT;
    int* er = s.e + static_cast<size_t>(m) * NT;
    unsigned char* fr = s.f + static_cast<size_t>(m) * NT;
    // lane aggregate over its run of threads
    int af = 0, ae = kEmptyE;
    long long aR = 0;
    bool ok = true;
    for (int i = 0; i < per; ++i) {
      const int t = lane * per + i;
      if (fr[t]) {
        af = 1, ae = er[t], aR = Rr[t];
      } else {
        int me;
        ok &= osum_merge_e(ae, er[t], &me);
        ae = me, aR += Rr[t];
      }
    }
    // warp inclusive scan of the lane aggregates with the segmented operator
    int sf = af, se = ae;
    long long sR = aR;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int pf = __shfl_up_sync(0xffffffffu, sf, o);
      const int pe = __shfl_up_sync(0xffffffffu, se, o);
      const long long pR = __shfl_up_sync(0xffffffffu, sR, o);
      if (lane >= o && !sf) {
        int me;
        ok &= osum_merge_e(pe, se, &me);
        sf = pf, se = me, sR += pR;
      }
    }
    // exclusive prefix for this lane
    int xf = __shfl_up_sync(0xffffffffu, sf, 1), xe = __shfl_up_sync(0xffffffffu, se, 1);
    long long xR = __shfl_up_sync(0xffffffffu, sR, 1);
    if (lane == 0) xf = 0, xe = kEmptyE, xR = 0;
    if (lane == 31) s.finR[m] = sR, s.fine[m] = se;
    for (int i = 0; i < per; ++i) {
      const int t = lane * per + i;
      const int tf = fr[t], te = er[t];
      const long long tR = Rr[t];
      er[t] = xe, Rr[t] = xR;  // exclusive value for thread t
      if (tf) {
        xf = 1, xe = te, xR = tR;
      } else {
        int me;
        ok &= osum_merge_e(xe, te, &me);
        xe = me, xR += tR;
      }
    }
    (void)xf;
    if (!ok) s.bad[m] = 1;
  }
}

// The engine.  `contrib(j, emit)` calls emit(m, v) for every sum element j
// feeds, with v >= 0.  bp: global scratch of M*kOsumBpCap records.
// Results land in s.result[m].  Must be called by all NT threads.
// stats (optional, global): [0] calls, [1] sums, [2] sums replayed by the
// serial fallback, [3] breakpoints, [4] elements
template <class Contrib>
__device__ void ordered_sums(int N, int M, const Contrib& contrib, OsumSmem& s, OsumBp* bp,
                             unsigned long long* stats = nullptr) {
  const int NT = blockDim.x, t = threadIdx.x;
  const int C = (N + NT - 1) / NT;
  const int j0 = min(N, t * C), j1 = min(N, j0 + C);
  // error of P relative to the true sequential sum: <= (N + 2C + 64) ulp-ish
  const double delta = static_cast<double>(N + 2 * C + 64) * 2.220446049250313e-16;
  const double lo_f = 1.0 - delta, hi_f = 1.0 + delta;

  for (int m = t; m < M; m += NT) s.nbp[m] = 0, s.bad[m] = 0;
  for (int m = 0; m < M; ++m) {
    s.run[m * NT + t] = 0.0;
    s.R[m * NT + t] = 0;
    s.e[m * NT + t] = kEmptyE;
    s.f[m * NT + t] = 0;
  }
  // ---- phase A: approximate chunk totals
  for (int j = j0; j < j1; ++j)
    contrib(j, [&](int m, double v) { s.run[m * NT + t] = xadd(s.run[m * NT + t], v); });
  __syncthreads();
  osum_scan_run(s, M, NT);
  __syncthreads();
  // ---- phase B: classify every step
  for (int j = j0; j < j1; ++j) {
    contrib(j, [&](int m, double v) {
      if (v == 0.0) return;  // fl(S + 0) == S: no effect on the sequence
      const int k = m * NT + t;
      const double P = s.run[k];
      const double Pn = xadd(P, v);
      s.run[k] = Pn;
      bool safe = false;
      long long r = 0;
      int e = kEmptyE;
      if (P > 0.0) {
        e = osum_exp(P);
        if (e != kEmptyE && e > -1000 && e < 1000 && osum_exp(xmul(P, lo_f)) == e && osum_exp(xmul(Pn, hi_f)) == e) {
          const double q = scalbn(v, 52 - e);  // exact power-of-two scaling
          const double fl = floor(q);
          const double fr = q - fl;  // exact
          if (fr != 0.5) {
            safe = true;
            r = static_cast<long long>(fl) + (fr > 0.5 ? 1 : 0);
          }
        }
      }
      if (safe) {
        int me;
        if (!osum_merge_e(s.e[k], e, &me)) s.bad[m] = 1;
        s.e[k] = me;
        s.R[k] += r;
      } else {
        const int idx = atomicAdd(&s.nbp[m], 1);
        if (idx < kOsumBpCap) {
          OsumBp& b = bp[m * kOsumBpCap + idx];
          b.R = s.R[k];
          b.e = s.e[k];
          b.v = v;
          b.j = j;
          b.t = t;
          b.first = !s.f[k];
        } else {
          s.bad[m] = 1;
        }
        s.f[k] = 1;
        s.R[k] = 0;
        s.e[k] = kEmptyE;
      }
    });
  }
  __syncthreads();
  // ---- phase C: segmented scan of pieces
  osum_scan_pieces(s, M, NT);
  __syncthreads();
  // fold the carried-in piece into each thread's first breakpoint
  for (int m = 0; m < M; ++m) {
    const int n = min(s.nbp[m], kOsumBpCap);
    for (int i = t; i < n; i += NT) {
      OsumBp& b = bp[m * kOsumBpCap + i];
      if (!b.first) continue;
      const int k = m * NT + b.t;
      int me;
      if (!osum_merge_e(s.e[k], b.e, &me)) s.bad[m] = 1;
      b.e = me;
      b.R += s.R[k];
    }
  }
  __syncthreads();
  // ---- phase D: rank breakpoints by element index (stable: j is unique per sum)
  //      rank stored in .t (no longer needed)
  for (int m = 0; m < M; ++m) {
    const int n = min(s.nbp[m], kOsumBpCap);
    for (int i = t; i < n; i += NT) {
      const int ji = bp[m * kOsumBpCap + i].j;
      int rank = 0;
      for (int q = 0; q < n; ++q) rank += bp[m * kOsumBpCap + q].j < ji;
      bp[m * kOsumBpCap + i].t = rank;
    }
  }
  __syncthreads();
  // serial replay, one thread per sum
  for (int m = t; m < M; m += NT) {
    double S = 0.0;
    bool ok = !s.bad[m];
    const int n = min(s.nbp[m], kOsumBpCap);
    // walk breakpoints in rank order; ranks are a permutation of 0..n-1
    for (int rk = 0; rk < n && ok; ++rk) {
      const OsumBp* b = nullptr;
      for (int q = 0; q < n; ++q)
        if (bp[m * kOsumBpCap + q].t == rk) {
          b = &bp[m * kOsumBpCap + q];
          break;
        }
      if (b->e != kEmptyE) {  // a run of safe steps predicted in binade e: verify, then add exactly
        if (osum_exp(S) != b->e) {
          ok = false;
          break;
        }
        const double S2 = xadd(S, scalbn(static_cast<double>(b->R), b->e - 52));
        if (osum_exp(S2) != b->e) {
          ok = false;
          break;
        }
        S = S2;
      }
      S = xadd(S, b->v);
    }
    if (ok && s.fine[m] != kEmptyE) {
      if (osum_exp(S) != s.fine[m]) {
        ok = false;
      } else {
        const double S2 = xadd(S, scalbn(static_cast<double>(s.finR[m]), s.fine[m] - 52));
        if (osum_exp(S2) != s.fine[m]) ok = false;
        else S = S2;
      }
    }
    s.result[m] = S;
    s.bad[m] = ok ? 0 : 1;
  }
  __syncthreads();
  if (stats && t == 0) {
    unsigned long long nb = 0, nbad = 0;
    for (int m = 0; m < M; ++m) nb += s.nbp[m], nbad += s.bad[m];
    atomicAdd(&stats[0], 1ull);
    atomicAdd(&stats[1], static_cast<unsigned long long>(M));
    atomicAdd(&stats[2], nbad);
    atomicAdd(&stats[3], nb);
    atomicAdd(&stats[4], static_cast<unsigned long long>(N));
  }
  // exact serial fallback for any sum whose prediction failed
  for (int m = 0; m < M; ++m) {
    if (!s.bad[m]) continue;  // uniform across the block
    if (t == 0) {
      double S = 0.0;
      for (int j = 0; j < N; ++j)
        contrib(j, [&](int mm, double v) {
          if (mm == m) S = xadd(S, v);
        });
      s.result[m] = S;
    }
  }
  __syncthreads();
}

}  // namespace trb
