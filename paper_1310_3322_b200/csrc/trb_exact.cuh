// trb_exact.cuh — bit-exact replicas of the host math the reference tracker
// depends on, usable on host and device.
//
//  * glibc_hypot: std::hypot as shipped by glibc 2.39 on x86-64 (the
//    reference's libm).  Restated from the machine code of
//    libm.so.6:__hypot (non-FMA kernel, SSE2): constants 2^511 / 2^-459 /
//    2^-54 / 2^+-600 / 2^54 were read from its rodata.  Pinned against the
//    live libm by tests/test_host.py (random + adversarial inputs) and
//    on the device by tests/test_gpu_tracker.py and, on 1e8 samples,
//    tests/test_gpu_bench_parity.py.
//  * Mt64: std::mt19937_64 (n=312, m=156) — quantize.hpp seeds it via
//    Rng(seed) (rng.hpp:12-51).
//
// Every floating-point operation is an explicit round-to-nearest intrinsic
// on the device so nvcc can never contract a*b+c into an FMA;
// host builds use -ffp-contract=off.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define TRB_HD __host__ __device__ __forceinline__
#else
#define TRB_HD inline
#include <cmath>
#endif

namespace trb {

#if defined(__CUDA_ARCH__)
TRB_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
TRB_HD double xsub(double a, double b) { return __dsub_rn(a, b); }
TRB_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
TRB_HD double xdiv(double a, double b) { return __ddiv_rn(a, b); }
TRB_HD double xsqrt(double a) { return __dsqrt_rn(a); }
#else
TRB_HD double xadd(double a, double b) { return a + b; }
TRB_HD double xsub(double a, double b) { return a - b; }
TRB_HD double xmul(double a, double b) { return a * b; }
TRB_HD double xdiv(double a, double b) { return a / b; }
TRB_HD double xsqrt(double a) { return std::sqrt(a); }
#endif

TRB_HD double xfabs(double a) { return a < 0.0 ? -a : (a == 0.0 ? 0.0 : a); }

// glibc 2.39 __hypot kernel, non-FMA variant:
//   h = sqrt(ax*ax + ay*ay)
//   if h <= 2*ay: d = h - ay; t1 = ax*(2d - ax); t2 = (d - 2(ax - ay))*d
//   else:         d = h - ax; t1 = 2d*(ax - 2ay); t2 = (4d - ay)*ay + d*d
//   h -= (t1 + t2) / (2h)
TRB_HD double glibc_hypot_kernel(double ax, double ay) {
  double h = xsqrt(xadd(xmul(ax, ax), xmul(ay, ay)));
  double t1, t2;
  if (h <= xadd(ay, ay)) {
    const double d = xsub(h, ay);
    t1 = xmul(ax, xsub(xadd(d, d), ax));
    t2 = xmul(xsub(d, xadd(xsub(ax, ay), xsub(ax, ay))), d);
  } else {
    const double d = xsub(h, ax);
    t1 = xmul(xadd(d, d), xsub(ax, xadd(ay, ay)));
    t2 = xadd(xmul(xsub(xmul(4.0, d), ay), ay), xmul(d, d));
  }
  return xsub(h, xdiv(xadd(t1, t2), xadd(h, h)));
}

TRB_HD double glibc_hypot(double x, double y) {
  // non-finite inputs: inf wins over nan (C99 F.10.4.3)
  const double fx = xfabs(x), fy = xfabs(y);
  if (!(fx <= 1.7976931348623157e308) || !(fy <= 1.7976931348623157e308)) {
    if (fx == __builtin_inf() || fy == __builtin_inf()) return __builtin_inf();
    return x + y;  // nan
  }
  double ax = fx < fy ? fy : fx;
  double ay = fx < fy ? fx : fy;
  const double kLarge = 6.703903964971299e153;    // 0x1p+511
  const double kTiny = 6.717876107567089e-139;    // 0x1p-459
  const double kEps = 5.551115123125783e-17;      // 0x1p-54
  const double kScaleDn = 2.409919865102884e-181;  // 0x1p-600
  const double kScaleUp = 4.149515568880993e180;   // 0x1p+600
  if (ax > kLarge) {
    if (ay <= xmul(ax, kEps)) return xadd(ax, ay);
    return xmul(glibc_hypot_kernel(xmul(ax, kScaleDn), xmul(ay, kScaleDn)), kScaleUp);
  }
  if (ay < kTiny) {
    if (ax >= xmul(ay, 18014398509481984.0 /* 0x1p54 */)) return xadd(ax, ay);
    return xmul(glibc_hypot_kernel(xmul(ax, kScaleUp), xmul(ay, kScaleUp)), kScaleDn);
  }
  if (ay <= xmul(ax, kEps)) return xadd(ax, ay);
  return glibc_hypot_kernel(ax, ay);
}

// std::lround for the tracker's window placement (tracking.hpp:62-63):
// round half away from zero.
TRB_HD long long xlround(double v) {
#if defined(__CUDA_ARCH__)
  return llround(v);
#else
  return std::llround(v);
#endif
}

// std::mt19937_64 restated from its published definition.
struct Mt64 {
  uint64_t mt[312];
  int idx;
  TRB_HD void seed(uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    idx = 312;
  }
  TRB_HD uint64_t next() {
    if (idx >= 312) {
      for (int i = 0; i < 312; ++i) {
        const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        mt[i] = mt[(i + 156) % 312] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
  }
  // Rng::uniform (rng.hpp:22) and Rng::uniform_int (rng.hpp:27-30)
  TRB_HD double uniform() { return (double)(next() >> 11) * 1.1102230246251565e-16 /* 0x1p-53 */; }
  TRB_HD int64_t uniform_int(int64_t lo, int64_t hi) {
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(next() % span);
  }
};

// mix_seed, rng.hpp:63-68
TRB_HD uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace trb

// Device bounds checks, compiled in with -DTRB_DEBUG (make DEBUG=1).
#if defined(TRB_DEBUG) && defined(__CUDA_ARCH__)
#include <cstdio>
#define TRB_CHECK(cond, what, a, b)                                                                  \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("TRB_CHECK failed: %s (%lld, %lld) block %d thread %d line %d\n", what, (long long)(a), \
             (long long)(b), blockIdx.x, threadIdx.x, __LINE__);                                     \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define TRB_CHECK(cond, what, a, b) ((void)0)
#endif
