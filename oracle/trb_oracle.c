/*
 * trb_oracle.c — TEST INFRASTRUCTURE ONLY (see trb_oracle.h).
 *
 * CPU restatement of the reference front end, one function per reference
 * routine, each citing the file:line it restates (paths relative to
 * /root/reference/proj/include/teamrec/).  Written in plain C so it shares
 * no code with the reference or with the CUDA product.  Compile with
 * -O2 -ffp-contract=off and NO -march=native.
 */
#include "trb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================
 * mt19937_64 + Rng (rng.hpp:12-68).  The standard 64-bit Mersenne twister
 * (n=312, m=156) restated from its published definition.
 * ==================================================================== */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->spare = 0.0;
  r->have_spare = 0;
}

static uint64_t rng_next(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* Rng::uniform, rng.hpp:22 */
static double rng_uniform(orc_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

/* Rng::uniform_int, rng.hpp:27-30 */
static int64_t rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi) {
  const uint64_t span = (uint64_t)(hi - lo) + 1;
  return lo + (int64_t)(rng_next(r) % span);
}

/* Rng::gaussian, rng.hpp:33-45 */
static double rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_uniform(r);
  while (u1 <= 0.0) u1 = rng_uniform(r);
  const double u2 = rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

/* mix_seed, rng.hpp:63-68 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double orc_libm_hypot(double x, double y) { return hypot(x, y); }
void orc_libm_hypot_n(const double* x, const double* y, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = hypot(x[i], y[i]);
}

/* ======================================================================
 * Motion (motion.hpp)
 * ==================================================================== */

/* window_background, motion.hpp:127-144 */
uint8_t orc_window_background(const uint8_t* vals, int n, int method, int bins) {
  if (method == TRB_BG_MEAN) {
    uint64_t sum = 0;
    for (int i = 0; i < n; ++i) sum += vals[i];
    return (uint8_t)((2 * sum + (uint64_t)n) / (2 * (uint64_t)n));
  }
  int count[256];
  memset(count, 0, sizeof(count));
  for (int i = 0; i < n; ++i) count[(vals[i] * bins) / 256] += 1;
  int best = 0;
  for (int b = 1; b < bins; ++b)
    if (count[b] > count[best]) best = b;
  uint64_t sum = 0, cnt = 0;
  for (int i = 0; i < n; ++i)
    if ((vals[i] * bins) / 256 == best) sum += vals[i], ++cnt;
  return (uint8_t)((2 * sum + cnt) / (2 * cnt));
}

struct orc_motion {
  trb_motion_config cfg;
  int w, h, seen;
  uint8_t* ring;  /* frame-major: ring[slot * px + p] (layout is free; semantics are motion.hpp:170-177) */
  uint64_t* sums; /* running window sum per pixel, motion.hpp:211 */
  uint8_t* scratch;
};

orc_motion* orc_motion_create(const trb_motion_config* cfg, int width, int height) {
  orc_motion* m = (orc_motion*)calloc(1, sizeof(orc_motion));
  m->cfg = *cfg;
  m->w = width;
  m->h = height;
  const size_t px = (size_t)width * height;
  m->ring = (uint8_t*)calloc(px * (size_t)cfg->window, 1);
  m->sums = (uint64_t*)calloc(px, sizeof(uint64_t));
  m->scratch = (uint8_t*)malloc((size_t)cfg->window);
  return m;
}

void orc_motion_destroy(orc_motion* m) {
  if (!m) return;
  free(m->ring);
  free(m->sums);
  free(m->scratch);
  free(m);
}

static uint8_t orc_bg_at(const orc_motion* m, size_t p) {
  const int W = m->cfg.window;
  const size_t px = (size_t)m->w * m->h;
  if (m->cfg.method == TRB_BG_MEAN) return (uint8_t)((2 * m->sums[p] + (uint64_t)W) / (2 * (uint64_t)W));
  for (int s = 0; s < W; ++s) m->scratch[s] = m->ring[(size_t)s * px + p];
  return orc_window_background(m->scratch, W, m->cfg.method, m->cfg.bins);
}

/* MotionDetector::push, motion.hpp:164-193 */
int orc_motion_push(orc_motion* m, const uint8_t* gray, uint8_t* mask_out) {
  const size_t px = (size_t)m->w * m->h;
  const int W = m->cfg.window;
  const size_t slot = (size_t)(m->seen % W);
  const int full_before = m->seen >= W;
  uint8_t* ring = m->ring + slot * px;
  for (size_t p = 0; p < px; ++p) {
    if (full_before) m->sums[p] -= ring[p];
    ring[p] = gray[p];
    m->sums[p] += ring[p];
  }
  ++m->seen;
  if (m->seen < W) return 0;
  for (size_t p = 0; p < px; ++p) {
    const int bg = orc_bg_at(m, p);
    const int diff = (int)gray[p] - bg;
    mask_out[p] = (diff > m->cfg.threshold || -diff > m->cfg.threshold) ? 1 : 0;
  }
  if (m->cfg.morph != TRB_MORPH_NONE) {
    uint8_t* tmp = (uint8_t*)malloc(px);
    memcpy(tmp, mask_out, px);
    orc_morph(tmp, m->w, m->h, m->cfg.morph, mask_out);
    free(tmp);
  }
  return 1;
}

/* MotionDetector::background, motion.hpp:196-203 */
void orc_motion_background(const orc_motion* m, uint8_t* out) {
  const size_t px = (size_t)m->w * m->h;
  for (size_t p = 0; p < px; ++p) out[p] = orc_bg_at(m, p);
}

/* luma / grayscale, frame.hpp:91-104 */
void orc_grayscale(const uint8_t* rgb, int64_t n_px, uint8_t* out) {
  for (int64_t i = 0; i < n_px; ++i)
    out[i] = (uint8_t)((77 * rgb[3 * i] + 150 * rgb[3 * i + 1] + 29 * rgb[3 * i + 2] + 128) >> 8);
}

/* warp_frame, motion.hpp:81-119.  Same expression trees as the reference
 * (left-to-right, no contraction): the inverse by cofactors / det, per pixel
 * w = inv20*x + inv21*y + inv22 (skipped when |w| < 1e-12), source
 * (sx, sy), floor, bilinear weights, clamp to [0, 255], lround. */
static double warp_tap(const uint8_t* f, int w, int h, int ch, int x, int y, int c) {
  if (x < 0 || y < 0 || x >= w || y >= h) return 0.0;
  return f[((size_t)y * w + x) * ch + c];
}
int orc_warp_frame(const uint8_t* f, int w, int hgt, int ch, const double* hm, uint8_t* out) {
  for (int i = 0; i < 9; ++i)
    if (!isfinite(hm[i])) return 1;
  if (hm[8] == 0.0) return 2;
#define H(r, c) hm[3 * (r) + (c)]
  const double det = H(0, 0) * (H(1, 1) * H(2, 2) - H(1, 2) * H(2, 1)) - H(0, 1) * (H(1, 0) * H(2, 2) - H(1, 2) * H(2, 0)) +
                     H(0, 2) * (H(1, 0) * H(2, 1) - H(1, 1) * H(2, 0));
  if (fabs(det) < 1e-12) return 3;
  const double inv[3][3] = {
      {(H(1, 1) * H(2, 2) - H(1, 2) * H(2, 1)) / det, (H(0, 2) * H(2, 1) - H(0, 1) * H(2, 2)) / det,
       (H(0, 1) * H(1, 2) - H(0, 2) * H(1, 1)) / det},
      {(H(1, 2) * H(2, 0) - H(1, 0) * H(2, 2)) / det, (H(0, 0) * H(2, 2) - H(0, 2) * H(2, 0)) / det,
       (H(0, 2) * H(1, 0) - H(0, 0) * H(1, 2)) / det},
      {(H(1, 0) * H(2, 1) - H(1, 1) * H(2, 0)) / det, (H(0, 1) * H(2, 0) - H(0, 0) * H(2, 1)) / det,
       (H(0, 0) * H(1, 1) - H(0, 1) * H(1, 0)) / det}};
#undef H
  memset(out, 0, (size_t)w * hgt * ch);
  for (int y = 0; y < hgt; ++y)
    for (int x = 0; x < w; ++x) {
      const double ww = inv[2][0] * x + inv[2][1] * y + inv[2][2];
      if (fabs(ww) < 1e-12) continue;
      const double sx = (inv[0][0] * x + inv[0][1] * y + inv[0][2]) / ww;
      const double sy = (inv[1][0] * x + inv[1][1] * y + inv[1][2]) / ww;
      const int x0 = (int)floor(sx), y0 = (int)floor(sy);
      const double dx = sx - x0, dy = sy - y0;
      for (int c = 0; c < ch; ++c) {
        const double v = (1 - dx) * (1 - dy) * warp_tap(f, w, hgt, ch, x0, y0, c) +
                         dx * (1 - dy) * warp_tap(f, w, hgt, ch, x0 + 1, y0, c) +
                         (1 - dx) * dy * warp_tap(f, w, hgt, ch, x0, y0 + 1, c) +
                         dx * dy * warp_tap(f, w, hgt, ch, x0 + 1, y0 + 1, c);
        const double lo = (0.0 < v) ? v : 0.0;        /* std::max(0.0, v) */
        const double cl = (lo < 255.0) ? lo : 255.0;  /* std::min(255.0, .) */
        out[((size_t)y * w + x) * ch + c] = (uint8_t)lround(cl);
      }
    }
  return 0;
}

/* extract_blob_features, segmentation.hpp:268-291: raster-order double
 * sums of the pixel values per label (luma for RGB, frame.hpp:91-93), then
 * sum / area and (x_max - x_min + 1) / (y_max - y_min + 1). */
int orc_blob_features(const int32_t* labels, int w, int h, const uint8_t* frame, int fw, int fh, int ch,
                      const trb_blob* blobs, int n, double* mean, double* aspect) {
  if (w != fw || h != fh) return -1;
  double* sum = (double*)calloc(n > 0 ? (size_t)n : 1, sizeof(double));
  for (int64_t p = 0; p < (int64_t)w * h; ++p) {
    const int l = labels[p];
    if (l == 0) continue;
    double v;
    if (ch == 1) {
      v = frame[p];
    } else {
      const uint8_t* q = frame + 3 * p;
      v = (double)(uint8_t)((77 * q[0] + 150 * q[1] + 29 * q[2] + 128) >> 8);
    }
    sum[l - 1] += v;
  }
  for (int i = 0; i < n; ++i) {
    mean[i] = sum[i] / blobs[i].area;
    aspect[i] = (double)(blobs[i].x_max - blobs[i].x_min + 1) / (double)(blobs[i].y_max - blobs[i].y_min + 1);
  }
  free(sum);
  return 0;
}

/* 3x3 morphology — new stage, no reference. */
static void morph_pass(const uint8_t* in, int w, int h, int dilate, uint8_t* out) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      int acc = dilate ? 0 : 1;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int nx = x + dx, ny = y + dy;
          if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
          const int v = in[(size_t)ny * w + nx] != 0;
          if (dilate) acc |= v;
          else acc &= v;
        }
      out[(size_t)y * w + x] = (uint8_t)acc;
    }
}

void orc_morph(const uint8_t* in, int width, int height, int op, uint8_t* out) {
  const size_t px = (size_t)width * height;
  uint8_t* tmp = (uint8_t*)malloc(px);
  switch (op) {
    case TRB_MORPH_ERODE: morph_pass(in, width, height, 0, out); break;
    case TRB_MORPH_DILATE: morph_pass(in, width, height, 1, out); break;
    case TRB_MORPH_OPEN:
      morph_pass(in, width, height, 0, tmp);
      morph_pass(tmp, width, height, 1, out);
      break;
    case TRB_MORPH_CLOSE:
      morph_pass(in, width, height, 1, tmp);
      morph_pass(tmp, width, height, 0, out);
      break;
    default:
      for (size_t p = 0; p < px; ++p) out[p] = in[p] != 0;
  }
  free(tmp);
}

/* ======================================================================
 * Labelling.  Output contract of finalize_labels (segmentation.hpp:88-149):
 * dense labels 1..k in raster order of each component's first pixel,
 * components with area < min_area dropped and the rest compacted; Blob
 * area/bbox/centroid accumulated in raster order.  Components are found
 * with an independent BFS flood fill (like tests/oracles.hpp:39-72).
 * ==================================================================== */
int orc_label(const uint8_t* mask, int w, int h, int connectivity, int min_area, int32_t* labels, trb_blob* blobs,
              int cap, int64_t* pixels) {
  const size_t px = (size_t)w * h;
  int32_t* comp = (int32_t*)calloc(px, sizeof(int32_t));
  int64_t* queue = (int64_t*)malloc(px * sizeof(int64_t) + 8);
  int32_t* area = (int32_t*)malloc((px + 2) * sizeof(int32_t));
  int ncomp = 0;
  for (size_t sp = 0; sp < px; ++sp) {
    if (!mask[sp] || comp[sp]) continue;
    ++ncomp;
    size_t qh = 0, qt = 0;
    queue[qt++] = (int64_t)sp;
    comp[sp] = ncomp;
    int a = 0;
    while (qh < qt) {
      const int64_t p = queue[qh++];
      ++a;
      const int x = (int)(p % w), y = (int)(p / w);
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy) continue;
          if (connectivity == TRB_CONN_FOUR && dx && dy) continue;
          const int nx = x + dx, ny = y + dy;
          if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
          const size_t np = (size_t)ny * w + nx;
          if (!mask[np] || comp[np]) continue;
          comp[np] = ncomp;
          queue[qt++] = (int64_t)np;
        }
    }
    area[ncomp] = a;
  }
  /* min_area compaction preserving order, segmentation.hpp:110-113 */
  int32_t* remap = (int32_t*)calloc((size_t)ncomp + 1, sizeof(int32_t));
  int next = 0;
  for (int d = 1; d <= ncomp; ++d)
    if (area[d] >= min_area) remap[d] = ++next;
  /* blob stats in raster order, segmentation.hpp:115-147 */
  int64_t* sx = (int64_t*)calloc((size_t)next + 1, sizeof(int64_t));
  int64_t* sy = (int64_t*)calloc((size_t)next + 1, sizeof(int64_t));
  int32_t* bx0 = (int32_t*)malloc(((size_t)next + 1) * sizeof(int32_t));
  int32_t* by0 = (int32_t*)malloc(((size_t)next + 1) * sizeof(int32_t));
  int32_t* bx1 = (int32_t*)malloc(((size_t)next + 1) * sizeof(int32_t));
  int32_t* by1 = (int32_t*)malloc(((size_t)next + 1) * sizeof(int32_t));
  int32_t* ba = (int32_t*)calloc((size_t)next + 1, sizeof(int32_t));
  for (int k = 0; k <= next; ++k) bx0[k] = w, by0[k] = h, bx1[k] = -1, by1[k] = -1;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t p = (size_t)y * w + x;
      const int lab = comp[p] ? remap[comp[p]] : 0;
      if (labels) labels[p] = lab;
      if (!lab) continue;
      ba[lab] += 1;
      if (x < bx0[lab]) bx0[lab] = x;
      if (y < by0[lab]) by0[lab] = y;
      if (x > bx1[lab]) bx1[lab] = x;
      if (y > by1[lab]) by1[lab] = y;
      sx[lab] += x;
      sy[lab] += y;
    }
  if (pixels) {
    int64_t* off = (int64_t*)calloc((size_t)next + 2, sizeof(int64_t));
    for (int k = 1; k <= next; ++k) off[k + 1] = off[k] + ba[k];
    for (size_t p = 0; p < px; ++p) {
      const int lab = comp[p] ? remap[comp[p]] : 0;
      if (lab) pixels[off[lab]++] = (int64_t)p;
    }
    free(off);
  }
  for (int k = 1; k <= next && k <= cap; ++k) {
    trb_blob* b = &blobs[k - 1];
    b->label = k;
    b->area = ba[k];
    b->x_min = bx0[k];
    b->y_min = by0[k];
    b->x_max = bx1[k];
    b->y_max = by1[k];
    /* the reference sums integer coordinates into a double (exact), then
       divides by the area: segmentation.hpp:139-147 */
    b->cx = (double)sx[k] / ba[k];
    b->cy = (double)sy[k] / ba[k];
  }
  free(comp), free(queue), free(area), free(remap), free(sx), free(sy);
  free(bx0), free(by0), free(bx1), free(by1), free(ba);
  return next;
}

/* ======================================================================
 * Quantizer (quantize.hpp)
 * ==================================================================== */

/* ColorQuantizer::assign, quantize.hpp:20-29 */
int orc_quantizer_assign(const double* c, int k, double r, double g, double b) {
  int best = 0;
  double best_d = INFINITY;
  for (int i = 0; i < k; ++i) {
    const double dr = r - c[3 * i], dg = g - c[3 * i + 1], db = b - c[3 * i + 2];
    const double d = dr * dr + dg * dg + db * db;
    if (d < best_d) best_d = d, best = i;
  }
  return best;
}

static double sq_dist3(const double* a, const double* b) {
  const double dr = a[0] - b[0], dg = a[1] - b[1], db = a[2] - b[2];
  return dr * dr + dg * dg + db * db;
}

/* quantize_colors, quantize.hpp:43-118 */
void orc_quantize_colors(const double* px, int64_t n, int k, int iters, uint64_t seed, double* centers) {
  orc_rng rng;
  rng_seed(&rng, seed);
  int nc = 0;
  const int64_t first = rng_uniform_int(&rng, 0, n - 1);
  memcpy(&centers[0], &px[3 * first], 3 * sizeof(double));
  nc = 1;
  double* d2 = (double*)malloc((size_t)n * sizeof(double));
  while (nc < k) {
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double best = INFINITY;
      for (int c = 0; c < nc; ++c) {
        const double d = sq_dist3(&px[3 * i], &centers[3 * c]);
        best = d < best ? d : best; /* std::min(best, d) == (d < best) ? d : best */
      }
      d2[i] = best;
      total += best;
    }
    int64_t pick = 0;
    if (total > 0.0) {
      const double r = rng_uniform(&rng) * total;
      double acc = 0.0;
      pick = n - 1;
      for (int64_t i = 0; i < n; ++i) {
        acc += d2[i];
        if (acc > r) {
          pick = i;
          break;
        }
      }
    }
    memcpy(&centers[3 * nc], &px[3 * pick], 3 * sizeof(double));
    ++nc;
  }
  int* assign = (int*)calloc((size_t)n, sizeof(int));
  double* sum = (double*)malloc((size_t)k * 3 * sizeof(double));
  int64_t* count = (int64_t*)malloc((size_t)k * sizeof(int64_t));
  for (int it = 0; it < iters; ++it) {
    int moved = 0;
    for (int64_t i = 0; i < n; ++i) assign[i] = orc_quantizer_assign(centers, k, px[3 * i], px[3 * i + 1], px[3 * i + 2]);
    memset(sum, 0, (size_t)k * 3 * sizeof(double));
    memset(count, 0, (size_t)k * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
      const int c = assign[i];
      sum[3 * c] += px[3 * i];
      sum[3 * c + 1] += px[3 * i + 1];
      sum[3 * c + 2] += px[3 * i + 2];
      count[c] += 1;
    }
    for (int c = 0; c < k; ++c) {
      double ncent[3];
      if (count[c] == 0) {
        int64_t far = 0;
        double far_d = -1.0;
        for (int64_t i = 0; i < n; ++i) {
          const double d = sq_dist3(&px[3 * i], &centers[3 * assign[i]]);
          if (d > far_d) far_d = d, far = i;
        }
        memcpy(ncent, &px[3 * far], sizeof(ncent));
      } else {
        const double m = (double)count[c];
        ncent[0] = sum[3 * c] / m;
        ncent[1] = sum[3 * c + 1] / m;
        ncent[2] = sum[3 * c + 2] / m;
      }
      if (ncent[0] != centers[3 * c] || ncent[1] != centers[3 * c + 1] || ncent[2] != centers[3 * c + 2]) moved = 1;
      memcpy(&centers[3 * c], ncent, sizeof(ncent));
    }
    if (!moved) break;
  }
  free(d2), free(assign), free(sum), free(count);
}

/* ======================================================================
 * Tracking (tracking.hpp)
 * ==================================================================== */
typedef struct {
  int x0, y0, x1, y1;
} orc_rect;

/* clip_window, tracking.hpp:61-66 */
static orc_rect clip_window(int fw, int fh, double cx, double cy, int w, int h) {
  const int x0 = (int)lround(cx) - w / 2;
  const int y0 = (int)lround(cy) - h / 2;
  orc_rect r;
  r.x0 = x0 > 0 ? x0 : 0;
  r.y0 = y0 > 0 ? y0 : 0;
  r.x1 = fw < x0 + w ? fw : x0 + w;
  r.y1 = fh < y0 + h ? fh : y0 + h;
  return r;
}
static int rect_empty(orc_rect r) { return r.x0 >= r.x1 || r.y0 >= r.y1; }

/* rgb_at, tracking.hpp:68-75 */
static void rgb_at(const uint8_t* f, int fw, int ch, int x, int y, double* o) {
  if (ch == 1) {
    const double v = f[(size_t)y * fw + x];
    o[0] = o[1] = o[2] = v;
    return;
  }
  const size_t p = ((size_t)y * fw + x) * 3;
  o[0] = f[p], o[1] = f[p + 1], o[2] = f[p + 2];
}

/* detail::histogram_opt, tracking.hpp:79-102 */
int orc_histogram(const uint8_t* frame, int fw, int fh, int ch, double cx, double cy, int w, int h,
                  const double* centers, int k, int epan, double* hist) {
  const orc_rect r = clip_window(fw, fh, cx, cy, w, h);
  if (rect_empty(r)) return 0;
  for (int i = 0; i < k; ++i) hist[i] = 0.0;
  const double hx = w / 2.0, hy = h / 2.0;
  double total = 0.0;
  for (int y = r.y0; y < r.y1; ++y)
    for (int x = r.x0; x < r.x1; ++x) {
      double wgt = 1.0;
      if (epan) {
        const double ux = (x - cx) / hx, uy = (y - cy) / hy;
        const double t = 1.0 - (ux * ux + uy * uy);
        wgt = (0.0 < t) ? t : 0.0; /* std::max(0.0, t) */
      }
      if (wgt <= 0.0) continue;
      double rgb[3];
      rgb_at(frame, fw, ch, x, y, rgb);
      hist[orc_quantizer_assign(centers, k, rgb[0], rgb[1], rgb[2])] += wgt;
      total += wgt;
    }
  if (total <= 0.0) return 0;
  for (int i = 0; i < k; ++i) hist[i] /= total;
  return 1;
}

/* bhattacharyya, tracking.hpp:114-119 */
static double bhattacharyya(const double* p, const double* q, int k) {
  double s = 0.0;
  for (int i = 0; i < k; ++i) s += sqrt(p[i] * q[i]);
  return s;
}

/* meanshift_step, tracking.hpp:125-157 */
void orc_meanshift_step(const uint8_t* frame, int fw, int fh, int ch, double* cxp, double* cyp, int w, int h,
                        const double* centers, const double* target, int k, int max_iters, double eps, int* status) {
  if (*status != TRB_TRACK_ACTIVE) return;
  double* p = (double*)malloc((size_t)k * sizeof(double));
  for (int it = 0; it < max_iters; ++it) {
    const int ok = orc_histogram(frame, fw, fh, ch, *cxp, *cyp, w, h, centers, k, 1, p);
    if (!ok || bhattacharyya(p, target, k) <= 0.0) {
      *status = TRB_TRACK_LOST;
      break;
    }
    const orc_rect r = clip_window(fw, fh, *cxp, *cyp, w, h);
    double sw = 0.0, sx = 0.0, sy = 0.0;
    for (int y = r.y0; y < r.y1; ++y)
      for (int x = r.x0; x < r.x1; ++x) {
        double rgb[3];
        rgb_at(frame, fw, ch, x, y, rgb);
        const int b = orc_quantizer_assign(centers, k, rgb[0], rgb[1], rgb[2]);
        if (p[b] <= 0.0) continue;
        const double wgt = sqrt(target[b] / p[b]);
        sw += wgt;
        sx += wgt * x;
        sy += wgt * y;
      }
    if (sw <= 0.0) {
      *status = TRB_TRACK_LOST;
      break;
    }
    const double nx = sx / sw, ny = sy / sw;
    const double shift = hypot(nx - *cxp, ny - *cyp);
    *cxp = nx;
    *cyp = ny;
    if (shift < eps) break;
  }
  free(p);
}

typedef struct {
  int id;
  double cx, cy;
  int w, h;
  double* hist;
  double* centers;
  int status, lost;
} orc_track;

struct orc_tracker {
  trb_tracker_config cfg;
  orc_track* tracks;
  int n, cap;
  trb_track_log_entry* log;
  int64_t nlog, logcap;
  int next_id, frame_no;
};

orc_tracker* orc_tracker_create(const trb_tracker_config* cfg) {
  orc_tracker* t = (orc_tracker*)calloc(1, sizeof(orc_tracker));
  t->cfg = *cfg;
  t->next_id = 1;
  return t;
}

static void track_free(orc_track* tr) {
  free(tr->hist);
  free(tr->centers);
}

void orc_tracker_destroy(orc_tracker* t) {
  if (!t) return;
  for (int i = 0; i < t->n; ++i) track_free(&t->tracks[i]);
  free(t->tracks);
  free(t->log);
  free(t);
}

/* Tracker::spawn_track, tracking.hpp:208-234 */
static void spawn_track(orc_tracker* t, const uint8_t* frame, int fw, int fh, int ch, const trb_blob* blob) {
  const int K = t->cfg.k_clusters;
  orc_track tr;
  memset(&tr, 0, sizeof(tr));
  tr.id = t->next_id++;
  tr.cx = blob->cx;
  tr.cy = blob->cy;
  tr.w = blob->x_max - blob->x_min + 1;
  if (tr.w < 3) tr.w = 3;
  tr.h = blob->y_max - blob->y_min + 1;
  if (tr.h < 3) tr.h = 3;
  while (tr.w * tr.h < K) {
    if (tr.w <= tr.h) ++tr.w;
    else ++tr.h;
  }
  const orc_rect r = clip_window(fw, fh, tr.cx, tr.cy, tr.w, tr.h);
  if (rect_empty(r)) return;
  const int64_t n = (int64_t)(r.x1 - r.x0) * (r.y1 - r.y0);
  if (n < K) return;
  double* px = (double*)malloc((size_t)n * 3 * sizeof(double));
  int64_t i = 0;
  for (int y = r.y0; y < r.y1; ++y)
    for (int x = r.x0; x < r.x1; ++x, ++i) rgb_at(frame, fw, ch, x, y, &px[3 * i]);
  tr.centers = (double*)malloc((size_t)K * 3 * sizeof(double));
  orc_quantize_colors(px, n, K, t->cfg.kmeans_iters, orc_mix_seed(t->cfg.seed, (uint64_t)tr.id), tr.centers);
  free(px);
  tr.hist = (double*)malloc((size_t)K * sizeof(double));
  if (!orc_histogram(frame, fw, fh, ch, tr.cx, tr.cy, tr.w, tr.h, tr.centers, K, 1, tr.hist)) {
    track_free(&tr);
    return;
  }
  tr.status = TRB_TRACK_ACTIVE;
  if (t->n == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 16;
    t->tracks = (orc_track*)realloc(t->tracks, (size_t)t->cap * sizeof(orc_track));
  }
  t->tracks[t->n++] = tr;
}

/* Tracker::process, tracking.hpp:179-205 */
void orc_tracker_process(orc_tracker* t, const uint8_t* frame, int fw, int fh, int ch, const trb_blob* blobs,
                         int n_blobs) {
  const int K = t->cfg.k_clusters;
  for (int i = 0; i < t->n; ++i) {
    orc_track* tr = &t->tracks[i];
    orc_meanshift_step(frame, fw, fh, ch, &tr->cx, &tr->cy, tr->w, tr->h, tr->centers, tr->hist, K,
                       t->cfg.max_iters, t->cfg.eps, &tr->status);
  }
  for (int b = 0; b < n_blobs; ++b) {
    int matched = 0;
    for (int i = 0; i < t->n; ++i) {
      const orc_track* tr = &t->tracks[i];
      const double d = hypot(blobs[b].cx - tr->cx, blobs[b].cy - tr->cy);
      const double diag = sqrt((double)tr->w * tr->w + (double)tr->h * tr->h); /* Track::window_diagonal, :49 */
      if (d <= 1.5 * diag) {
        matched = 1;
        break;
      }
    }
    if (!matched) spawn_track(t, frame, fw, fh, ch, &blobs[b]);
  }
  for (int i = 0; i < t->n; ++i)
    if (t->tracks[i].status == TRB_TRACK_LOST) t->tracks[i].lost += 1;
  int j = 0;
  for (int i = 0; i < t->n; ++i) {
    if (t->tracks[i].status == TRB_TRACK_LOST && t->tracks[i].lost >= 5) {
      track_free(&t->tracks[i]);
      continue;
    }
    t->tracks[j++] = t->tracks[i];
  }
  t->n = j;
  for (int i = 0; i < t->n; ++i) {
    if (t->nlog == t->logcap) {
      t->logcap = t->logcap ? 2 * t->logcap : 256;
      t->log = (trb_track_log_entry*)realloc(t->log, (size_t)t->logcap * sizeof(trb_track_log_entry));
    }
    trb_track_log_entry* e = &t->log[t->nlog++];
    memset(e, 0, sizeof(*e));
    e->frame = t->frame_no;
    e->track_id = t->tracks[i].id;
    e->x = t->tracks[i].cx;
    e->y = t->tracks[i].cy;
    e->w = t->tracks[i].w;
    e->h = t->tracks[i].h;
    e->status = t->tracks[i].status;
  }
  ++t->frame_no;
}

int orc_tracker_num_tracks(const orc_tracker* t) { return t->n; }

void orc_tracker_tracks(const orc_tracker* t, trb_track* out) {
  for (int i = 0; i < t->n; ++i) {
    const orc_track* tr = &t->tracks[i];
    trb_track* o = &out[i];
    memset(o, 0, sizeof(*o));
    o->track_id = tr->id;
    o->w = tr->w;
    o->h = tr->h;
    o->status = tr->status;
    o->lost_frames = tr->lost;
    o->k = t->cfg.k_clusters;
    o->cx = tr->cx;
    o->cy = tr->cy;
  }
}

void orc_tracker_track_model(const orc_tracker* t, int i, double* centers, double* hist) {
  const int K = t->cfg.k_clusters;
  if (centers) memcpy(centers, t->tracks[i].centers, (size_t)K * 3 * sizeof(double));
  if (hist) memcpy(hist, t->tracks[i].hist, (size_t)K * sizeof(double));
}

int64_t orc_tracker_log_size(const orc_tracker* t) { return t->nlog; }

void orc_tracker_log(const orc_tracker* t, trb_track_log_entry* out) {
  memcpy(out, t->log, (size_t)t->nlog * sizeof(trb_track_log_entry));
}

/* ======================================================================
 * Synthetic clips (synth.hpp:45-101)
 * ==================================================================== */
struct orc_synth {
  int w, h, ch, n, t;
  uint8_t bg;
  int32_t* si;
  double* sd;
  orc_rng rng;
};

orc_synth* orc_synth_create(int width, int height, int channels, uint8_t background, int n_shapes,
                            const int32_t* shape_int, const double* shape_dbl, uint64_t seed) {
  orc_synth* s = (orc_synth*)calloc(1, sizeof(orc_synth));
  s->w = width, s->h = height, s->ch = channels, s->n = n_shapes, s->bg = background;
  s->si = (int32_t*)malloc((size_t)n_shapes * 5 * sizeof(int32_t) + 4);
  s->sd = (double*)malloc((size_t)n_shapes * 5 * sizeof(double) + 8);
  memcpy(s->si, shape_int, (size_t)n_shapes * 5 * sizeof(int32_t));
  memcpy(s->sd, shape_dbl, (size_t)n_shapes * 5 * sizeof(double));
  rng_seed(&s->rng, seed);
  return s;
}

void orc_synth_destroy(orc_synth* s) {
  if (!s) return;
  free(s->si), free(s->sd), free(s);
}

int orc_synth_next(orc_synth* s, uint8_t* out, int32_t* rects) {
  const int t = s->t++;
  const size_t px = (size_t)s->w * s->h;
  memset(out, s->bg, px * (size_t)s->ch);
  for (int k = 0; k < s->n; ++k) {
    const int32_t* si = &s->si[5 * k];
    const double* sd = &s->sd[5 * k];
    double x = sd[0] + sd[2] * t;
    double y = sd[1] + sd[3] * t;
    if (sd[4] > 0.0) {
      x += 0.0 + sd[4] * rng_gaussian(&s->rng);
      y += 0.0 + sd[4] * rng_gaussian(&s->rng);
    }
    const int ix = (int)lround(x), iy = (int)lround(y);
    if (ix < 0 || iy < 0 || ix + si[0] > s->w || iy + si[1] > s->h) return -1;
    if (rects) rects[4 * k] = ix, rects[4 * k + 1] = iy, rects[4 * k + 2] = si[0], rects[4 * k + 3] = si[1];
    for (int yy = iy; yy < iy + si[1]; ++yy)
      for (int xx = ix; xx < ix + si[0]; ++xx) {
        if (s->ch == 1) {
          out[(size_t)yy * s->w + xx] = (uint8_t)si[2];
        } else {
          uint8_t* p = &out[((size_t)yy * s->w + xx) * 3];
          p[0] = (uint8_t)si[2], p[1] = (uint8_t)si[3], p[2] = (uint8_t)si[4];
        }
      }
  }
  return 0;
}

#include "plane_hash.h"
uint64_t orc_plane_hash(const void* data, int64_t n) { return trb_plane_hash(data, n); }
