/* plane_hash.h — TEST INFRASTRUCTURE ONLY.  A position-keyed 64-bit digest
 * of a byte plane (mask, label image) shared by the reference shim
 * (ref_driver.cpp) and the C restatement (trb_oracle.c), so per-frame
 * outputs of the GPU path can be compared with the reference's without
 * storing whole planes.  h = n + sum_i mix(word_i + (i+1) * phi) mod 2^64
 * over little-endian 8-byte words (the tail zero-padded); mix is the
 * splitmix64 finaliser.  Not cryptographic: a checker, not a proof. */
#ifndef TRB_PLANE_HASH_H_
#define TRB_PLANE_HASH_H_
#include <stdint.h>
#include <string.h>

static inline uint64_t trb_ph_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static inline uint64_t trb_plane_hash(const void* data, int64_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = (uint64_t)n;
  int64_t nw = n / 8, i;
  for (i = 0; i < nw; ++i) {
    uint64_t w;
    memcpy(&w, p + 8 * i, 8);
    h += trb_ph_mix(w + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ULL);
  }
  if (n % 8) {
    uint64_t w = 0;
    memcpy(&w, p + 8 * nw, (size_t)(n % 8));
    h += trb_ph_mix(w + (uint64_t)(nw + 1) * 0x9e3779b97f4a7c15ULL);
  }
  return h;
}
#endif
