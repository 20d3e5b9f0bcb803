/*
 * csp_synth.h -- seeded, counter-based synthetic random binary CSP generator.
 *
 * This module is INPUT GENERATION ONLY.  It holds none of the method's
 * arithmetic (no support test, no recurrence, no arc consistency): it only
 * answers "is pair {x,y} constrained?" and "is value pair (a,b) allowed in
 * rel(c_xy)?" for a seeded random instance, and "is bit (x,a) kept?" for
 * seeded random domain states.  It is the one piece of code the CPU oracle
 * (oracle/) and the CUDA path (paper_2407_11388_b200/csrc/) both use, as the
 * task rules permit ("only the seeded input generators serve both, from a
 * module of their own").  synth/__init__.py is an independent numpy port of
 * the same functions; tests check the three agree bit for bit.
 *
 * Workload shape follows PAPER.md §5.2 (Benchmark, lines 232-236): "for a
 * number of n variables and a given constraint density d ... each pair of
 * them is assigned with a constraint with the possibility of d".  The paper
 * does not state domain size or tightness; they are explicit parameters here
 * (SPEC.md instance_gen, lines 433-456: tightness = probability that a value
 * pair is FORBIDDEN, drawn per cell).
 *
 * Counter-based (not sequential) so host C, CUDA and numpy produce identical
 * bits in any order and in parallel (SURVEY.md §8(d) "Generator").
 *
 * Frozen specification (also in DESIGN.md §"Input recipe"):
 *   mix64(z)       = splitmix64 finalizer
 *   key(seed, tag) = mix64(seed ^ tag)
 *   present(x<y)   = (mix64(key(seed,TAG_PRES) ^ mix64(x*n + y)) >> 32) < dens_q32
 *                    dens_q32 = round(density * 2^32) in [0, 2^32]
 *   allowed(x<y,a,b): q = ceil(d/4); pk = mix64(key(seed,TAG_CELL) ^ mix64(x*n + y))
 *                    h = mix64(pk + (a*q + b/4 + 1) * GAMMA)   (a splitmix64 stream per pair)
 *                    allowed iff ((h >> 16*(b%4)) & 0xFFFF) >= t_q16
 *                    t_q16 = round(tightness * 65536) in [0, 65536]
 *   rel(c_yx) for x<y is the transpose: (b,a) allowed in c_yx iff (a,b) in c_xy.
 *   keep(x,a) (W-rand) = (mix64(key(seed,TAG_KEEP) ^ mix64(x*64 + a)) & 0xFFFF) < keep_q16
 *   pick(seed, k, m) = mix64(key(seed,TAG_PICK) ^ mix64(k)) % m   (seeded choices)
 */
#ifndef CSP_SYNTH_H
#define CSP_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_FN static __host__ __device__ __forceinline__
#else
#define SYNTH_FN static inline
#endif

#define SYNTH_TAG_PRES 0x50524553454E4345ULL /* "PRESENCE" */
#define SYNTH_TAG_CELL 0x43454C4C42495453ULL /* "CELLBITS" */
#define SYNTH_TAG_KEEP 0x4B454550424954ULL   /* "KEEPBIT"  */
#define SYNTH_TAG_PICK 0x5049434B43484F49ULL /* "PICKCHOI" */
#define SYNTH_GAMMA 0x9E3779B97F4A7C15ULL

SYNTH_FN uint64_t synth_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

SYNTH_FN uint64_t synth_key(uint64_t seed, uint64_t tag) { return synth_mix64(seed ^ tag); }

/* Is the unordered pair {x,y} (x < y) constrained?  dens_q32 in [0, 2^32]. */
SYNTH_FN int synth_present(uint64_t seed, uint32_t n, uint32_t x, uint32_t y, uint64_t dens_q32) {
  uint64_t h = synth_mix64(synth_key(seed, SYNTH_TAG_PRES) ^ synth_mix64((uint64_t)x * n + y));
  return (h >> 32) < dens_q32;
}

/* Per-pair stream key of c_xy, x < y. */
SYNTH_FN uint64_t synth_pair_key(uint64_t seed, uint32_t n, uint32_t x, uint32_t y) {
  return synth_mix64(synth_key(seed, SYNTH_TAG_CELL) ^ synth_mix64((uint64_t)x * n + y));
}

/* The 64-bit word holding cells (a, 4*bq .. 4*bq+3) of the pair with stream key pk. */
SYNTH_FN uint64_t synth_cell_word_pk(uint64_t pk, uint32_t d, uint32_t a, uint32_t bq) {
  uint64_t q = (d + 3u) / 4u;
  return synth_mix64(pk + ((uint64_t)a * q + bq + 1u) * SYNTH_GAMMA);
}

SYNTH_FN uint64_t synth_cell_word(uint64_t seed, uint32_t n, uint32_t d, uint32_t x, uint32_t y,
                                  uint32_t a, uint32_t bq) {
  return synth_cell_word_pk(synth_pair_key(seed, n, x, y), d, a, bq);
}

/* Is (a,b) allowed in rel(c_xy), x < y?  t_q16 in [0, 65536]. */
SYNTH_FN int synth_allowed(uint64_t seed, uint32_t n, uint32_t d, uint32_t x, uint32_t y,
                           uint32_t a, uint32_t b, uint32_t t_q16) {
  uint64_t h = synth_cell_word(seed, n, d, x, y, a, b >> 2);
  uint32_t v = (uint32_t)((h >> (16u * (b & 3u))) & 0xFFFFu);
  return v >= t_q16;
}

/* Row a of rel(c_xy), x < y, as a bitset over b (bit b set iff (a,b) allowed); d <= 64. */
SYNTH_FN uint64_t synth_row(uint64_t seed, uint32_t n, uint32_t d, uint32_t x, uint32_t y,
                            uint32_t a, uint32_t t_q16) {
  uint64_t row = 0;
  uint64_t pk = synth_pair_key(seed, n, x, y);
  for (uint32_t bq = 0; bq * 4u < d; ++bq) {
    uint64_t h = synth_cell_word_pk(pk, d, a, bq);
    for (uint32_t j = 0; j < 4u && bq * 4u + j < d; ++j) {
      uint32_t v = (uint32_t)((h >> (16u * j)) & 0xFFFFu);
      if (v >= t_q16) row |= 1ULL << (bq * 4u + j);
    }
  }
  return row;
}

/* W-rand workload: keep bit (x,a) of a domain state with probability keep_q16/65536. */
SYNTH_FN int synth_keep(uint64_t seed, uint32_t x, uint32_t a, uint32_t keep_q16) {
  uint64_t h = synth_mix64(synth_key(seed, SYNTH_TAG_KEEP) ^ synth_mix64((uint64_t)x * 64u + a));
  return (uint32_t)(h & 0xFFFFu) < keep_q16;
}

/* Seeded choice k in [0, m). */
SYNTH_FN uint64_t synth_pick(uint64_t seed, uint64_t k, uint64_t m) {
  return synth_mix64(synth_key(seed, SYNTH_TAG_PICK) ^ synth_mix64(k)) % m;
}

#endif /* CSP_SYNTH_H */
