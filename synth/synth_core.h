/*
 * synth_core.h — counter-based synthetic read generator.
 *
 * This module is the ONLY code shared by the oracle side and the CUDA side.
 * It holds no arithmetic of the counting method: it draws a random genome and
 * simulated sequencing reads from it. Every random draw is a pure function of
 * (seed, stream, counter) — splitmix64-style mixing — so any read (or any base
 * of any read) can be regenerated independently on the host or the device,
 * bit-identically.
 *
 * Recipe:
 *   genome: G iid uniform bases, base g = "ACGT"[rng(GENOME, g) >> 62]
 *   read i: start ~ U[0, G-L] (rng mod (G-L+1)), strand reverse w.p. 1/2
 *           base j = genome[start+j] (forward) or complement(genome[start+L-1-j])
 *           then, per base, with rng(BASE, i*L+j) = r:
 *             (uint32)r < n_thr            → 'N' (undetermined)
 *             else (uint32)(r>>32) < s_thr → substituted by one of the other 3
 *   thresholds are probabilities × 2^32, rounded, fixed by the host so that
 *   host and device agree exactly (no floating point inside the generator).
 */
#ifndef SYNTH_CORE_H
#define SYNTH_CORE_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

enum { SYNTH_STREAM_GENOME = 1, SYNTH_STREAM_START = 2, SYNTH_STREAM_STRAND = 3,
       SYNTH_STREAM_BASE = 4 };

typedef struct {
  uint64_t seed;
  uint64_t genome_len;   /* G */
  uint64_t read_len;     /* L (all reads have length L) */
  uint64_t n_reads;      /* reads in this batch */
  uint64_t first_read;   /* global index of the batch's first read (sharding) */
  uint32_t n_thr;        /* P(N) × 2^32 */
  uint32_t s_thr;        /* P(substitution) × 2^32 */
} synth_params;

SYNTH_HD uint64_t synth_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

SYNTH_HD uint64_t synth_rng(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return synth_mix64(synth_mix64(seed ^ (stream * 0xD1B54A32D192ED03ull)) + ctr);
}

/* Nucleotide index 0..3 of "ACGT" at genome position g. */
SYNTH_HD uint32_t synth_genome_base(uint64_t seed, uint64_t g) {
  return (uint32_t)(synth_rng(seed, SYNTH_STREAM_GENOME, g) >> 62);
}

/* Nucleotide index 0..3 of "ACGT", or 4 for 'N', of base j of read i
 * (i is the global read index). */
SYNTH_HD uint32_t synth_read_base(const synth_params* p, uint64_t i, uint64_t j) {
  uint64_t span = p->genome_len - p->read_len + 1;
  uint64_t start = synth_rng(p->seed, SYNTH_STREAM_START, i) % span;
  uint32_t rev = (uint32_t)(synth_rng(p->seed, SYNTH_STREAM_STRAND, i) & 1u);
  uint32_t c;
  if (rev)
    c = 3u - synth_genome_base(p->seed, start + p->read_len - 1 - j);
  else
    c = synth_genome_base(p->seed, start + j);
  uint64_t r = synth_rng(p->seed, SYNTH_STREAM_BASE, i * p->read_len + j);
  uint32_t un = (uint32_t)r, us = (uint32_t)(r >> 32);
  if (un < p->n_thr) return 4u;
  if (us < p->s_thr) c = (c + 1u + (us % 3u)) & 3u;
  return c;
}

#endif /* SYNTH_CORE_H */
