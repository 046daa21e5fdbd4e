// table_inline.cuh — "inline" table kind for k <= 46.
//
// When the canonical k-mer fits two 31-base chunks with at least 32 unused
// low bits in the second (k <= 46), a slot is 16 bytes:
//     w0 = chunk0 (bit 63 set)    w1 = chunk1 (bit 63 set; absent for k <= 31) | count (low 32 bits)
// A bucket is 4 slots = 64 B (two 32-byte sectors, fetched together).
// Alg. 1: a matching k-mer is counted with one RED on the
// embedded count; an empty slot is claimed with ONE 128-bit CAS that writes
// the whole key and count = 1 atomically — no publish step, no waiting, and
// (no deletions, one probe order per key) a key lives in at most one slot.
#pragma once
#include "table.cuh"

namespace gerbil {

__host__ __device__ inline bool table_inline(uint32_t k) { return k <= 46; }
constexpr uint64_t kInlineBucketBytes = 64;

struct Slot16 {
  uint64_t w0, w1;
};

__device__ __forceinline__ void ld_bucket_inline(const uint64_t* p, uint64_t (&w)[8]) {
  asm volatile("ld.global.relaxed.gpu.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
               : "l"(p)
               : "memory");
  asm volatile("ld.global.relaxed.gpu.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[4]), "=l"(w[5]), "=l"(w[6]), "=l"(w[7])
               : "l"(p + 4)
               : "memory");
}

__device__ __forceinline__ void ld_slot16(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.global.relaxed.gpu.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// 128-bit CAS: returns the previous 16 bytes
__device__ __forceinline__ Slot16 cas128(uint64_t* p, uint64_t c0, uint64_t c1, uint64_t s0, uint64_t s1) {
  Slot16 r;
  asm volatile(
      "{ .reg .b128 t, c, s;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 s, {%4, %5};\n\t"
      "atom.global.cas.b128 t, [%6], c, s;\n\t"
      "mov.b128 {%0, %1}, t; }"
      : "=l"(r.w0), "=l"(r.w1)
      : "l"(c0), "l"(c1), "l"(s0), "l"(s1), "l"(p)
      : "memory");
  return r;
}

__device__ __forceinline__ uint32_t* inline_count(uint64_t* slot) {
  return reinterpret_cast<uint32_t*>(slot + 1);  // low 32 bits of w1 (little endian)
}

__device__ __forceinline__ bool inline_match(uint64_t w0, uint64_t w1, uint64_t c0, uint64_t c1) {
  return w0 == c0 && (w1 >> 32) == (c1 >> 32);
}

// The 256-bit loads are not promised to be single-copy atomic: a slot could be
// seen with the new w0 and the old (zero) w1. For k > 31 a complete w1 has its
// flag set, so such a half-written view is recognised and re-read.
template <bool TWO>
__device__ __forceinline__ void settle(uint64_t* slot, uint64_t& w0, uint64_t& w1) {
  if (TWO) {
    while (w0 != 0ull && !(w1 >> 63)) ld_slot16(slot, w0, w1);
  }
}

// Returns buckets probed (>= 1), or 0 after θ buckets (→ emergency mechanism).
template <bool TWO>
__device__ __forceinline__ uint32_t inline_insert(unsigned char* table, uint64_t nb, uint32_t theta,
                                                  uint64_t c0, uint64_t c1, uint64_t b, uint64_t (&w)[8]) {
  for (uint32_t probe = 1; probe <= theta; ++probe) {
    uint64_t* bk = reinterpret_cast<uint64_t*>(table + b * kInlineBucketBytes);
    if (probe > 1) ld_bucket_inline(bk, w);
#pragma unroll
    for (int s = 0; s < 4; ++s) settle<TWO>(bk + 2 * s, w[2 * s], w[2 * s + 1]);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (inline_match(w[2 * s], w[2 * s + 1], c0, c1)) {  // matching k-mer → count + 1
        atomicAdd(inline_count(bk + 2 * s), 1u);
        return probe;
      }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (w[2 * s] == 0ull) {  // empty entry → (x, 1)
        const Slot16 old = cas128(bk + 2 * s, 0ull, 0ull, c0, c1 | 1ull);
        if (old.w0 == 0ull) return probe;
        if (inline_match(old.w0, old.w1, c0, c1)) {
          atomicAdd(inline_count(bk + 2 * s), 1u);
          return probe;
        }
      }
    }
    b = (b + 1 == nb) ? 0 : b + 1;  // entries locked by other k-mers → next trial
  }
  return 0;
}

}  // namespace gerbil
