// table.cuh — the per-wave k-mer hash table (steps d and e).
//
// PAPER.md:63 (§2.2): "a hash table that implements open addressing";
// Alg. 1; §3.3.1: probe a window of
// adjacent entries with one memory access, lock entries with atomics.
//
// Layout. A canonical k-mer is stored as WP = ceil(k/31)
// "chunks": chunk j = bit 63 set (written flag) | bases [31j, 31j+31) packed
// 2 bits/base MSB-first in bits 61..0 (zero padded). A bucket holds 4 slots:
//     [ 4 × chunk0 (32 B) ][ 4 × u32 count (16 B) | 16 B pad ][ 4 × (WP-1) chunks ]
// so one probe = ONE 32-byte sector load (LDG.256) of the chunk0 words,
// whatever k is (the paper's 128-byte window held fewer entries as k grew,
// PAPER.md:314).
// Claim: CAS(chunk0: 0 → chunk0). The remaining chunks are plain stores;
// every chunk carries its own written flag, so a reader that matched chunk0
// re-reads a chunk until its flag is set — no release fence is needed, and a
// key lives in at most one slot (all threads of a key probe one sequence and
// slots never empty during a wave). Counts are atomicAdd'ed (also by the
// claimer), so their order never matters.
#pragma once
#include "common.cuh"

namespace gerbil {

constexpr uint64_t kFlag = 1ull << 63;
constexpr uint32_t kSlots = 4;  // slots per bucket

__host__ __device__ inline uint32_t chunk_words(uint32_t k) { return (k + 30) / 31; }
__host__ __device__ inline uint64_t table_bucket_bytes(uint32_t k) { return 32 + 32ull * chunk_words(k); }

// standard W-word key (32 bases per word) → WP flagged 31-base chunks
template <int W, int WP>
__device__ __forceinline__ void to_chunks(const uint64_t (&c)[W], uint64_t (&t)[WP]) {
#pragma unroll
  for (int j = 0; j < WP; ++j) {
    const int b = 62 * j, wi = b >> 6, off = b & 63;
    const uint64_t hi = wi < W ? c[wi] : 0ull;
    const uint64_t lo = wi + 1 < W ? c[wi + 1] : 0ull;
    const uint64_t v = off ? ((hi << off) | (lo >> (64 - off))) : hi;
    t[j] = kFlag | (v >> 2);
  }
}

// WP chunks → standard W words (runtime W for the compaction pass)
__device__ __forceinline__ void from_chunks(const uint64_t* t, uint32_t WP, uint64_t* out, uint32_t W) {
  for (uint32_t i = 0; i < W; ++i) out[i] = 0ull;
  for (uint32_t j = 0; j < WP; ++j) {
    const uint64_t p = t[j] << 2;  // 62 payload bits, left-aligned
    const uint32_t b = 62 * j, wi = b >> 6, off = b & 63;
    out[wi] |= p >> off;
    if (off > 2 && wi + 1 < W) out[wi + 1] |= p << (64 - off);
  }
}

struct Bucket {
  uint64_t* c0;     // [4] first chunks
  uint32_t* cnt;    // [4]
  uint64_t* rest;   // [4][WP-1]
};

__device__ __forceinline__ Bucket bucket_at(unsigned char* table, uint64_t b, uint32_t WP) {
  unsigned char* p = table + b * (32 + 32ull * WP);
  return Bucket{reinterpret_cast<uint64_t*>(p), reinterpret_cast<uint32_t*>(p + 32),
                reinterpret_cast<uint64_t*>(p + 64)};
}

__device__ __forceinline__ uint64_t bucket_of(uint64_t h, uint64_t nb) { return ((h >> 32) * nb) >> 32; }

// one 32-byte sector: the 4 chunk0 words of a bucket (served by L2)
__device__ __forceinline__ void ld_c0(const uint64_t* p, uint64_t (&w)[4]) {
  asm volatile("ld.global.relaxed.gpu.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
               : "l"(p)
               : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.relaxed.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// chunks 1..WP-1 of slot s equal t[1..]? Waits for chunks not yet written.
template <int WP>
__device__ __forceinline__ bool rest_equal(const uint64_t* rest, int s, const uint64_t (&t)[WP]) {
  bool eq = true;
#pragma unroll
  for (int j = 1; j < WP; ++j) {
    const uint64_t* p = rest + s * (WP - 1) + (j - 1);
    uint64_t v = ld_relaxed_u64(p);
    for (uint32_t spins = 0; !(v & kFlag); ++spins) {
      if (spins > (1u << 24)) __trap();  // watchdog: a lost publish must fail, not hang
      v = ld_relaxed_u64(p);
    }
    eq &= (v == t[j]);
  }
  return eq;
}

// Alg. 1 with bucketised linear probing. w holds the prefetched chunk0 words
// of bucket b. Returns buckets probed (>= 1), or 0 after θ buckets (→
// emergency mechanism).
template <int WP>
__device__ __forceinline__ uint32_t table_insert(unsigned char* table, uint64_t nb, uint32_t theta,
                                                 const uint64_t (&t)[WP], uint64_t b, uint64_t (&w)[4]) {
  for (uint32_t probe = 1; probe <= theta; ++probe) {
    const Bucket bk = bucket_at(table, b, WP);
    if (probe > 1) ld_c0(bk.c0, w);
    // matching k-mer → count + 1
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (w[s] == t[0] && rest_equal<WP>(bk.rest, s, t)) {
        atomicAdd(bk.cnt + s, 1u);
        return probe;
      }
    }
    // empty entry → claim it: (x, 1)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (w[s] == 0ull) {
        const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long*>(bk.c0 + s), 0ull,
                                       (unsigned long long)t[0]);
        if (old == 0ull) {
#pragma unroll
          for (int j = 1; j < WP; ++j) bk.rest[s * (WP - 1) + (j - 1)] = t[j];
          atomicAdd(bk.cnt + s, 1u);
          return probe;
        }
        if (old == t[0] && rest_equal<WP>(bk.rest, s, t)) {  // lost the race to an equal key
          atomicAdd(bk.cnt + s, 1u);
          return probe;
        }
      }
    }
    // entries locked by other k-mers → next trial
    b = (b + 1 == nb) ? 0 : b + 1;
  }
  return 0;
}

}  // namespace gerbil
