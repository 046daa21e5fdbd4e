// common.cuh — device helpers of the Gerbil counting path (sm_100a).
//
// Packed layouts are defined in include/gerbil.h: 2-bit codes A=0,C=1,G=2,T=3
// (App. C), first base in the most significant bits of a u64
// word; N-mask and read-start bitmaps are MSB-first too.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gerbil {

constexpr int kMaxW = 15;         // k <= 479 → W = ceil(k/32) <= 15
constexpr uint32_t kSlotsPerBucket = 4;  // table.cuh bucket layout
constexpr uint32_t kReady = 0x80000000u;
constexpr uint32_t kFpMask = 0x7fffffffu;
constexpr int kNwinBits = 11;     // super-mer descriptor: pos << 11 | (nwin-1)
constexpr uint32_t kTile = 2048;  // window positions per step-(b) tile (= max super-mer windows)

__host__ __device__ inline uint32_t key_words(uint32_t k) { return (k + 31) / 32; }


__device__ __forceinline__ uint64_t fmix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h;
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// Reverse the order of the 32 2-bit groups of a word.
__device__ __forceinline__ uint64_t rev_pairs(uint64_t v) {
  v = __brevll(v);
  return ((v >> 1) & 0x5555555555555555ull) | ((v & 0x5555555555555555ull) << 1);
}

// Bases [q, q+k) of a packed stream as W left-aligned words, pad bits zero.
// Reads only the words the k-mer touches (never past the stream end).
template <int W>
__device__ __forceinline__ void extract_kmer(const uint64_t* __restrict__ codes, uint64_t q,
                                             uint32_t k, uint64_t (&x)[W]) {
  const uint64_t w0 = q >> 5;
  const uint32_t s = (uint32_t)(q & 31) * 2;
  const uint32_t need = ((uint32_t)(q & 31) + k + 31) >> 5;  // words touched
  uint64_t a[W + 1];
#pragma unroll
  for (int i = 0; i <= W; ++i) a[i] = (i < (int)need) ? __ldg(codes + w0 + i) : 0ull;
#pragma unroll
  for (int i = 0; i < W; ++i) x[i] = s ? ((a[i] << s) | (a[i + 1] >> (64 - s))) : a[i];
  const uint32_t tail = 2 * k - 64 * (W - 1);  // meaningful bits of the last word, 1..64
  if (tail < 64) x[W - 1] &= ~0ull << (64 - tail);
}

// Reverse complement (§2.4.2): reverse the 2k-bit string in
// 2-bit units and complement each base (A<->T = 00<->11, C<->G = 01<->10).
template <int W>
__device__ __forceinline__ void reverse_complement(const uint64_t (&x)[W], uint32_t k,
                                                   uint64_t (&r)[W]) {
  uint64_t y[W];
#pragma unroll
  for (int i = 0; i < W; ++i) y[i] = rev_pairs(~x[W - 1 - i]);
  const uint32_t pad = 64 * W - 2 * k;  // 0..62; the complemented pad sits on top of y[0]
#pragma unroll
  for (int i = 0; i < W; ++i) {
    uint64_t nxt = (i + 1 < W) ? y[i + 1] : 0ull;
    r[i] = pad ? ((y[i] << pad) | (nxt >> (64 - pad))) : y[i];
  }
}

// Lexicographic (A<C<G<T) comparison of left-aligned word arrays.
template <int W>
__device__ __forceinline__ bool key_less(const uint64_t (&a)[W], const uint64_t (&b)[W]) {
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}

// Table hash of a canonical key: multiply-xorshift over the words (one 64-bit
// multiply per word plus one finaliser). Only its distribution matters — it is
// not observable in the output (reading Q11).
template <int W>
__device__ __forceinline__ uint64_t key_hash(const uint64_t (&c)[W]) {
  uint64_t h = c[0] * 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int i = 1; i < W; ++i) h = (h ^ (h >> 29)) + c[i] * 0xC2B2AE3D27D4EB4Full;
  h ^= h >> 32;
  h *= 0xD6E8FEB86659FD93ull;
  h ^= h >> 32;
  return h;
}

// ---- memory-model helpers (gpu scope; L1 is not coherent) -----------------
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// 16-byte load served by L2 (.cg: not cached in the incoherent L1).
__device__ __forceinline__ uint4 ld_cg_v4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

}  // namespace gerbil
