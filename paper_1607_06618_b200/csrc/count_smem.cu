// count_smem.cu — steps (d)+(e) for small bins: one shared-memory hash table
// per bin, owned by one warp.
//
// The paper counts each temporary file in its own hash table and outputs the
// table when the file is done (§2.3.2 steps 2-3; Alg. 1,
// PAPER.md:65-84). Here a "file" is a bin small enough that its distinct
// k-mers fit a table in one warp's share of shared memory (DESIGN.md "Kernel
// (d) smem"). Minimizer bins of m >= ~12 with ~10^5-10^6 bins are that small,
// so the whole counting phase runs without a single global atomic per k-mer:
//
//  - a warp walks a static round-robin share of the bin list; the descriptors
//    and packed words of the next chunk of 32 super-mers are in flight
//    (registers / cp.async into the other half of a double-buffered stage)
//    while the current chunk is counted — across bin boundaries too;
//  - lanes take consecutive windows (32 per round), extract from the stage,
//    canonicalise c = min(x, rc x) and hash;
//  - insertion into the warp's private table ("lock entries
//    with atomics", here shared-memory atomics of one warp): every pending lane
//    probes linearly (plain shared loads) until it sees its key or an empty
//    slot; after a __syncwarp (all probes of the step done before any write) a
//    lane that found its key adds 1 to the count (atomicAdd) and is done; a
//    lane at an empty slot claims it with atomicCAS(count: 0 → 1) and, if it
//    won, writes its key and appends the slot to the warp's list of occupied
//    slots; losers re-probe from that slot in the next step (after a
//    __syncwarp the winner's key is complete), where a same-key loser finds
//    it. A key lives in at most one slot: a slot is claimed once and probes
//    see only complete keys;
//  - when the bin is done its occupied-slot list is compacted: counts >=
//    min_count are written as (W key words, u32 count) at a range reserved
//    with one global atomic per bin (reading Q5), Σcount and
//    distinct are accumulated, and the listed slots are cleared for the next
//    bin (the scan touches the bin's distinct k-mers, not its table).
//
// A bin whose distinct k-mers exceed max_fill (a skewed bin the host's ρ̂
// estimate did not predict) is abandoned without output and its list index
// recorded; the host counts it in the L2 wave path instead (api.cu), so the
// result stays exact.
#include <cstdio>

#include "common.cuh"
#include "count_inline.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

__host__ __device__ inline bool smem_pack(uint32_t k) { return k <= 48; }

// Slot layouts. PACK (W == 1, or W == 2 with k <= 48): 16 bytes
//   {c[0], c[1] (top 32 bits; zero for W == 1) | count (low 32 bits)};
// otherwise keys u64[cap][W] followed by counts u32[cap]. count == 0 ⇔ empty.
template <int W, bool PACK>
struct SmemTable {
  unsigned char* base;
  uint32_t cap;
  __device__ __forceinline__ ulonglong2* slots() const { return reinterpret_cast<ulonglong2*>(base); }
  __device__ __forceinline__ uint64_t* keys() const { return reinterpret_cast<uint64_t*>(base); }
  __device__ __forceinline__ uint32_t* counts() const {
    return reinterpret_cast<uint32_t*>(base + (size_t)cap * W * 8);
  }
  // count of slot s (0 = empty) and whether it holds key c
  __device__ __forceinline__ uint32_t probe(uint32_t s, const uint64_t (&c)[W], bool& eq) const {
    if (PACK) {
      const ulonglong2 v = slots()[s];
      const uint64_t khi = W == 2 ? c[W - 1] : 0ull;
      eq = v.x == c[0] && (v.y & 0xffffffff00000000ull) == khi;
      return (uint32_t)v.y;
    } else {
      const uint32_t n = counts()[s];
      bool e = true;
#pragma unroll
      for (int v = 0; v < W; ++v) e = e && keys()[(size_t)s * W + v] == c[v];
      eq = e;
      return n;
    }
  }
  __device__ __forceinline__ void put(uint32_t s, const uint64_t (&c)[W], uint32_t n) const {
    if (PACK) {
      const uint64_t khi = W == 2 ? c[W - 1] : 0ull;
      slots()[s] = make_ulonglong2(c[0], khi | n);
    } else {
#pragma unroll
      for (int v = 0; v < W; ++v) keys()[(size_t)s * W + v] = c[v];
      counts()[s] = n;
    }
  }
  __device__ __forceinline__ void set_count(uint32_t s, uint32_t n) const {
    if (PACK) reinterpret_cast<uint32_t*>(slots() + s)[2] = n;  // low half of .y (little endian)
    else counts()[s] = n;
  }
  __device__ __forceinline__ uint32_t count(uint32_t s) const {
    return PACK ? (uint32_t)slots()[s].y : counts()[s];
  }
  __device__ __forceinline__ void key(uint32_t s, uint64_t (&c)[W]) const {
    if (PACK) {
      const ulonglong2 v = slots()[s];
      c[0] = v.x;
      if (W == 2) c[W - 1] = v.y & 0xffffffff00000000ull;
    } else {
#pragma unroll
      for (int v = 0; v < W; ++v) c[v] = keys()[(size_t)s * W + v];
    }
  }
  __device__ __forceinline__ void clear(uint32_t s) const {
    if (PACK) slots()[s] = make_ulonglong2(0ull, 0ull);
    else counts()[s] = 0u;
  }
  __device__ __forceinline__ uint32_t* count_ptr(uint32_t s) const {
    return PACK ? reinterpret_cast<uint32_t*>(slots() + s) + 2 : counts() + s;  // low half of .y
  }
  // the key of a slot this lane just claimed (its count is already set)
  __device__ __forceinline__ void put_key(uint32_t s, const uint64_t (&c)[W]) const {
    if (PACK) {
      uint64_t* q = reinterpret_cast<uint64_t*>(slots() + s);
      q[0] = c[0];
      if (W == 2) reinterpret_cast<uint32_t*>(q)[3] = (uint32_t)(c[W - 1] >> 32);  // high half of .y
    } else {
#pragma unroll
      for (int v = 0; v < W; ++v) keys()[(size_t)s * W + v] = c[v];
    }
  }
};

// k-mer of k bases at base offset o of a staged stream (S words), W left-aligned words
template <int W, int S>
__device__ __forceinline__ void extract_stage(const uint64_t* s, uint32_t o, uint32_t k, uint64_t (&x)[W]) {
  const uint32_t w0 = o >> 5, sh = (o & 31) * 2;
  uint64_t a[W + 1];
#pragma unroll
  for (int i = 0; i <= W; ++i) a[i] = (w0 + i < (uint32_t)S) ? s[w0 + i] : 0ull;
#pragma unroll
  for (int i = 0; i < W; ++i) x[i] = sh ? ((a[i] << sh) | (a[i + 1] >> (64 - sh))) : a[i];
  const uint32_t tail = 2 * k - 64 * (W - 1);
  if (tail < 64) x[W - 1] &= ~0ull << (64 - tail);
}

// Same without bounds checks, from 32-bit funnel shifts: words past the k-mer may be
// read (they stay inside the warp's shared memory: rc stage and table follow the
// stages) but only feed bits that the tail mask clears. The stream's 32-bit units in
// order are hi(w0), lo(w0), hi(w1), ...; the k-mer starts in unit 2*(o/32) + (o%32)/16.
template <int W>
__device__ __forceinline__ void extract_fast(const uint64_t* s, uint32_t o, uint64_t tmask, uint64_t (&x)[W]) {
  const uint64_t* p = s + (o >> 5);
  const bool odd = (o & 16u) != 0;   // starts in the low half of word o/32
  const uint32_t r = (o & 15u) * 2;  // bit shift inside the 32-bit unit
  uint32_t u[2 * W + 2];
#pragma unroll
  for (int i = 0; i <= W; ++i) {
    const uint64_t a = p[i];
    u[2 * i] = (uint32_t)(a >> 32);
    u[2 * i + 1] = (uint32_t)a;
  }
  uint32_t v[2 * W + 1];
#pragma unroll
  for (int n = 0; n <= 2 * W; ++n) v[n] = odd ? u[n + 1] : u[n];
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const uint32_t hi = __funnelshift_l(v[2 * i + 1], v[2 * i], r);
    const uint32_t lo = __funnelshift_l(v[2 * i + 2], v[2 * i + 1], r);
    x[i] = ((uint64_t)hi << 32) | lo;
  }
  x[W - 1] &= tmask;
}

// 32-bit hash of a canonical key for the small shared-memory tables (not observable)
template <int W>
__device__ __forceinline__ uint32_t smem_hash(const uint64_t (&c)[W]) {
  uint32_t x = (uint32_t)(c[0] >> 32) * 0x9E3779B1u ^ (uint32_t)c[0] * 0x85EBCA77u;
#pragma unroll
  for (int v = 1; v < W; ++v) x ^= (uint32_t)(c[v] >> 32) * 0xC2B2AE3Du ^ (uint32_t)c[v] * 0x27D4EB2Fu;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  return x;
}


#ifndef GERBIL_SMEM_RCSTAGE
#define GERBIL_SMEM_RCSTAGE 0
#endif
constexpr bool kRcStage = GERBIL_SMEM_RCSTAGE != 0;  // rc stream staged per chunk (else bit reversal)
__host__ __device__ constexpr int smem_stage_words(bool pack) { return pack ? 4 : kStageWords; }
__host__ __device__ constexpr uint32_t smem_overhead(int S) {
  return 2u * 32u * S * 8u /* forward, double-buffered */ + (kRcStage ? 32u * S * 8u : 0u) /* reverse complement */;
}

// Per-warp shared memory: [fwd stage 2][32][S] u64 | [rc stage][32][S] u64 |
// table (cap slots) | occupied-slot list u16[cap]
template <int W, bool PACK>
__global__ void __launch_bounds__(kSmemMaxWarps * 32, 1) count_smem_kernel(SmemCountArgs a, uint32_t warp_bytes) {
  constexpr int S = smem_stage_words(PACK);
  extern __shared__ __align__(16) unsigned char s_raw[];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  unsigned char* wbase = s_raw + (size_t)wib * warp_bytes;
  uint64_t* stage = reinterpret_cast<uint64_t*>(wbase);              // [2][32 * S]
  uint64_t* rcs = stage + 2 * 32 * S;                                // [32 * S]
  unsigned char* tab = reinterpret_cast<unsigned char*>(rcs + (kRcStage ? 32 * S : 0));
  const uint32_t cap = a.cap;
  const uint32_t tail = 2 * a.k - 64 * (W - 1);  // meaningful bits of the last key word
  const uint64_t tmask = tail < 64 ? ~0ull << (64 - tail) : ~0ull;
  SmemTable<W, PACK> T{tab, cap};
  uint16_t* occ = reinterpret_cast<uint16_t*>(tab + (size_t)cap * (PACK ? 16u : 8u * W + 4u));
  for (uint32_t s = lane; s < cap; s += 32) T.clear(s);
  __syncwarp();

  // ---- static round-robin walk over the bin list, in chunks of 32 descriptors
  const uint32_t G = gridDim.x * (blockDim.x >> 5);
  uint32_t wi = blockIdx.x * (blockDim.x >> 5) + wib;  // list entry of the walker's bin
  uint64_t wd0 = 0, wd1 = 0, nd0 = 0, nd1 = 0, wc = 0;
  auto load_range = [&](uint32_t i, uint64_t& r0, uint64_t& r1) {
    r0 = r1 = 0;
    if (i < a.n_list) {
      r0 = __ldg(a.range + 2 * (size_t)i);
      r1 = __ldg(a.range + 2 * (size_t)i + 1);
    }
  };
  load_range(wi, wd0, wd1);
  load_range(wi + G, nd0, nd1);
  // item flags: 1 = first chunk of its bin, 2 = last chunk, 4 = valid; bits 8.. = the bin's table slots
  auto next_item = [&](uint64_t& d, uint32_t& li) -> uint32_t {
    li = wi;
    d = ~0ull;
    if (wi >= a.n_list) return 0u;
    const uint64_t e = wd1 & kRangeEndMask;
    const uint64_t b0 = wd0 + wc * 32;
    uint32_t f = 4u | (wc == 0 ? 1u : 0u) | (b0 + 32 >= e ? 2u : 0u);
    // slots for this bin: distinct <= windows, so a table of windows + 1/4 + 32 never fills
    f |= ((a.dbg & 8u) ? cap : smem_bin_slots(wd1 >> kRangeWinShift, cap)) << 8;
    if (b0 + lane < e) d = __ldg(a.desc + b0 + lane);
    if (f & 2u) {
      wi += G;
      wd0 = nd0;
      wd1 = nd1;
      wc = 0;
      load_range(wi + G, nd0, nd1);
    } else {
      ++wc;
    }
    return f;
  };
  auto issue_words = [&](uint64_t d, uint64_t* dst) {  // one cp.async group per chunk
    uint32_t nwords = 0;
    const uint64_t* src = a.codes;
    if (d != ~0ull) {
      const uint64_t p = d >> kNwinBits;
      const uint32_t n = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
      nwords = ((uint32_t)(p & 31) + n + a.k - 1 + 31) >> 5;
      src += p >> 5;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) cp_async8(dst + s, src + (s < (int)nwords ? s : 0), s < (int)nwords);
    cp_async_commit();
  };

  uint64_t d0, d1, d2;
  uint32_t l0, l1, l2;
  uint32_t f0 = next_item(d0, l0);
  issue_words(d0, stage + lane * S);
  uint32_t f1 = next_item(d1, l1);
  uint32_t buf = 0;
  uint32_t n_distinct = 0;  // warp-uniform: distinct k-mers of the current bin so far
  bool abandoned = false;   // warp-uniform
  unsigned long long acc_sum = 0, acc_dist = 0;  // per lane, flushed at the end

  while (f0 & 4u) {
    issue_words(d1, stage + (buf ^ 1) * 32 * S + lane * S);
    const uint32_t f2 = next_item(d2, l2);
    const uint32_t cb = f0 >> 8;  // this bin's table slots
    const uint32_t fill = cb == cap ? a.max_fill : cb;
    if (f0 & 1u) {
      n_distinct = 0;
      abandoned = false;
    }
    const uint64_t* stg = stage + buf * 32 * S;
    const uint64_t pos = d0 == ~0ull ? 0ull : d0 >> kNwinBits;
    const uint32_t nw = d0 == ~0ull ? 0u : (uint32_t)(d0 & ((1u << kNwinBits) - 1)) + 1;
    const uint32_t o = (uint32_t)(pos & 31), L = nw + a.k - 1;  // stage offset, super-mer bases
    const bool staged = o + L <= 32u * S;
    cp_async_wait<1>();
    __syncwarp();

    if (!abandoned) {
      const uint32_t incl = warp_incl_scan_u32(nw), excl = incl - nw;
      const uint32_t total = __shfl_sync(kFull, incl, 31);
      const uint32_t stage_mask = __ballot_sync(kFull, staged);
      // reverse-complement stream of every staged super-mer: rc base t = comp(fwd base o+L-1-t)
      const bool rcst = kRcStage && a.canonical && !(a.dbg & 1u);
      if (rcst && staged && nw) {
        const uint64_t* f = stg + lane * S;
        uint64_t* r = rcs + lane * S;
        const uint32_t nr = (L + 31) >> 5;
        for (uint32_t u = 0; u < nr; ++u) {
          const int e = (int)(o + L) - 32 * (int)u;  // forward bases [e-32, e) → rc word u
          const int s0 = e - 32;
          uint64_t v;
          if (s0 >= 0) {
            const uint32_t w0 = (uint32_t)s0 >> 5, sh = ((uint32_t)s0 & 31) * 2;
            const uint64_t hi = f[w0], lo = (w0 + 1 < (uint32_t)S) ? f[w0 + 1] : 0ull;
            v = sh ? ((hi << sh) | (lo >> (64 - sh))) : hi;
          } else {
            v = f[0] >> (2 * (uint32_t)(-s0));
          }
          r[u] = rev_pairs(~v);
        }
      }
      __syncwarp();
      // window i → super-mer (lane) j: lanes hold consecutive window ranges [excl, incl)
      // (empty lanes only at the end of a bin's last chunk), so j = #super-mers starting at
      // or before i, minus 1 — the round's start bits come from one OR-reduction
      uint32_t n_before = 0;  // super-mers starting before the current round
      for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t i = base + lane;
        const bool act = i < total;
        const uint32_t rel = excl - base;
        const uint32_t starts = __reduce_or_sync(kFull, (nw && rel < 32u) ? 1u << rel : 0u);
        int j = (int)(n_before + __popc(starts & ((2u << lane) - 1u))) - 1;
        n_before += __popc(starts);
        if (!act) j = 31;
        const uint64_t pj = __shfl_sync(kFull, pos, j);
        const uint32_t ej = __shfl_sync(kFull, excl, j);
        const uint32_t Lj = __shfl_sync(kFull, L, j);
        const uint32_t q = act ? i - ej : 0u;  // window of super-mer j
        uint64_t c[W];
        if ((stage_mask >> j) & 1u) {
          extract_fast<W>(stg + j * S, (uint32_t)(pj & 31) + q, tmask, c);
          if (rcst) {  // warp-uniform
            uint64_t r[W];
            extract_fast<W>(rcs + j * S, act ? Lj - q - a.k : 0u, tmask, r);
            if (key_less<W>(r, c)) {
#pragma unroll
              for (int v = 0; v < W; ++v) c[v] = r[v];
            }
          } else if (a.canonical) {  // no rc stage: reverse complement by bit reversal
            uint64_t r[W];
            reverse_complement<W>(c, a.k, r);
            if (key_less<W>(r, c)) {
#pragma unroll
              for (int v = 0; v < W; ++v) c[v] = r[v];
            }
          }
        } else {
          extract_kmer<W>(a.codes, act ? pj + q : 0ull, a.k, c);
          if (a.canonical) {
            uint64_t r[W];
            reverse_complement<W>(c, a.k, r);
            if (key_less<W>(r, c)) {
#pragma unroll
              for (int v = 0; v < W; ++v) c[v] = r[v];
            }
          }
        }
        uint32_t h = (uint32_t)(((uint64_t)smem_hash<W>(c) * cb) >> 32);

        // insertion into the warp's private table (header). A table never fills
        // (abandonment at max_fill <= cap - 32, or windows < slots), so probing ends.
        bool pend = act;
        for (;;) {
          bool found = false;
          if (pend) {
            for (;;) {
              bool eq;
              const uint32_t cnt = T.probe(h, c, eq);
              if (cnt == 0u) break;
              if (eq) {
                found = true;
                break;
              }
              h = (h + 1 == cb) ? 0u : h + 1;
            }
          }
          __syncwarp();  // every probe of this step before any write
          bool won = false;
          if (pend) {
            if (found) {
              atomicAdd(T.count_ptr(h), 1u);
              pend = false;
            } else if (atomicCAS(T.count_ptr(h), 0u, 1u) == 0u) {
              T.put_key(h, c);
              won = true;
              pend = false;
            }
          }
          const uint32_t wm = __ballot_sync(kFull, won);
          if (won) occ[n_distinct + __popc(wm & ((1u << lane) - 1u))] = (uint16_t)h;
          n_distinct += __popc(wm);
          const bool more = __any_sync(kFull, pend);
          __syncwarp();  // claimed keys complete before anyone probes again
          if (!more) break;
        }
        if (n_distinct > fill) abandoned = true;
        if (abandoned) break;
      }
    }

    if (f0 & 2u) {  // last chunk of the bin: output or abandon; clear the occupied slots
      __syncwarp();
      if (!abandoned) {
        uint32_t keep = n_distinct;  // min_count 1: every occupied slot is output
        if (a.min_count > 1) {
          keep = 0;
          for (uint32_t i = lane; i < n_distinct; i += 32) keep += T.count(occ[i]) >= a.min_count ? 1u : 0u;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) keep += __shfl_xor_sync(kFull, keep, off);
        }
        unsigned long long off = 0;
        if (lane == 0 && keep) off = atomicAdd(a.out_n, (unsigned long long)keep);
        off = __shfl_sync(kFull, off, 0);
        for (uint32_t i0 = 0; i0 < n_distinct; i0 += 32) {
          const uint32_t i = i0 + lane;
          const uint32_t s = i < n_distinct ? occ[i] : 0u;
          const uint32_t n = i < n_distinct ? T.count(s) : 0u;
          const bool kp = n >= a.min_count && n != 0u;
          const uint32_t km = __ballot_sync(kFull, kp);
          acc_sum += n;
          if (kp) {
            const unsigned long long oi = off + __popc(km & ((1u << lane) - 1u));
            if (oi < a.out_cap) {
              uint64_t c[W];
              T.key(s, c);
#pragma unroll
              for (int v = 0; v < W; ++v) a.out_keys[oi * W + v] = c[v];
              a.out_counts[oi] = n;
            }
          }
          off += __popc(km);
          if (i < n_distinct) T.clear(s);
        }
        acc_dist += lane == 0 ? n_distinct : 0u;
      } else {
        for (uint32_t i = lane; i < n_distinct; i += 32) T.clear(occ[i]);
        if (lane == 0) {
          const unsigned long long e = atomicAdd(a.n_failed, 1ull);
          a.failed[2 * e] = a.range[2 * (size_t)l0];  // the bin's range entry, for the L2 recount
          a.failed[2 * e + 1] = a.range[2 * (size_t)l0 + 1];
        }
      }
      __syncwarp();
    }

    __syncwarp();  // the stage half just read is refilled next iteration
    f0 = f1;
    d0 = d1;
    l0 = l1;
    f1 = f2;
    d1 = d2;
    l1 = l2;
    buf ^= 1;
  }
  cp_async_wait<0>();
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    acc_sum += __shfl_xor_sync(kFull, acc_sum, off);
    acc_dist += __shfl_xor_sync(kFull, acc_dist, off);
  }
  if (lane == 0) {
    if (acc_sum) atomicAdd(a.sum_counts, acc_sum);
    if (acc_dist) atomicAdd(a.distinct, acc_dist);
  }
}

// desc ranges [r0, r1) of the listed bins → contiguous dst from dst_off[i]; a warp per range
__global__ void gather_ranges_kernel(const uint64_t* __restrict__ src, const unsigned long long* __restrict__ ranges,
                                     const unsigned long long* __restrict__ dst_off, uint32_t n,
                                     uint64_t* __restrict__ dst) {
  const uint32_t lane = lane_id();
  const uint32_t G = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += G) {
    const uint64_t r0 = ranges[2 * (size_t)i], r1 = ranges[2 * (size_t)i + 1], o = dst_off[i];
    for (uint64_t j = lane; j < r1 - r0; j += 32) dst[o + j] = src[r0 + j];
  }
}

template <int W, bool PACK>
cudaError_t launch_smem(const SmemCountArgs& a, int sms, cudaStream_t st) {
  const int warps = a.warps ? a.warps : smem_count_warps(a.k);
  const uint32_t wb = smem_warp_bytes(a.k, a.cap);
  SmemCountArgs b = a;
  if (const char* e = getenv("GERBIL_SMEM_DBG")) b.dbg = (uint32_t)atoi(e);
  const size_t dyn = (size_t)warps * wb;
  cudaError_t e = cudaFuncSetAttribute(count_smem_kernel<W, PACK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn);
  if (e != cudaSuccess) return e;
  uint64_t grid = (uint64_t)sms;
  const uint64_t need = (a.n_list + warps - 1) / warps;
  if (grid > need) grid = need;
  if (grid == 0) return cudaSuccess;
  count_smem_kernel<W, PACK><<<(unsigned)grid, warps * 32, dyn, st>>>(b, wb);
  return cudaGetLastError();
}

}  // namespace

// Warps per CTA (one CTA per SM): more warps hide more latency (the insert chain is a
// string of dependent shared-memory round trips) but split the shared memory into
// smaller tables. 16 for the 17-byte slots of k <= 48, 8 up to W = 3, else 4.
int smem_count_warps(uint32_t k) {
  static const int env = [] {
    const char* e = getenv("GERBIL_SMEM_WARPS");
    return (e && *e) ? atoi(e) : 0;
  }();
  int v = env ? env : (smem_pack(k) ? 16 : (key_words(k) <= 3 ? 8 : 4));
  return v < 1 ? 1 : (v > kSmemMaxWarps ? kSmemMaxWarps : v);
}

uint32_t smem_slot_bytes(uint32_t k) { return (smem_pack(k) ? 16u : 8u * key_words(k) + 4u) + 2u /* list */; }

uint32_t smem_warp_bytes(uint32_t k, uint32_t cap) {
  return (smem_overhead(smem_stage_words(smem_pack(k))) + cap * smem_slot_bytes(k) + 15u) & ~15u;
}

uint32_t smem_table_slots(uint32_t k, size_t smem_per_block, int warps_in) {
  const int warps = warps_in ? warps_in : smem_count_warps(k);
  const size_t per_warp = smem_per_block / warps;
  const uint32_t ovh = smem_overhead(smem_stage_words(smem_pack(k)));
  if (per_warp <= ovh + 64u * 16u) return 0;
  uint32_t cap = (uint32_t)((per_warp - ovh) / smem_slot_bytes(k));
  cap &= ~31u;
  while (cap && smem_warp_bytes(k, cap) * (size_t)warps > smem_per_block) cap -= 32;
  return cap;
}

cudaError_t launch_gather_ranges(const uint64_t* src, const unsigned long long* ranges,
                                 const unsigned long long* dst_off, uint32_t n, uint64_t* dst, int sms,
                                 cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  uint64_t grid = (n + 7) / 8;
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  gather_ranges_kernel<<<(unsigned)grid, 256, 0, st>>>(src, ranges, dst_off, n, dst);
  return cudaGetLastError();
}

// Device-side bin plan (single rank, many bins): per bin with super-mers, either an
// entry of the shared-memory list (predicted to fit: windows <= thr) or a rest triple
// (first descriptor, end descriptor, windows) for the L2 wave tables.
__global__ void __launch_bounds__(256) plan_bins_kernel(PlanBinsArgs a) {
  // block-aggregated: list positions with one atomic per block iteration and list; the window
  // sums once per warp at the end (round 2: per-warp atomics on five hot counters, 0.57 ms at
  // 4M bins, serialised in L2)
  constexpr int kWarps = 256 / 32;
  __shared__ uint32_t s_ce[kWarps], s_cr[kWarps];
  __shared__ unsigned long long s_be, s_br;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t stride = gridDim.x * blockDim.x;
  unsigned long long acc_we = 0, acc_wf = 0, acc_wm = 0;
  for (uint32_t base = blockIdx.x * blockDim.x; base < a.n_bins; base += stride) {  // block-uniform
    const uint32_t b = base + threadIdx.x;
    unsigned long long w = 0, d0 = 0, d1 = 0;
    bool has = false;
    if (b < a.n_bins) {
      w = a.win[b];
      d0 = a.off[b];
      d1 = a.off[b + 1];
      has = d1 != d0;
    }
    const bool el = has && w <= a.thr, rs = has && !el;
    const uint32_t me = __ballot_sync(kFull, el), mr = __ballot_sync(kFull, rs);
    if (el) {
      acc_we += w;
      acc_wf += smem_bin_out_bound(w, a.cap, a.max_fill);
    }
    if (has) acc_wm = max(acc_wm, w);
    if (lane == 0) {
      s_ce[warp] = __popc(me);
      s_cr[warp] = __popc(mr);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t te = 0, tr = 0;
      for (int q = 0; q < kWarps; ++q) {
        te += s_ce[q];
        tr += s_cr[q];
      }
      s_be = te ? atomicAdd(&a.sums[0], (unsigned long long)te) : 0ull;
      s_br = tr ? atomicAdd(&a.sums[3], (unsigned long long)tr) : 0ull;
    }
    __syncthreads();
    uint32_t pe = 0, pr = 0;
    for (uint32_t q = 0; q < warp; ++q) {
      pe += s_ce[q];
      pr += s_cr[q];
    }
    const uint32_t below = (1u << lane) - 1u;
    if (el) {
      const unsigned long long i = s_be + pe + __popc(me & below);
      a.elig[2 * i] = d0;
      a.elig[2 * i + 1] = d1 | ((w < (1ull << 24) ? w : (1ull << 24) - 1) << kRangeWinShift);
    } else if (rs) {
      const unsigned long long i = s_br + pr + __popc(mr & below);
      a.rest[3 * i] = d0;
      a.rest[3 * i + 1] = d1;
      a.rest[3 * i + 2] = w;
    }
    __syncthreads();  // s_ce / s_be are rewritten by the next iteration
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_we += __shfl_xor_sync(kFull, acc_we, o);
    acc_wf += __shfl_xor_sync(kFull, acc_wf, o);
    acc_wm = max(acc_wm, __shfl_xor_sync(kFull, acc_wm, o));
  }
  if (lane == 0) {
    if (acc_we) atomicAdd(&a.sums[1], acc_we);
    if (acc_wf) atomicAdd(&a.sums[2], acc_wf);
    if (acc_wm) atomicMax(a.max_win, acc_wm);
  }
}

cudaError_t launch_plan_bins(const PlanBinsArgs& a, int sms, cudaStream_t st) {
  if (a.n_bins == 0) return cudaSuccess;
  uint64_t grid = (a.n_bins + 255) / 256;
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  plan_bins_kernel<<<(unsigned)grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_count_smem(const SmemCountArgs& a, int sms, cudaStream_t st) {
  if (a.n_list == 0) return cudaSuccess;
  if (key_words(a.k) >= 4 || a.warps < 0) return launch_count_ref(a, sms, st);  // CTA-wide reference tables
  switch (key_words(a.k)) {
    case 1: return launch_smem<1, true>(a, sms, st);
    case 2: return smem_pack(a.k) ? launch_smem<2, true>(a, sms, st) : launch_smem<2, false>(a, sms, st);
    case 3: return launch_smem<3, false>(a, sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gerbil
