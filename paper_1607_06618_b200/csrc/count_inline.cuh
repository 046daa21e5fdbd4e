// count_inline.cuh — step (d) kernel for the inline table kind (k <= 46).
//
// Alg. 1 over the windows of the super-mers of one wave.
// DESIGN.md "Kernel (d)":
//  - a warp takes 32 bin-ordered descriptors at a time (dynamic counter);
//    lane j gathers super-mer j's packed words (<= kStageWords) into a per-warp
//    shared-memory stage, and the NEXT chunk's words are prefetched into
//    registers while the current chunk is counted, so no DRAM latency sits on
//    the per-window chain;
//  - lanes walk the chunk's windows 32 at a time, extract each k-mer from
//    smem, canonicalise, hash, load the bucket (two 32-byte
//    sectors) and resolve it in ONE probe: a matching k-mer → RED on its
//    count; an empty slot → one 128-bit CAS claim;
//  - the few windows that do not resolve there (bucket full → next trial, lost
//    CAS race, half-visible slot) are pushed to a per-warp retry queue in
//    shared memory and drained 32 at a time, so a rare second probe never
//    costs a whole warp-round; after θ buckets a k-mer goes to the emergency
//    area.
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "table_inline.cuh"

namespace gerbil {

constexpr int kStageWords = 8;  // packed words staged per super-mer (≤ 256 bases)
constexpr int kQueue = 64;      // per-warp retry queue entries

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (uint32_t)o) v += t;
  }
  return v;
}

// k-mer at base offset o of a staged super-mer (smem words), W left-aligned words
template <int W>
__device__ __forceinline__ void extract_smem(const uint64_t* s, uint32_t o, uint32_t k, uint64_t (&x)[W]) {
  const uint32_t w0 = o >> 5, sh = (o & 31) * 2;
  uint64_t a[W + 1];
#pragma unroll
  for (int i = 0; i <= W; ++i) a[i] = (w0 + i < (uint32_t)kStageWords) ? s[w0 + i] : 0ull;
#pragma unroll
  for (int i = 0; i < W; ++i) x[i] = sh ? ((a[i] << sh) | (a[i + 1] >> (64 - sh))) : a[i];
  const uint32_t tail = 2 * k - 64 * (W - 1);
  if (tail < 64) x[W - 1] &= ~0ull << (64 - tail);
}

struct RetryQueue {
  uint64_t k0[kQueue], k1[kQueue], bkt[kQueue];
  uint32_t probes[kQueue];
};

// One probe of bucket b for key (k0, k1). Returns 0 = resolved, 1 = retry the
// same bucket (lost race / half-visible slot), 2 = bucket full (next trial).
template <bool TWO>
__device__ __forceinline__ int probe_once(unsigned char* table, uint64_t b, uint64_t k0, uint64_t k1,
                                          const uint64_t (&w)[8]) {
  uint64_t* bk = reinterpret_cast<uint64_t*>(table + b * kInlineBucketBytes);
  int ms = -1, es = -1;
  bool torn = false;
#pragma unroll
  for (int s = 3; s >= 0; --s) {
    if (inline_match(w[2 * s], w[2 * s + 1], k0, k1)) ms = s;
    if (w[2 * s] == 0ull) es = s;
    if (TWO) torn |= (w[2 * s] != 0ull) && !(w[2 * s + 1] >> 63);
  }
  if (ms >= 0) {  // matching k-mer → count + 1
    atomicAdd(inline_count(bk + 2 * ms), 1u);
    return 0;
  }
  if (torn) return 1;  // a slot was read mid-claim: look again
  if (es < 0) return 2;
  const Slot16 old = cas128(bk + 2 * es, 0ull, 0ull, k0, k1 | 1ull);  // empty entry → (x, 1)
  if (old.w0 == 0ull) return 0;
  if (inline_match(old.w0, old.w1, k0, k1)) {
    atomicAdd(inline_count(bk + 2 * es), 1u);
    return 0;
  }
  return 1;  // lost the slot to another k-mer: re-examine this bucket
}

template <int W, bool TWO>
__global__ void __launch_bounds__(128) count_inline_kernel(CountArgs a) {
  __shared__ uint64_t s_stage[4][32 * kStageWords];
  __shared__ RetryQueue s_q[4];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  uint64_t* stage = s_stage[wib];
  RetryQueue& q = s_q[wib];
  uint32_t qn = 0;  // warp-uniform queue length
  const uint64_t n_chunks = (a.d1 - a.d0 + 31) / 32;
  uint32_t first = 0, more = 0, maxp = 0;

  // push the lanes in `mask` (each with its own entry) to the retry queue
  auto push = [&](uint32_t mask, uint64_t k0, uint64_t k1, uint64_t b, uint32_t p) {
    if ((mask >> lane) & 1u) {
      const uint32_t i = qn + __popc(mask & ((1u << lane) - 1u));
      q.k0[i] = k0;
      q.k1[i] = k1;
      q.bkt[i] = b;
      q.probes[i] = p;
    }
    qn += __popc(mask);
  };
  // resolve one probe for the lanes in `act`; returns the lanes to requeue
  auto settle_lanes = [&](bool act, uint64_t k0, uint64_t k1, uint64_t& b, uint32_t& p,
                          const uint64_t (&w)[8]) -> bool {
    bool again = false;
    if (act) {
      const int r = probe_once<TWO>(a.t.table, b, k0, k1, w);
      if (r == 0) {
        if (p == 1) ++first;
        else { ++more; maxp = max(maxp, p); }
      } else if (r == 2 && p >= a.t.max_probes) {  // θ trials exhausted → emergency
        uint64_t ch[2] = {k0, k1}, key[2];
        from_chunks(ch, TWO ? 2u : 1u, key, (uint32_t)W);
        const unsigned long long e = atomicAdd(a.t.ovf_n, 1ull);
        if (e < a.t.ovf_cap) {
#pragma unroll
          for (int v = 0; v < W; ++v) a.t.ovf[e * W + v] = key[v];
        }
      } else {
        if (r == 2) {  // bucket occupied by other k-mers → next trial
          b = (b + 1 == a.t.nb) ? 0 : b + 1;
          ++p;
        }
        again = true;
      }
    }
    return again;
  };
  // drain 32 queued windows (one per lane), requeueing the unresolved
  auto drain = [&]() {
    const uint32_t base = qn - 32;
    uint64_t k0 = q.k0[base + lane], k1 = q.k1[base + lane], b = q.bkt[base + lane];
    uint32_t p = q.probes[base + lane];
    __syncwarp();
    qn = base;
    uint64_t w[8];
    ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + b * kInlineBucketBytes), w);
    const bool again = settle_lanes(true, k0, k1, b, p, w);
    push(__ballot_sync(0xffffffffu, again), k0, k1, b, p);
    __syncwarp();
  };

  // prefetch state of the next chunk (registers)
  unsigned long long nxt = 0;
  uint64_t n_pos = 0;
  uint32_t n_nw = 0;
  uint64_t n_words[kStageWords];
  auto fetch = [&](unsigned long long chk) {
    n_pos = 0;
    n_nw = 0;
    if (chk >= n_chunks) return;
    const uint64_t di = a.d0 + chk * 32 + lane;
    if (di < a.d1) {
      const uint64_t d = __ldg(a.desc + di);
      n_pos = d >> kNwinBits;
      n_nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
      const uint32_t nwords = ((uint32_t)(n_pos & 31) + n_nw + a.k - 1 + 31) >> 5;
      const uint64_t* src = a.codes + (n_pos >> 5);
#pragma unroll
      for (int s = 0; s < kStageWords; ++s) n_words[s] = (s < (int)nwords) ? __ldg(src + s) : 0ull;
    }
  };
  if (lane == 0) nxt = atomicAdd(a.work, 1ull);
  nxt = __shfl_sync(0xffffffffu, nxt, 0);
  fetch(nxt);

  for (;;) {
    const unsigned long long chk = nxt;
    if (chk >= n_chunks) break;
    // install the prefetched chunk, start fetching the following one
    const uint64_t pos = n_pos;
    const uint32_t nw = n_nw;
    __syncwarp();
#pragma unroll
    for (int s = 0; s < kStageWords; ++s) stage[lane * kStageWords + s] = n_words[s];
    const bool staged = ((uint32_t)(pos & 31) + nw + a.k - 1) <= 32u * kStageWords;
    if (lane == 0) nxt = atomicAdd(a.work, 1ull);
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
    fetch(nxt);
    __syncwarp();

    const uint32_t incl = warp_incl_scan_u32(nw), excl = incl - nw;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t stage_mask = __ballot_sync(0xffffffffu, staged);
    for (uint32_t base = 0; base < total; base += 32) {
      const uint32_t i = base + lane;
      int j = 0;  // super-mer (lane) holding window i: #lanes with incl <= i
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, j + step - 1);
        if (v <= i) j += step;
      }
      const uint64_t pj = __shfl_sync(0xffffffffu, pos, j);
      const uint32_t ej = __shfl_sync(0xffffffffu, excl, j);
      const bool act = i < total;
      uint64_t x[W], r[W], c[W];
      if ((stage_mask >> j) & 1u) {
        extract_smem<W>(stage + j * kStageWords, (uint32_t)(pj & 31) + (i - ej), a.k, x);
      } else {
        extract_kmer<W>(a.codes, act ? pj + (i - ej) : 0ull, a.k, x);
      }
      bool use_r = false;
      if (a.canonical) {  // warp-uniform
        reverse_complement<W>(x, a.k, r);
        use_r = key_less<W>(r, x);
      }
#pragma unroll
      for (int v = 0; v < W; ++v) c[v] = use_r ? r[v] : x[v];
      uint64_t ch[2];
      to_chunks<W, 2>(c, ch);
      const uint64_t k0 = ch[0], k1 = TWO ? ch[1] : 0ull;
      uint64_t b = bucket_of(key_hash<W>(c), a.t.nb);
      uint32_t p = 1;
      uint64_t w[8];
      if (act) ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + b * kInlineBucketBytes), w);
      const bool again = settle_lanes(act, k0, k1, b, p, w);
      push(__ballot_sync(0xffffffffu, again), k0, k1, b, p);
      __syncwarp();
      while (qn >= 32) drain();
    }
  }
  // finish the queue: full batches first, then the remainder (lanes >= qn idle)
  while (qn >= 32) drain();
  while (qn > 0) {
    const bool mine = lane < qn;
    uint64_t k0 = 0, k1 = 0, b = 0;
    uint32_t p = 0;
    if (mine) {
      k0 = q.k0[lane];
      k1 = q.k1[lane];
      b = q.bkt[lane];
      p = q.probes[lane];
    }
    __syncwarp();
    qn = 0;
    uint64_t w[8];
    if (mine) ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + b * kInlineBucketBytes), w);
    const bool again = settle_lanes(mine, k0, k1, b, p, w);
    push(__ballot_sync(0xffffffffu, again), k0, k1, b, p);
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    first += __shfl_down_sync(0xffffffffu, first, o);
    more += __shfl_down_sync(0xffffffffu, more, o);
    maxp = max(maxp, __shfl_down_sync(0xffffffffu, maxp, o));
  }
  if (lane == 0 && a.t.probe_hist) {
    if (first) atomicAdd(&a.t.probe_hist[0], (unsigned long long)first);
    if (more) atomicAdd(&a.t.probe_hist[1], (unsigned long long)more);
    if (maxp) atomicMax(&a.t.probe_hist[2], (unsigned long long)maxp);
  }
}

}  // namespace gerbil
