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
//    smem, canonicalise, hash and load the bucket (two 32-byte
//    sectors): a matching k-mer → fire-and-forget RED on its count;
//  - everything else goes to a per-warp queue in shared memory that is
//    drained 32 entries per memory round trip: new k-mers (an empty slot in
//    the view) as deferred 128-bit CAS claims, and the rare re-probes (bucket
//    full → next trial, claim lost, half-visible slot). So a warp round waits
//    on one L2 round trip (the bucket load), never on a CAS; after θ buckets
//    a k-mer goes to the emergency area.
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "table_inline.cuh"

#include <cstdio>

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

// 8-byte cp.async global → shared; zero-fills when !valid
__device__ __forceinline__ void cp_async8(uint64_t* dst, const uint64_t* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct RetryQueue {
  uint64_t k0[kQueue], k1[kQueue], bkt[kQueue];
  uint32_t probes[kQueue];
};

// One look at the view w of bucket b for key (k0, k1). Returns 0 = counted
// (RED on the matching slot), 1 = look again (a slot read mid-claim),
// 2 = bucket full (next trial), 3 + s = claim the first empty slot s.
template <bool TWO>
__device__ __forceinline__ int probe_view(unsigned char* table, uint64_t b, uint64_t k0, uint64_t k1,
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
  if (torn) return 1;
  if (es < 0) return 2;
  return 3 + es;
}

// Deferred claim of slot s (empty in an earlier view): ONE 128-bit CAS writes
// (x, 1). Slots fill in order and never empty within a wave, so a CAS that
// finds the slot taken by another k-mer only means the view was old: look
// again. Returns true when x was counted.
template <bool TWO>
__device__ __forceinline__ bool claim_slot(unsigned char* table, uint64_t b, uint32_t s, uint64_t k0,
                                           uint64_t k1) {
  uint64_t* slot = reinterpret_cast<uint64_t*>(table + b * kInlineBucketBytes) + 2 * s;
  const Slot16 old = cas128(slot, 0ull, 0ull, k0, k1 | 1ull);  // empty entry → (x, 1)
  if (old.w0 == 0ull) return true;
  if (inline_match(old.w0, old.w1, k0, k1)) {
    atomicAdd(inline_count(slot), 1u);
    return true;
  }
  return false;
}

template <int W, bool TWO>
__global__ void __launch_bounds__(128) count_inline_kernel(CountArgs a) {
  __shared__ __align__(16) uint64_t s_stage[4][2][32 * kStageWords];
  __shared__ RetryQueue s_q[4];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  RetryQueue& q = s_q[wib];
  uint32_t qn = 0;  // warp-uniform queue length
  const uint32_t dpc = a.dpc ? a.dpc : 32u;
  const uint64_t n_chunks = (a.d1 - a.d0 + dpc - 1) / dpc;
  uint32_t first = 0, more = 0, maxp = 0;

  // Queue entries: key, bucket, probes | op << 24 — op 0 = look at the bucket,
  // op 1 + s = claim slot s. A warp round never waits on a CAS: claims are
  // queued and 32 of them are issued together by one drain.
  auto push = [&](uint32_t mask, uint64_t k0, uint64_t k1, uint64_t b, uint32_t pq) {
    // the queue is warp-shared state: every lane reaches each push / drain together (under
    // independent thread scheduling a lane that left a divergent probe or emergency path late
    // must not race the others' queue accesses; compute-sanitizer memcheck caught this with
    // theta = 1 on over-full tables)
    __syncwarp();
#ifdef GERBIL_QDEBUG
    {
      int pred = 0;
      __match_all_sync(0xffffffffu, qn, &pred);
      if (qn + __popc(mask) > kQueue || !pred) printf("push: qn=%u mask=%08x lane=%u blk=%d\n", qn, mask, lane, blockIdx.x);
    }
#endif
    if ((mask >> lane) & 1u) {
      const uint32_t i = qn + __popc(mask & ((1u << lane) - 1u));
      q.k0[i] = k0;
      q.k1[i] = k1;
      q.bkt[i] = b;
      q.probes[i] = pq;
    }
    qn += __popc(mask);
  };
  auto resolved = [&](uint32_t p) {
    if (p == 1) ++first;
    else { ++more; maxp = max(maxp, p); }
  };
  // act on one bucket view; returns the entry to queue (probes | op << 24) or ~0u
  auto settle_view = [&](uint64_t k0, uint64_t k1, uint64_t& b, uint32_t& p, const uint64_t (&w)[8]) -> uint32_t {
    const int r = probe_view<TWO>(a.t.table, b, k0, k1, w);
    if (r == 0) {
      resolved(p);
      return ~0u;
    }
    if (r >= 3) return p | ((uint32_t)(r - 2) << 24);  // deferred claim of slot r - 3
    if (r == 2) {
      if (p >= a.t.max_probes) {  // θ trials exhausted → emergency area
        uint64_t ch[2] = {k0, k1}, key[2];
        from_chunks(ch, TWO ? 2u : 1u, key, (uint32_t)W);
        const unsigned long long e = atomicAdd(a.t.ovf_n, 1ull);
        if (e < a.t.ovf_cap) {
#pragma unroll
          for (int v = 0; v < W; ++v) a.t.ovf[e * W + v] = key[v];
        }
        return ~0u;
      }
      b = (b + 1 == a.t.nb) ? 0 : b + 1;  // bucket occupied by other k-mers → next trial
      ++p;
    }
    return p;
  };
  // one memory round trip for `n` queued entries taken from the top (lanes < n)
  auto drain_n = [&](uint32_t n) {
    __syncwarp();

#ifdef GERBIL_QDEBUG
    {
      int pred = 0;
      __match_all_sync(0xffffffffu, qn, &pred);
      if (qn < n || qn > kQueue || !pred) printf("drain: qn=%u n=%u lane=%u blk=%d\n", qn, n, lane, blockIdx.x);
    }
#endif
    const uint32_t base = qn - n;
    const bool mine = lane < n;
    uint64_t k0 = 0, k1 = 0, b = 0;
    uint32_t pq = 0;
    if (mine) {
      k0 = q.k0[base + lane];
      k1 = q.k1[base + lane];
      b = q.bkt[base + lane];
      pq = q.probes[base + lane];
    }
    __syncwarp();
    qn = base;
    uint32_t p = pq & 0xffffffu, op = pq >> 24, nq = ~0u;
    if (mine) {
      if (op == 0) {
        uint64_t w[8];
        ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + b * kInlineBucketBytes), w);
        nq = settle_view(k0, k1, b, p, w);
      } else if (claim_slot<TWO>(a.t.table, b, op - 1, k0, k1)) {
        resolved(p);
      } else {
        nq = p;  // the slot was taken: look at the bucket again
      }
    }
    push(__ballot_sync(0xffffffffu, nq != ~0u), k0, k1, b, nq);
    __syncwarp();
  };

  // Chunk pipeline (per warp): the claim of chunk c+2 (lane 0's atomic), the
  // descriptors of chunk c+1 (registers) and the packed words of chunk c+1
  // (cp.async into the other half of a double-buffered stage) are in flight
  // while chunk c is counted — no prefetch held in registers, no DRAM latency
  // on the per-window chain.
  unsigned long long claim = 0;
  auto claim_issue = [&]() {
    if (lane == 0) claim = atomicAdd(a.work, 1ull);
  };
  auto claimed = [&]() -> unsigned long long { return __shfl_sync(0xffffffffu, claim, 0); };
  auto desc_load = [&](unsigned long long chk) -> uint64_t {  // ~0 = no super-mer
    const uint64_t di = a.d0 + chk * dpc + lane;
    return (chk < n_chunks && lane < dpc && di < a.d1) ? __ldg(a.desc + di) : ~0ull;
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
    for (int s = 0; s < kStageWords; ++s) cp_async8(dst + s, src + (s < (int)nwords ? s : 0), s < (int)nwords);
    cp_async_commit();
  };
  claim_issue();
  unsigned long long id0 = claimed();
  claim_issue();
  unsigned long long id1 = claimed();
  uint64_t d0 = desc_load(id0);
  issue_words(d0, s_stage[wib][0] + lane * kStageWords);
  uint64_t d1 = desc_load(id1);
  claim_issue();
  uint32_t buf = 0;

  for (;;) {
    if (id0 >= n_chunks) break;
    const unsigned long long id2 = claimed();
    issue_words(d1, s_stage[wib][buf ^ 1] + lane * kStageWords);
    const uint64_t d2 = desc_load(id2);
    claim_issue();
    const uint64_t* stage = s_stage[wib][buf];
    const uint64_t pos = d0 == ~0ull ? 0ull : d0 >> kNwinBits;
    const uint32_t nw = d0 == ~0ull ? 0u : (uint32_t)(d0 & ((1u << kNwinBits) - 1)) + 1;
    const bool staged = ((uint32_t)(pos & 31) + nw + a.k - 1) <= 32u * kStageWords;
    cp_async_wait<1>();
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
      uint32_t nq = ~0u;
      if (act) {
        uint64_t w[8];
        ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + b * kInlineBucketBytes), w);
        nq = settle_view(k0, k1, b, p, w);
      }
      push(__ballot_sync(0xffffffffu, nq != ~0u), k0, k1, b, nq);
      __syncwarp();
      while (qn >= 32) drain_n(32);
    }
    __syncwarp();  // the stage half just read is refilled next iteration
    id0 = id1;
    d0 = d1;
    id1 = id2;
    d1 = d2;
    buf ^= 1;
  }
  cp_async_wait<0>();
  // finish the queue: full batches first, then the remainder (lanes >= qn idle)
  while (qn >= 32) drain_n(32);
  while (qn > 0) drain_n(qn);
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
