// count_inline.cuh — step (d) kernel for the inline table kind (k <= 46).
//
// Alg. 1 over the windows of the super-mers of one wave.
// DESIGN.md "Kernel (d)":
//  - a warp takes 32 bin-ordered descriptors at a time (dynamic counter);
//    lane j gathers super-mer j's packed words (<= kStageWords) into a per-warp
//    shared-memory stage, and the NEXT chunk's words are prefetched into
//    registers while the current chunk is counted, so no DRAM latency sits on
//    the per-window chain;
//  - lanes walk the chunk's windows 32·U at a time, extract each k-mer from
//    smem, canonicalise, hash;
//  - probing runs in batched rounds: every pending window examines one bucket
//    (both 32-byte sectors prefetched), REDs are fired, CASes are issued for
//    all windows before any result is consumed; windows whose bucket is full
//    move to the next bucket in the next round (θ buckets, then the emergency
//    area).
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "table_inline.cuh"

namespace gerbil {

constexpr int kStageWords = 8;  // packed words staged per super-mer (≤ 256 bases)

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

template <int W, bool TWO, int U>
__global__ void __launch_bounds__(128) count_inline_kernel(CountArgs a) {
  __shared__ uint64_t s_stage[4][32 * kStageWords];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  uint64_t* stage = s_stage[wib];
  const uint64_t n_chunks = (a.d1 - a.d0 + 31) / 32;
  uint32_t first = 0, more = 0, maxp = 0;

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
      for (int q = 0; q < kStageWords; ++q) n_words[q] = (q < (int)nwords) ? __ldg(src + q) : 0ull;
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
    for (int q = 0; q < kStageWords; ++q) stage[lane * kStageWords + q] = n_words[q];
    const bool staged = ((uint32_t)(pos & 31) + nw + a.k - 1) <= 32u * kStageWords;
    if (lane == 0) nxt = atomicAdd(a.work, 1ull);
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
    fetch(nxt);
    __syncwarp();

    const uint32_t incl = warp_incl_scan_u32(nw), excl = incl - nw;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t stage_mask = __ballot_sync(0xffffffffu, staged);
    for (uint32_t base = 0; base < total; base += 32 * U) {
      uint64_t k0[U], k1[U], bkt[U], w[U][8];
      uint64_t ckey[U][W];
      bool pend[U];
      uint32_t probes[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = base + u * 32 + lane;
        int j = 0;  // super-mer (lane) holding window i: #lanes with incl <= i
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, j + step - 1);
          if (v <= i) j += step;
        }
        const uint64_t pj = __shfl_sync(0xffffffffu, pos, j);
        const uint32_t ej = __shfl_sync(0xffffffffu, excl, j);
        pend[u] = i < total;
        probes[u] = pend[u] ? 1u : 0xffffffffu;
        uint64_t x[W], r[W];
        if ((stage_mask >> j) & 1u) {
          extract_smem<W>(stage + j * kStageWords, (uint32_t)(pj & 31) + (i - ej), a.k, x);
        } else {
          extract_kmer<W>(a.codes, pend[u] ? pj + (i - ej) : 0ull, a.k, x);
        }
        reverse_complement<W>(x, a.k, r);
        const bool use_r = key_less<W>(r, x);
#pragma unroll
        for (int v = 0; v < W; ++v) ckey[u][v] = use_r ? r[v] : x[v];
        uint64_t ch[2];
        to_chunks<W, 2>(ckey[u], ch);
        k0[u] = ch[0];
        k1[u] = TWO ? ch[1] : 0ull;
        bkt[u] = bucket_of(key_hash<W>(ckey[u]), a.t.nb);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pend[u]) ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + bkt[u] * kInlineBucketBytes), w[u]);
      // batched probe rounds (Alg. 1 trials)
      for (;;) {
        bool anyp = false;
#pragma unroll
        for (int u = 0; u < U; ++u) anyp |= pend[u];
        if (!__any_sync(0xffffffffu, anyp)) break;
        int cas_slot[U];
        Slot16 old[U];
        bool reload[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          cas_slot[u] = -1;
          reload[u] = false;
          if (!pend[u]) continue;
          uint64_t* bk = reinterpret_cast<uint64_t*>(a.t.table + bkt[u] * kInlineBucketBytes);
#pragma unroll
          for (int s = 0; s < 4; ++s) settle<TWO>(bk + 2 * s, w[u][2 * s], w[u][2 * s + 1]);
          int ms = -1, es = -1;
#pragma unroll
          for (int s = 3; s >= 0; --s) {
            if (inline_match(w[u][2 * s], w[u][2 * s + 1], k0[u], k1[u])) ms = s;
            if (w[u][2 * s] == 0ull) es = s;
          }
          if (ms >= 0) {  // matching k-mer → count + 1
            atomicAdd(inline_count(bk + 2 * ms), 1u);
            pend[u] = false;
          } else if (es >= 0) {  // empty entry → claim (x, 1)
            cas_slot[u] = es;
            old[u] = cas128(bk + 2 * es, 0ull, 0ull, k0[u], k1[u] | 1ull);
          } else if (probes[u] >= a.t.max_probes) {  // θ trials exhausted → emergency
            const unsigned long long e = atomicAdd(a.t.ovf_n, 1ull);
            if (e < a.t.ovf_cap) {
#pragma unroll
              for (int v = 0; v < W; ++v) a.t.ovf[e * W + v] = ckey[u][v];
            }
            pend[u] = false;
            probes[u] = 0;
          } else {  // bucket occupied by other k-mers → next trial
            bkt[u] = (bkt[u] + 1 == a.t.nb) ? 0 : bkt[u] + 1;
            ++probes[u];
            reload[u] = true;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (cas_slot[u] < 0) continue;
          if (old[u].w0 == 0ull) {
            pend[u] = false;
          } else if (inline_match(old[u].w0, old[u].w1, k0[u], k1[u])) {
            uint64_t* bk = reinterpret_cast<uint64_t*>(a.t.table + bkt[u] * kInlineBucketBytes);
            atomicAdd(inline_count(bk + 2 * cas_slot[u]), 1u);
            pend[u] = false;
          } else {
            reload[u] = true;  // lost the slot to another k-mer: re-examine this bucket
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (reload[u])
            ld_bucket_inline(reinterpret_cast<const uint64_t*>(a.t.table + bkt[u] * kInlineBucketBytes), w[u]);
          if (!pend[u] && !reload[u] && probes[u] != 0xffffffffu) {
            // resolved this round: record probe statistics once
            const uint32_t p = probes[u];
            if (p == 1) ++first;
            else if (p > 1) { ++more; maxp = max(maxp, p); }
            probes[u] = 0xffffffffu;
          }
        }
      }
    }
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
