// count_kernels.cuh — the step-(d) kernels of count.cu as templates, shared by the
// translation units that instantiate them (count.cu: W <= 7; count_wide.cu: W = 8..15,
// k up to 479). Documentation: count.cu.
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "table.cuh"
#include "table_inline.cuh"
#include "count_inline.cuh"

#include <stdlib.h>

namespace gerbil {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (uint32_t)o) v += t;
  }
  return v;
}

template <int W>
__device__ __forceinline__ void emergency(const TableArgs& t, const uint64_t (&c)[W]) {
  const unsigned long long i = atomicAdd(t.ovf_n, 1ull);
  if (i < t.ovf_cap) {
#pragma unroll
    for (int w = 0; w < W; ++w) t.ovf[i * W + w] = c[w];
  }
}

struct ProbeStats {
  uint32_t first = 0, more = 0, maxp = 0;
  __device__ void add(uint32_t p) {
    if (p == 1) ++first;
    else if (p > 1) { ++more; maxp = max(maxp, p); }
  }
  __device__ void flush(const TableArgs& t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      first += __shfl_down_sync(0xffffffffu, first, o);
      more += __shfl_down_sync(0xffffffffu, more, o);
      maxp = max(maxp, __shfl_down_sync(0xffffffffu, maxp, o));
    }
    if (lane_id() == 0 && t.probe_hist) {
      if (first) atomicAdd(&t.probe_hist[0], (unsigned long long)first);
      if (more) atomicAdd(&t.probe_hist[1], (unsigned long long)more);
      if (maxp) atomicMax(&t.probe_hist[2], (unsigned long long)maxp);
    }
  }
};

template <int W, int WP, int U>
__global__ void __launch_bounds__(kThreads) count_kernel(CountArgs a) {
  const uint32_t lane = lane_id();
  const uint32_t dpc = a.dpc ? a.dpc : 32u;
  const uint64_t n_chunks = (a.d1 - a.d0 + dpc - 1) / dpc;
  ProbeStats ps;
  for (;;) {
    unsigned long long chk = 0;
    if (lane == 0) chk = atomicAdd(a.work, 1ull);
    chk = __shfl_sync(0xffffffffu, chk, 0);
    if (chk >= n_chunks) break;
    const uint64_t di = a.d0 + chk * dpc + lane;
    uint64_t pos = 0;
    uint32_t nw = 0;
    if (lane < dpc && di < a.d1) {
      const uint64_t d = __ldg(a.desc + di);
      pos = d >> kNwinBits;
      nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
    }
    const uint32_t incl = warp_incl_scan(nw), excl = incl - nw;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t base = 0; base < total; base += 32 * U) {
      uint64_t q[U];
      bool act[U];
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
        act[u] = i < total;
        q[u] = pj + (i - ej);
      }
      uint64_t c[U][W], ch[U][WP], bkt[U], w[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint64_t x[W], r[W];
        extract_kmer<W>(a.codes, act[u] ? q[u] : 0ull, a.k, x);
        bool use_r = false;
        if (a.canonical) {  // warp-uniform
          reverse_complement<W>(x, a.k, r);
          use_r = key_less<W>(r, x);
        }
#pragma unroll
        for (int v = 0; v < W; ++v) c[u][v] = use_r ? r[v] : x[v];
        to_chunks<W, WP>(c[u], ch[u]);
        bkt[u] = bucket_of(key_hash<W>(c[u]), a.t.nb);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act[u]) ld_c0(bucket_at(a.t.table, bkt[u], WP).c0, w[u]);
      // Batched first probe: classify each window from its prefetched sector,
      // then issue every CAS / rest-chunk load before consuming any result,
      // so the U round trips overlap. Anything unusual (full bucket, equal
      // chunk0 of a different key, lost race) takes the generic Alg. 1 loop.
      int slot[U];
      bool match[U];
      uint64_t old[U], r1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        slot[u] = -1;
        match[u] = false;
#pragma unroll
        for (int s = 3; s >= 0; --s)
          if (w[u][s] == ch[u][0]) slot[u] = s;
        if (slot[u] >= 0) {
          match[u] = true;
        } else {
#pragma unroll
          for (int s = 3; s >= 0; --s)
            if (w[u][s] == 0ull) slot[u] = s;
        }
        if (!act[u]) slot[u] = -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (slot[u] < 0) continue;
        const Bucket bk = bucket_at(a.t.table, bkt[u], WP);
        if (match[u]) {
          if (WP > 1) r1[u] = ld_relaxed_u64(bk.rest + slot[u] * (WP - 1));
        } else {
          old[u] = atomicCAS(reinterpret_cast<unsigned long long*>(bk.c0 + slot[u]), 0ull,
                             (unsigned long long)ch[u][0]);
        }
      }
      // Pass A publishes every successful claim (rest chunks + count) BEFORE
      // any lane may spin in the generic path below: a thread never waits
      // while holding an unpublished claim, so no circular wait can form.
      bool done[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        done[u] = !act[u];
        if (slot[u] < 0) continue;
        const Bucket bk = bucket_at(a.t.table, bkt[u], WP);
        const int s = slot[u];
        if (match[u]) {
          // WP == 1: chunk0 is the whole key. WP == 2: one rest chunk, already loaded.
          if (WP == 1 || (WP == 2 && r1[u] == ch[u][1])) {
            atomicAdd(bk.cnt + s, 1u);
            done[u] = true;
          }
        } else if (old[u] == 0ull) {
#pragma unroll
          for (int j = 1; j < WP; ++j) bk.rest[s * (WP - 1) + (j - 1)] = ch[u][j];
          atomicAdd(bk.cnt + s, 1u);
          done[u] = true;
        }
        if (done[u]) ps.add(1);
      }
      // Pass B: generic path (re-reads the bucket): full bucket, WP > 2, races, equal chunk0
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (done[u]) continue;
        uint64_t wb[4];
        ld_c0(bucket_at(a.t.table, bkt[u], WP).c0, wb);
        const uint32_t p = table_insert<WP>(a.t.table, a.t.nb, a.t.max_probes, ch[u], bkt[u], wb);
        if (p == 0) emergency<W>(a.t, c[u]);
        ps.add(p);
      }
    }
  }
  ps.flush(a.t);
}

// ---- inline table kind (k <= 46, table_inline.cuh) ---------------------------------
template <int W, bool TWO>
__device__ __noinline__ uint32_t inline_generic(const TableArgs t, uint64_t c0, uint64_t c1, uint64_t b) {
  uint64_t w[8];
  ld_bucket_inline(reinterpret_cast<const uint64_t*>(t.table + b * kInlineBucketBytes), w);
  return inline_insert<TWO>(t.table, t.nb, t.max_probes, c0, c1, b, w);
}

template <int W, bool TWO>
__global__ void __launch_bounds__(kThreads) count_keys_inline_kernel(CountKeysArgs a) {
  ProbeStats ps;
  for (uint64_t i = blockIdx.x * (uint64_t)kThreads + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * kThreads) {
    uint64_t c[W], ch[2];
#pragma unroll
    for (int v = 0; v < W; ++v) c[v] = a.keys[i * W + v];
    to_chunks<W, 2>(c, ch);
    const uint64_t k1 = TWO ? ch[1] : 0ull;
    const uint32_t p = inline_generic<W, TWO>(a.t, ch[0], k1, bucket_of(key_hash<W>(c), a.t.nb));
    if (p == 0) emergency<W>(a.t, c);
    ps.add(p);
  }
  ps.flush(a.t);
}

// Emergency path: count the overflow k-mers exactly in a fresh table whose θ
// covers every bucket.
template <int W, int WP>
__global__ void __launch_bounds__(kThreads) count_keys_kernel(CountKeysArgs a) {
  ProbeStats ps;
  for (uint64_t i = blockIdx.x * (uint64_t)kThreads + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * kThreads) {
    uint64_t c[W], ch[WP], w[4];
#pragma unroll
    for (int v = 0; v < W; ++v) c[v] = a.keys[i * W + v];
    to_chunks<W, WP>(c, ch);
    const uint64_t b = bucket_of(key_hash<W>(c), a.t.nb);
    ld_c0(bucket_at(a.t.table, b, WP).c0, w);
    const uint32_t p = table_insert<WP>(a.t.table, a.t.nb, a.t.max_probes, ch, b, w);
    if (p == 0) emergency<W>(a.t, c);
    ps.add(p);
  }
  ps.flush(a.t);
}

template <int W, int WP>
cudaError_t launch_count_w(const CountArgs& a, int sms, cudaStream_t st) {
  constexpr int U = W <= 2 ? 4 : (W <= 4 ? 2 : 1);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_kernel<W, WP, U>, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t dpc = a.dpc ? a.dpc : 32u;
  const uint64_t chunks = (a.d1 - a.d0 + dpc - 1) / dpc;
  uint64_t grid = (uint64_t)sms * per_sm;
  const uint64_t need = (chunks + kThreads / 32 - 1) / (kThreads / 32);
  if (grid > need) grid = need;
  if (grid == 0) return cudaSuccess;
  count_kernel<W, WP, U><<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

template <int W, int WP>
cudaError_t launch_count_keys_w(const CountKeysArgs& a, int sms, cudaStream_t st) {
  uint64_t grid = (a.n + kThreads - 1) / kThreads;
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  if (grid == 0) return cudaSuccess;
  count_keys_kernel<W, WP><<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace
}  // namespace gerbil
