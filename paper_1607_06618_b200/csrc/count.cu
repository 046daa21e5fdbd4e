// count.cu — step (d): split super-mers into canonical k-mers and count them.
//
// PAPER.md:113-115 (§2.3.2 steps 2-3): "split the super-mers into k-mers" and
// "insert the k-mers into their thread-own hash tables"; Alg. 1
// (PAPER.md:65-84): for trial i < θ, p ← hash(x, i); matching k-mer → count+1;
// empty entry → (x, 1); otherwise next trial; after θ trials, "Start emergency
// mechanism". §3.3.1: each probe scans a 128-byte window of
// adjacent entries in one memory access; atomics lock entries.
//
// B200 design ("Table"):
//  - work distribution: a warp takes 32 super-mer descriptors, prefix-sums
//    their window counts, and its lanes walk the union of windows 32 at a
//    time (lane ↔ window), so long and short super-mers balance the same way;
//  - extraction: each lane funnel-shifts its W-word k-mer out of the packed
//    stream (read-only path), computes rc and the canonical
//    c = min(x, rc x) in registers;
//  - table: buckets of 8 slots = [8 u32 tags][8 u32 counts][8 × W u64 keys];
//    one 32-byte sector of tags is the paper's "scan adjacent entries in one
//    access", decoupled from k (the window shrank with k);
//  - claim/publish (multi-word keys up to W = 7): CAS tag EMPTY → fp (busy),
//    store key words and count = 1, st.release tag = fp | READY. A reader
//    whose fingerprint matches a busy tag waits for READY, then compares the
//    full key; a match is counted with atomicAdd;
//  - buckets probe linearly (next bucket) for θ buckets; a k-mer that finds
//    none is appended to the overflow area, counted exactly
//    by count_keys_kernel afterwards. With no deletions and one probe order
//    per key, a key lives wholly in the table or wholly in the overflow area.
#include "common.cuh"
#include "kernels.h"

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
__device__ __forceinline__ bool key_equal(const uint64_t* slot_key, const uint64_t (&c)[W]) {
  bool eq = true;
#pragma unroll
  for (int i = 0; i < W; ++i) eq &= (ld_cg_u64(slot_key + i) == c[i]);
  return eq;
}

// Returns the number of buckets probed (1 = first bucket), or 0 on overflow.
template <int W>
__device__ __forceinline__ uint32_t table_insert(const TableArgs& t, const uint64_t (&c)[W],
                                                 uint64_t h) {
  uint32_t fp = (uint32_t)h & kFpMask;
  fp = fp ? fp : 1u;
  uint64_t b = ((h >> 32) * t.nb) >> 32;
  constexpr uint64_t kBB = 64 + 64 * W;
  for (uint32_t probe = 1; probe <= t.max_probes; ++probe) {
    unsigned char* bucket = t.table + b * kBB;
    uint32_t* tags = reinterpret_cast<uint32_t*>(bucket);
    uint32_t* cnts = tags + kSlotsPerBucket;
    uint64_t* keys = reinterpret_cast<uint64_t*>(bucket + 64);
    const uint4 t0 = ld_cg_v4(tags), t1 = ld_cg_v4(tags + 4);
    const uint32_t tg[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
    // (1) matching k-mer detected → count + 1
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if ((tg[s] & kFpMask) == fp) {
        uint32_t tv = tg[s];
        while (!(tv & kReady)) tv = ld_acquire_u32(tags + s);
        if (key_equal<W>(keys + s * W, c)) {
          atomicAdd(cnts + s, 1u);
          return probe;
        }
      }
    }
    // (2) empty entry → claim it and store (x, 1)
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (tg[s] == 0u) {
        const uint32_t old = atomicCAS(tags + s, 0u, fp);
        if (old == 0u) {
#pragma unroll
          for (int i = 0; i < W; ++i) keys[s * W + i] = c[i];
          cnts[s] = 1u;
          st_release_u32(tags + s, fp | kReady);
          return probe;
        }
        if ((old & kFpMask) == fp) {  // raced with an equal fingerprint
          uint32_t tv = old;
          while (!(tv & kReady)) tv = ld_acquire_u32(tags + s);
          if (key_equal<W>(keys + s * W, c)) {
            atomicAdd(cnts + s, 1u);
            return probe;
          }
        }
      }
    }
    // (3) entry occupied by other k-mers → next trial
    b = (b + 1 == t.nb) ? 0 : b + 1;
  }
  return 0;
}

template <int W>
__device__ __forceinline__ void emergency(const TableArgs& t, const uint64_t (&c)[W]) {
  const unsigned long long i = atomicAdd(t.ovf_n, 1ull);
  if (i < t.ovf_cap) {
#pragma unroll
    for (int w = 0; w < W; ++w) t.ovf[i * W + w] = c[w];
  }
}

__device__ __forceinline__ void flush_probe_stats(const TableArgs& t, uint32_t first, uint32_t more,
                                                  uint32_t maxp) {
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

template <int W>
__global__ void __launch_bounds__(kThreads) count_kernel(CountArgs a) {
  const uint32_t lane = lane_id();
  const uint64_t nd = a.d1 - a.d0, n_chunks = (nd + 31) / 32;
  const uint64_t warp = (blockIdx.x * (uint64_t)kThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kThreads) >> 5;
  uint32_t first = 0, more = 0, maxp = 0;
  for (uint64_t ch = warp; ch < n_chunks; ch += n_warps) {
    const uint64_t di = a.d0 + ch * 32 + lane;
    uint64_t pos = 0;
    uint32_t nw = 0;
    if (di < a.d1) {
      const uint64_t d = __ldg(a.desc + di);
      pos = d >> kNwinBits;
      nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
    }
    const uint32_t incl = warp_incl_scan(nw), excl = incl - nw;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
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
      if (i < total) {
        uint64_t x[W], r[W], c[W];
        extract_kmer<W>(a.codes, pj + (i - ej), a.k, x);
        reverse_complement<W>(x, a.k, r);
        const bool use_r = key_less<W>(r, x);
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] = use_r ? r[w] : x[w];
        const uint32_t p = table_insert<W>(a.t, c, key_hash<W>(c));
        if (p == 0) {
          emergency<W>(a.t, c);
        } else if (p == 1) {
          ++first;
        } else {
          ++more;
          maxp = max(maxp, p);
        }
      }
    }
  }
  flush_probe_stats(a.t, first, more, maxp);
}

// Emergency path: count the overflow k-mers exactly in a fresh table whose θ
// covers every bucket ("counted via a sorting and
// compression approach" — here a second, large-enough table).
template <int W>
__global__ void __launch_bounds__(kThreads) count_keys_kernel(CountKeysArgs a) {
  uint32_t first = 0, more = 0, maxp = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)kThreads + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * kThreads) {
    uint64_t c[W];
#pragma unroll
    for (int w = 0; w < W; ++w) c[w] = a.keys[i * W + w];
    const uint32_t p = table_insert<W>(a.t, c, key_hash<W>(c));
    if (p == 0) emergency<W>(a.t, c);
    else if (p == 1) ++first;
    else { ++more; maxp = max(maxp, p); }
  }
  flush_probe_stats(a.t, first, more, maxp);
}

template <int W>
cudaError_t launch_count_w(const CountArgs& a, int sms, cudaStream_t st) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_kernel<W>, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const uint64_t chunks = (a.d1 - a.d0 + 31) / 32;
  uint64_t grid = (uint64_t)sms * per_sm;
  const uint64_t need = (chunks + kThreads / 32 - 1) / (kThreads / 32);
  if (grid > need) grid = need;
  if (grid == 0) return cudaSuccess;
  count_kernel<W><<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

template <int W>
cudaError_t launch_count_keys_w(const CountKeysArgs& a, int sms, cudaStream_t st) {
  uint64_t grid = (a.n + kThreads - 1) / kThreads;
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  if (grid == 0) return cudaSuccess;
  count_keys_kernel<W><<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_count(const CountArgs& a, uint32_t W, int sms, cudaStream_t st) {
  if (a.d1 <= a.d0) return cudaSuccess;
  switch (W) {
    case 1: return launch_count_w<1>(a, sms, st);
    case 2: return launch_count_w<2>(a, sms, st);
    case 3: return launch_count_w<3>(a, sms, st);
    case 4: return launch_count_w<4>(a, sms, st);
    case 5: return launch_count_w<5>(a, sms, st);
    case 6: return launch_count_w<6>(a, sms, st);
    case 7: return launch_count_w<7>(a, sms, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_count_keys(const CountKeysArgs& a, uint32_t W, int sms, cudaStream_t st) {
  switch (W) {
    case 1: return launch_count_keys_w<1>(a, sms, st);
    case 2: return launch_count_keys_w<2>(a, sms, st);
    case 3: return launch_count_keys_w<3>(a, sms, st);
    case 4: return launch_count_keys_w<4>(a, sms, st);
    case 5: return launch_count_keys_w<5>(a, sms, st);
    case 6: return launch_count_keys_w<6>(a, sms, st);
    case 7: return launch_count_keys_w<7>(a, sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gerbil
