// shuffle.cu — step (c), local part: group super-mer descriptors by bin.
//
// PAPER.md:49 ("all occurrences of a certain k-mer are stored in the same
// temporary file") and :97 (single writer fills the temporary files). Here the
// "files" are bin-contiguous ranges of a descriptor array in HBM: a counting
// sort with per-bin cursors pre-set to the bin offsets (exclusive scan of the
// per-bin super-mer counts from step (b)). Each CTA ranks its chunk inside
// shared memory and reserves one global range per (CTA chunk, bin), so global
// atomics scale with distinct bins per chunk, not with super-mers. Order
// inside a bin is unspecified (counting is order-insensitive).
// For world > 1 the same kernel regroups received descriptors (pos_add
// rebases them into the receive buffer) and builds the per-destination send
// order (bin index = dest * n_bins + bin, see api.cu).
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>
#include <type_traits>

namespace gerbil {
namespace {

// kThreads x kPer descriptors per CTA chunk: one global atomic per (chunk, distinct bin),
// so many bins want big chunks (2048 for <= 2048 bins, 8192 above).
template <int kThreads, int kPer>
__global__ void __launch_bounds__(kThreads)
scatter_smem_kernel(ScatterArgs a, uint64_t n_chunks) {
  constexpr int kChunk = kThreads * kPer;
  extern __shared__ uint32_t s_mem[];
  uint32_t* s_cnt = s_mem;                                   // [n_bins]
  const uint32_t nb = ((a.n_bins - 1) >> a.bin_shift) + 1;  // groups (bins when bin_shift == 0)
  unsigned long long* s_base = (unsigned long long*)(s_mem + ((nb + 1) & ~1u));
  const uint32_t tid = threadIdx.x;
  for (uint32_t b = tid; b < nb; b += kThreads) s_cnt[b] = 0;
  __syncthreads();
  for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const uint64_t i0 = c * kChunk;
    uint32_t bins[kPer], rank[kPer];
    uint64_t desc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint64_t i = i0 + j * kThreads + tid;
      bins[j] = 0xffffffffu;
      if (i < a.n) {
        const uint32_t b = a.bin_in[i] >> a.bin_shift;
        if (!a.keep || a.keep[b]) {
          bins[j] = b;
          desc[j] = a.desc_in[i];
          rank[j] = atomicAdd(&s_cnt[b], 1u);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (bins[j] != 0xffffffffu && rank[j] == 0)
        s_base[bins[j]] = atomicAdd(&a.cursor[bins[j]], (unsigned long long)s_cnt[bins[j]]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (bins[j] != 0xffffffffu) {
        const uint64_t d = s_base[bins[j]] + rank[j];
        if (a.pack_low_bits) {  // one 8-byte store per descriptor: the fine bin rides in bits 54..
          const uint32_t full = a.bin_in[i0 + j * kThreads + tid];
          a.desc_out[d] = desc[j] | ((uint64_t)(full & ((1u << a.pack_low_bits) - 1u)) << kDescPackShift);
        } else {
          a.desc_out[d] = desc[j] + (a.pos_add << kNwinBits);
          if (a.bin_out) a.bin_out[d] = a.bin_shift ? a.bin_in[i0 + j * kThreads + tid] : bins[j];
        }
      }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (bins[j] != 0xffffffffu && rank[j] == 0) s_cnt[bins[j]] = 0;
    __syncthreads();
  }
}

__global__ void scatter_global_kernel(ScatterArgs a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = a.bin_in[i] >> a.bin_shift;
    if (a.keep && !a.keep[b]) continue;
    const uint64_t d = atomicAdd(&a.cursor[b], 1ull);
    a.desc_out[d] = a.desc_in[i] + (a.pos_add << kNwinBits);
    if (a.bin_out) a.bin_out[d] = a.bin_in[i];
  }
}

__global__ void pack_kernel(PackArgs a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = a.desc_in[i];
    const uint32_t b = a.bin_in[i];
    const uint64_t pos = d >> kNwinBits;
    const uint32_t nwin = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
    const uint64_t L = nwin + a.k - 1;
    const uint32_t nw = (uint32_t)((L + 31) / 32);
    const uint64_t j = atomicAdd(&a.cur_desc[b], 1ull);
    const uint64_t wo = atomicAdd(&a.cur_words[b], (unsigned long long)nw);
    a.send_desc[j] = (((wo - a.seg_word_base[b]) * 32) << kNwinBits) | (nwin - 1);
    a.send_bin[j] = b;
    for (uint32_t t = 0; t < nw; ++t) {
      const uint64_t q = pos + 32ull * t;
      const uint64_t e = (q + 32 < pos + L) ? q + 32 : pos + L;  // bases [q, e)
      const uint64_t w0 = q >> 5;
      const uint32_t s = (uint32_t)(q & 31) * 2;
      const uint64_t hi = __ldg(a.codes + w0);
      const uint64_t lo = (((e - 1) >> 5) > w0) ? __ldg(a.codes + w0 + 1) : 0ull;
      uint64_t v = s ? ((hi << s) | (lo >> (64 - s))) : hi;
      const uint32_t nb = (uint32_t)(e - q);
      if (nb < 32) v &= ~0ull << (64 - 2 * nb);
      a.send_payload[wo + t] = v;
    }
  }
}

constexpr int kFineThreads = 512;

__global__ void __launch_bounds__(kFineThreads) regroup_fine_kernel(const uint64_t* __restrict__ desc_in,
                                                                    const uint32_t* __restrict__ bin_in,
                                                                    const unsigned long long* __restrict__ off,
                                                                    uint32_t n_bins, uint32_t shift,
                                                                    uint64_t* __restrict__ desc_out) {
  extern __shared__ uint32_t s_cur[];  // [1 << shift] cursors relative to the group's first descriptor
  const uint32_t g = blockIdx.x, fan = 1u << shift, b0 = g << shift;
  const uint32_t b1 = min(b0 + fan, n_bins);
  const uint64_t i0 = off[b0], i1 = off[b1];
  for (uint32_t t = threadIdx.x; t < fan; t += blockDim.x) s_cur[t] = b0 + t < b1 ? (uint32_t)(off[b0 + t] - i0) : 0u;
  __syncthreads();
  for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const uint32_t b = bin_in[i] & (fan - 1u);
    const uint32_t p = atomicAdd(&s_cur[b], 1u);
    desc_out[i0 + p] = desc_in[i];
  }
}

__global__ void __launch_bounds__(kFineThreads) regroup_fine_packed_kernel(const uint64_t* __restrict__ desc_in,
                                                                           const unsigned long long* __restrict__ off,
                                                                           uint32_t n_bins, uint32_t shift,
                                                                           uint64_t* __restrict__ desc_out) {
  extern __shared__ uint32_t s_cur[];  // [1 << shift] cursors relative to the group's first descriptor
  const uint32_t g = blockIdx.x, fan = 1u << shift, b0 = g << shift;
  const uint32_t b1 = min(b0 + fan, n_bins);
  const uint64_t i0 = off[b0], i1 = off[b1];
  for (uint32_t t = threadIdx.x; t < fan; t += blockDim.x) s_cur[t] = b0 + t < b1 ? (uint32_t)(off[b0 + t] - i0) : 0u;
  __syncthreads();
  constexpr uint64_t kLow = (1ull << kDescPackShift) - 1;
  for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const uint64_t d = desc_in[i];
    const uint32_t p = atomicAdd(&s_cur[(uint32_t)(d >> kDescPackShift)], 1u);
    desc_out[i0 + p] = d & kLow;
  }
}

// ---- group-major bin shuffle (single rank, many bins) -------------------------------
// Super-mers are grouped by bin in three passes, none with a per-super-mer global atomic:
//   0. group histogram: counts per group g = bin >> 10 (<= 4096 groups), one shared-memory
//      histogram per CTA;
//   A. partition by the group's high digit g >> 6 (64 buckets), B. partition every
//      high-digit segment by the low digit g & 63 (64 buckets): a chunk ranks its elements
//      per bucket with warp-aggregated shared-memory counters, reserves one global range per
//      (chunk, bucket), stages the chunk bucket-major in shared memory and writes runs
//      (coalesced). Pass B stores 8 bytes: the fine bin (bin & 1023) rides in descriptor
//      bits 54.. (kDescPackShift);
//   C. per group: counts and windows of its 1024 fine bins (shared memory), their offsets and
//      windows to global memory (the bin plan's inputs), then the fine scatter.

constexpr int kGroupShift = 10;   // fine bins per group = 1024
constexpr int kDigits = 64;       // buckets per partition pass
constexpr int kPartThreads = 256;
#ifndef GERBIL_PART_PER
#define GERBIL_PART_PER 8  // elements per thread and chunk (registers: ~8 per element; 8 at 4 CTAs/SM beat 16 at 2)
#endif
constexpr int kPartPer = GERBIL_PART_PER;
constexpr int kPartChunk = kPartThreads * kPartPer;

__global__ void __launch_bounds__(256) group_hist_kernel(const uint32_t* __restrict__ bin, uint64_t n, uint32_t G,
                                                         unsigned long long* __restrict__ cnt) {
  extern __shared__ uint32_t s_h[];
  for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) s_h[g] = 0;
  __syncthreads();
  // 16-byte loads (4 bins) for the bulk, then the tail
  const uint64_t n4 = n / 4, stride = (uint64_t)gridDim.x * blockDim.x;
  const uint4* b4 = reinterpret_cast<const uint4*>(bin);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const uint4 v = __ldg(b4 + i);
    atomicAdd(&s_h[v.x >> kGroupShift], 1u);
    atomicAdd(&s_h[v.y >> kGroupShift], 1u);
    atomicAdd(&s_h[v.z >> kGroupShift], 1u);
    atomicAdd(&s_h[v.w >> kGroupShift], 1u);
  }
  for (uint64_t i = 4 * n4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(&s_h[__ldg(bin + i) >> kGroupShift], 1u);
  __syncthreads();
  for (uint32_t g = threadIdx.x; g < G; g += blockDim.x)
    if (s_h[g]) atomicAdd(&cnt[g], (unsigned long long)s_h[g]);
}

// One CTA: group offsets (exclusive scan of cnt[G], padded with the total up to
// 64 * n_seg + 1 entries), pass-A cursors (the high digits' first groups), pass-B cursors
// (every group's start), pass-B segment bounds and first chunk per segment.
__global__ void __launch_bounds__(1024) part_setup_kernel(const unsigned long long* __restrict__ cnt, uint32_t G,
                                                          uint32_t n_seg, unsigned long long* goff,
                                                          unsigned long long* cur_a, unsigned long long* cur_b,
                                                          unsigned long long* seg_b, unsigned long long* chunk_b,
                                                          uint64_t n, unsigned long long* seg_a,
                                                          unsigned long long* chunk_a) {
  __shared__ unsigned long long s_w[32];
  if (threadIdx.x == 0) {  // pass A: one segment [0, n)
    seg_a[0] = 0ull;
    seg_a[1] = n;
    chunk_a[0] = 0ull;
    chunk_a[1] = (n + kPartChunk - 1) / kPartChunk;
  }
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t padded = n_seg * kDigits;  // >= G
  const uint32_t per = (padded + 1023) / 1024;
  unsigned long long v[8];  // padded <= 4096 + 63 → per <= 5
  unsigned long long s = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t g = tid * per + j;
    v[j] = g < G ? cnt[g] : 0ull;
    s += v[j];
  }
  unsigned long long incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long x = s_w[lane], y = x;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= (uint32_t)o) y += t;
    }
    s_w[lane] = y - x;
  }
  __syncthreads();
  unsigned long long run = s_w[warp] + incl - s;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t g = tid * per + j;
    if (g < padded) {
      goff[g] = run;
      if (g < G) cur_b[g] = run;
      if ((g & (kDigits - 1)) == 0) {
        cur_a[g / kDigits] = run;
        seg_b[g / kDigits] = run;
      }
    }
    run += v[j];
  }
  if (tid == 1023) {
    goff[padded] = run;  // run = total
    seg_b[n_seg] = run;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long c = 0;
    for (uint32_t q = 0; q < n_seg; ++q) {
      chunk_b[q] = c;
      const unsigned long long len = seg_b[q + 1] - seg_b[q];
      c += (len + kPartChunk - 1) / kPartChunk;
    }
    chunk_b[n_seg] = c;
  }
}

// One partition pass (A: n_seg == 1 over [0, n); B: n_seg segments from seg[], chunks
// numbered per chunk_first[]). digit = (bin >> shift) & 63; cursors cur[seg * 64 + digit].
#ifndef GERBIL_PART_MINB
#define GERBIL_PART_MINB 4
#endif
template <bool PACK_OUT>
__global__ void __launch_bounds__(kPartThreads, GERBIL_PART_MINB) partition64_kernel(
    const uint64_t* __restrict__ desc_in, const uint32_t* __restrict__ bin_in, uint32_t n_seg,
    const unsigned long long* __restrict__ seg, const unsigned long long* __restrict__ chunk_first, uint32_t shift,
    unsigned long long* cur, uint64_t* __restrict__ desc_out, uint32_t* __restrict__ bin_out) {
  extern __shared__ uint64_t s_desc[];  // [kPartChunk], then u32 bins [kPartChunk]
  uint32_t* s_bin = reinterpret_cast<uint32_t*>(s_desc + kPartChunk);
  __shared__ uint32_t s_cnt[kDigits], s_loc[kDigits];
  __shared__ unsigned long long s_gb[kDigits];
  __shared__ unsigned long long s_chunk[65];
  const uint32_t tid = threadIdx.x, lane = lane_id();
  for (uint32_t q = tid; q <= n_seg; q += blockDim.x) s_chunk[q] = chunk_first[q];
  __syncthreads();
  const unsigned long long n_chunks = s_chunk[n_seg];
  for (unsigned long long c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    uint32_t sg = 0;  // segment of chunk c: last q with s_chunk[q] <= c
    for (uint32_t step = 32; step >= 1; step >>= 1)
      if (sg + step <= n_seg - 1 && s_chunk[sg + step] <= c) sg += step;
    const unsigned long long e = seg[sg + 1];
    const unsigned long long i0 = seg[sg] + (c - s_chunk[sg]) * kPartChunk;
    if (tid < kDigits) s_cnt[tid] = 0;
    __syncthreads();
    uint64_t d[kPartPer];
    uint32_t b[kPartPer], rk[kPartPer];
#pragma unroll
    for (int j = 0; j < kPartPer; ++j) {
      const unsigned long long i = i0 + j * kPartThreads + tid;
      const bool act = i < e;
      d[j] = act ? __ldg(desc_in + i) : 0ull;
      b[j] = act ? __ldg(bin_in + i) : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < kPartPer; ++j) {
      const bool act = b[j] != 0xffffffffu;
      const uint32_t dg = act ? (b[j] >> shift) & (kDigits - 1) : kDigits + lane;  // inactive lanes stay alone
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      const uint32_t leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (act && lane == leader) base = atomicAdd(&s_cnt[dg], (uint32_t)__popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      rk[j] = base + __popc(peers & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (tid < 32) {  // local exclusive offsets of the 64 buckets, global ranges
      const uint32_t x0 = s_cnt[2 * tid], x1 = s_cnt[2 * tid + 1];
      uint32_t incl = x0 + x1;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      const uint32_t ex = incl - x0 - x1;
      s_loc[2 * tid] = ex;
      s_loc[2 * tid + 1] = ex + x0;
      if (x0) s_gb[2 * tid] = atomicAdd(&cur[sg * kDigits + 2 * tid], (unsigned long long)x0);
      if (x1) s_gb[2 * tid + 1] = atomicAdd(&cur[sg * kDigits + 2 * tid + 1], (unsigned long long)x1);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPartPer; ++j) {
      if (b[j] == 0xffffffffu) continue;
      const uint32_t p = s_loc[(b[j] >> shift) & (kDigits - 1)] + rk[j];
      s_desc[p] = d[j];
      s_bin[p] = b[j];
    }
    __syncthreads();
    const uint32_t tot = e - i0 < (unsigned long long)kPartChunk ? (uint32_t)(e - i0) : (uint32_t)kPartChunk;
    for (uint32_t p = tid; p < tot; p += kPartThreads) {
      const uint32_t bb = s_bin[p];
      const uint32_t dg = (bb >> shift) & (kDigits - 1);
      const unsigned long long o = s_gb[dg] + (p - s_loc[dg]);
      if (PACK_OUT) {
        desc_out[o] = s_desc[p] | ((uint64_t)(bb & ((1u << kGroupShift) - 1u)) << kDescPackShift);
      } else {
        desc_out[o] = s_desc[p];
        bin_out[o] = bb;
      }
    }
    __syncthreads();
  }
}

// Pass C: one CTA per group. Fine-bin counts and windows, the bins' offsets/windows out,
// then the scatter into bin order (descriptor bits 54.. cleared).
#ifndef GERBIL_REGROUP_STAGE
#define GERBIL_REGROUP_STAGE 1
#endif
constexpr int kFineT = 512;
constexpr int kFineU = 8;
template <bool WIDE>  // WIDE: a fine bin may hold >= 2^32 windows (u64 shared counters, CAS loops)
__global__ void __launch_bounds__(kFineT) regroup_counted_kernel(const uint64_t* __restrict__ desc_in,
                                                                 const unsigned long long* __restrict__ goff,
                                                                 uint32_t n_bins, unsigned long long* __restrict__ off,
                                                                 unsigned long long* __restrict__ win,
                                                                 uint64_t* __restrict__ desc_out) {
  constexpr uint32_t kFan = 1u << kGroupShift;
  using WinT = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  __shared__ uint32_t s_cur[kFan];
  __shared__ WinT s_win[kFan];
  __shared__ uint32_t s_w[kFineT / 32];
  const uint32_t g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t b0 = g << kGroupShift;
  const unsigned long long i0 = goff[g], i1 = goff[g + 1];
  for (uint32_t t = tid; t < kFan; t += kFineT) {
    s_cur[t] = 0;
    s_win[t] = 0;
  }
  __syncthreads();
  constexpr uint64_t kLow = (1ull << kDescPackShift) - 1;
  for (unsigned long long base = i0; base < i1; base += (unsigned long long)kFineT * kFineU) {
    uint64_t d[kFineU];
#pragma unroll
    for (int u = 0; u < kFineU; ++u) {
      const unsigned long long i = base + u * kFineT + tid;
      d[u] = i < i1 ? __ldg(desc_in + i) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < kFineU; ++u)
      if (d[u] != ~0ull) {
        const uint32_t f = (uint32_t)(d[u] >> kDescPackShift);
        atomicAdd(&s_cur[f], 1u);
        atomicAdd(&s_win[f], (WinT)((d[u] & ((1u << kNwinBits) - 1)) + 1));
      }
  }
  __syncthreads();
  // exclusive scan of the 1024 counts: 2 per thread
  const uint32_t x0 = s_cur[2 * tid], x1 = s_cur[2 * tid + 1];
  uint32_t incl = x0 + x1;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = lane < kFineT / 32 ? s_w[lane] : 0u;
    uint32_t y = x;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= (uint32_t)o) y += t;
    }
    if (lane < kFineT / 32) s_w[lane] = y - x;
  }
  __syncthreads();
  const uint32_t ex = s_w[warp] + incl - x0 - x1;
  s_cur[2 * tid] = ex;
  s_cur[2 * tid + 1] = ex + x0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t b = b0 + 2 * tid + q;
    if (b < n_bins) {
      off[b] = i0 + (q ? ex + x0 : ex);
      win[b] = (unsigned long long)s_win[2 * tid + q];
    }
  }
  if (b0 + kFan >= n_bins && tid == 0) off[n_bins] = i1;  // the last group closes the offsets
  __syncthreads();
#if GERBIL_REGROUP_STAGE
  // scatter in chunks of kFineT * kU descriptors staged in shared memory in fine-bin order:
  // a bin's run of the chunk then leaves as consecutive 8-byte stores (round 2: one scattered
  // store per descriptor left DRAM writes at ~2x the bytes)
  constexpr int kU = WIDE ? kFineU / 2 : kFineU;  // WIDE: u64 window counters leave less room
  __shared__ uint64_t s_stage[kFineT * kU];
  __shared__ uint32_t s_lc[kFan];  // the chunk's count per fine bin, then its local offset
  for (unsigned long long base = i0; base < i1; base += (unsigned long long)kFineT * kU) {
    uint64_t d[kU];
    uint32_t r[kU];
    for (uint32_t t = tid; t < kFan; t += kFineT) s_lc[t] = 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned long long i = base + u * kFineT + tid;
      d[u] = i < i1 ? __ldg(desc_in + i) : ~0ull;
      if (d[u] != ~0ull) r[u] = atomicAdd(&s_lc[(uint32_t)(d[u] >> kDescPackShift)], 1u);
    }
    __syncthreads();
    // exclusive scan of the chunk's 1024 counts (2 per thread), kept beside the counts
    const uint32_t c0 = s_lc[2 * tid], c1 = s_lc[2 * tid + 1];
    uint32_t in2 = c0 + c1;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, in2, o);
      if (lane >= (uint32_t)o) in2 += t;
    }
    if (lane == 31) s_w[warp] = in2;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = lane < kFineT / 32 ? s_w[lane] : 0u;
      uint32_t y = x;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= (uint32_t)o) y += t;
      }
      if (lane < kFineT / 32) s_w[lane] = y - x;
    }
    __syncthreads();
    const uint32_t e2 = s_w[warp] + in2 - c0 - c1;
    s_lc[2 * tid] = e2;
    s_lc[2 * tid + 1] = e2 + c0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (d[u] != ~0ull) s_stage[s_lc[(uint32_t)(d[u] >> kDescPackShift)] + r[u]] = d[u];
    __syncthreads();
    const uint32_t tot = i1 - base < (unsigned long long)(kFineT * kU) ? (uint32_t)(i1 - base) : kFineT * kU;
    for (uint32_t x = tid; x < tot; x += kFineT) {
      const uint64_t v = s_stage[x];
      const uint32_t f = (uint32_t)(v >> kDescPackShift);
      desc_out[i0 + s_cur[f] + (x - s_lc[f])] = v & kLow;
    }
    __syncthreads();
    // the chunk's runs are placed: advance the bins' cursors (2 bins per thread)
    s_cur[2 * tid] += c0;
    s_cur[2 * tid + 1] += c1;
    __syncthreads();
  }
#else
  for (unsigned long long base = i0; base < i1; base += (unsigned long long)kFineT * kFineU) {
    uint64_t d[kFineU];
    uint32_t p[kFineU];
#pragma unroll
    for (int u = 0; u < kFineU; ++u) {
      const unsigned long long i = base + u * kFineT + tid;
      d[u] = i < i1 ? __ldg(desc_in + i) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < kFineU; ++u)
      if (d[u] != ~0ull) p[u] = atomicAdd(&s_cur[(uint32_t)(d[u] >> kDescPackShift)], 1u);
#pragma unroll
    for (int u = 0; u < kFineU; ++u)
      if (d[u] != ~0ull) desc_out[i0 + p[u]] = d[u] & kLow;
  }
#endif
}

// ---- multi-rank exchange of whole groups (a group = 1024 consecutive bins) ----------------
// group_stats: per group g of the bin-ordered descriptors: windows, super-mers and the payload
// words its super-mers take once relocated (ceil((nwin + k - 1) / 32) each), laid out
// [3][G] like the histograms of exchange_plan.
__global__ void __launch_bounds__(256) group_stats_kernel(const uint64_t* __restrict__ desc,
                                                          const unsigned long long* __restrict__ off,
                                                          uint32_t n_bins, uint32_t k, unsigned long long* st) {
  const uint32_t g = blockIdx.x, G = gridDim.x;
  const uint32_t b0 = g << kGroupShift, b1 = min(b0 + (1u << kGroupShift), n_bins);
  const unsigned long long i0 = off[b0], i1 = off[b1];
  unsigned long long w = 0, pw = 0;
  for (unsigned long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const uint32_t nw = (uint32_t)(__ldg(desc + i) & ((1u << kNwinBits) - 1)) + 1;
    w += nw;
    pw += (nw + k - 1 + 31) / 32;
  }
  __shared__ unsigned long long s_w[8], s_p[8];
  for (int o = 16; o > 0; o >>= 1) {
    w += __shfl_xor_sync(0xffffffffu, w, o);
    pw += __shfl_xor_sync(0xffffffffu, pw, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_w[threadIdx.x >> 5] = w;
    s_p[threadIdx.x >> 5] = pw;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tw = 0, tp = 0;
    for (int q = 0; q < 8; ++q) {
      tw += s_w[q];
      tp += s_p[q];
    }
    st[g] = tw;
    st[G + g] = i1 - i0;
    st[2 * G + g] = tp;
  }
}

// group_pack: one CTA per group copies the group's super-mers into the send buffers at the
// group's place in its owner's segment: descriptor (position rebased to the owner's receive
// payload buffer: abs_word[g] words plus the super-mer's offset inside the group), its bin,
// and the payload (bases [pos, pos + nwin + k - 1) re-aligned to word boundaries).
__global__ void __launch_bounds__(256) group_pack_kernel(const uint64_t* __restrict__ desc,
                                                         const unsigned long long* __restrict__ off,
                                                         uint32_t n_bins, const uint64_t* __restrict__ codes,
                                                         uint32_t k, const unsigned long long* __restrict__ base3,
                                                         uint64_t* __restrict__ send_desc,
                                                         uint32_t* __restrict__ send_bin,
                                                         uint64_t* __restrict__ send_payload) {
  constexpr uint32_t kFan = 1u << kGroupShift;
  __shared__ unsigned long long s_off[kFan + 1];
  __shared__ uint32_t s_wsum[8];
  const uint32_t g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t b0 = g << kGroupShift, nb = min(kFan, n_bins - b0);
  for (uint32_t t = tid; t <= nb; t += blockDim.x) s_off[t] = off[b0 + t];
  __syncthreads();
  const unsigned long long i0 = s_off[0], i1 = s_off[nb];
  const unsigned long long dbase = base3[g], wbase = base3[G + g], abase = base3[2 * G + g];
  unsigned long long run = 0;  // payload words of the group's earlier super-mers
  for (unsigned long long c0 = i0; c0 < i1; c0 += blockDim.x) {
    const unsigned long long i = c0 + tid;
    uint64_t d = 0;
    uint32_t nw = 0, wds = 0;
    if (i < i1) {
      d = __ldg(desc + i);
      nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
      wds = (nw + k - 1 + 31) / 32;
    }
    uint32_t incl = wds;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t wex = 0, tot = 0;
    for (uint32_t q = 0; q < blockDim.x / 32; ++q) {
      if (q < warp) wex += s_wsum[q];
      tot += s_wsum[q];
    }
    const unsigned long long woff = run + wex + incl - wds;
    if (i < i1) {
      // bin: the last f with s_off[f] <= i (bins of the group are consecutive ranges)
      uint32_t f = 0;
      for (uint32_t step = kFan >> 1; step >= 1; step >>= 1)
        if (f + step < nb && s_off[f + step] <= i) f += step;
      const uint64_t pos = d >> kNwinBits, L = nw + k - 1;
      uint64_t* dst = send_payload + wbase + woff;
      for (uint32_t u = 0; u < wds; ++u) {
        const uint64_t q = pos + 32ull * u;
        const uint64_t e = (q + 32 < pos + L) ? q + 32 : pos + L;  // bases [q, e)
        const uint64_t w0 = q >> 5;
        const uint32_t sh = (uint32_t)(q & 31) * 2;
        const uint64_t hi = __ldg(codes + w0);
        const uint64_t lo = (((e - 1) >> 5) > w0) ? __ldg(codes + w0 + 1) : 0ull;
        uint64_t v = sh ? ((hi << sh) | (lo >> (64 - sh))) : hi;
        const uint32_t nbs = (uint32_t)(e - q);
        if (nbs < 32) v &= ~0ull << (64 - 2 * nbs);
        dst[u] = v;
      }
      const unsigned long long j = dbase + (i - i0);
      send_desc[j] = (((abase + woff) * 32ull) << kNwinBits) | (nw - 1);
      send_bin[j] = b0 + f;
    }
    run += tot;
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_group_stats(const uint64_t* desc, const unsigned long long* off, uint32_t n_bins, uint32_t k,
                               unsigned long long* st, cudaStream_t s) {
  const uint32_t G = ((n_bins - 1) >> kGroupShift) + 1;
  group_stats_kernel<<<G, 256, 0, s>>>(desc, off, n_bins, k, st);
  return cudaGetLastError();
}

cudaError_t launch_group_pack(const uint64_t* desc, const unsigned long long* off, uint32_t n_bins,
                              const uint64_t* codes, uint32_t k, const unsigned long long* base3, uint64_t* send_desc,
                              uint32_t* send_bin, uint64_t* send_payload, cudaStream_t s) {
  const uint32_t G = ((n_bins - 1) >> kGroupShift) + 1;
  group_pack_kernel<<<G, 256, 0, s>>>(desc, off, n_bins, codes, k, base3, send_desc, send_bin, send_payload);
  return cudaGetLastError();
}

uint32_t group_shuffle_groups(uint32_t n_bins) { return ((n_bins - 1) >> kGroupShift) + 1; }

cudaError_t launch_group_shuffle(const GroupShuffleArgs& a, int sms, cudaStream_t st) {
  const uint32_t G = group_shuffle_groups(a.n_bins);
  if (G > kDigits * kDigits) return cudaErrorInvalidValue;
  const uint32_t n_seg = (G + kDigits - 1) / kDigits;
  unsigned long long* cnt = a.scratch;                    // [G]
  unsigned long long* goff = cnt + G;                     // [64 n_seg + 1]
  unsigned long long* cur_a = goff + n_seg * kDigits + 1; // [64]
  unsigned long long* cur_b = cur_a + kDigits;            // [G]
  unsigned long long* seg_a = cur_b + G;                  // [2]
  unsigned long long* chunk_a = seg_a + 2;                // [2]
  unsigned long long* seg_b = chunk_a + 2;                // [n_seg + 1]
  unsigned long long* chunk_b = seg_b + n_seg + 1;        // [n_seg + 1]
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)G * 8, st);
  if (e != cudaSuccess) return e;
  if (a.n == 0) {
    e = cudaMemsetAsync(a.off, 0, ((size_t)a.n_bins + 1) * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.win, 0, (size_t)a.n_bins * 8, st);
    return e;
  }
  {
    const size_t dyn = (size_t)G * 4;
    e = cudaFuncSetAttribute(group_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    uint64_t grid = (a.n / 4 + 255) / 256 + 1;
    if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
    group_hist_kernel<<<(unsigned)grid, 256, dyn, st>>>(a.bin_in, a.n, G, cnt);
  }
  part_setup_kernel<<<1, 1024, 0, st>>>(cnt, G, n_seg, goff, cur_a, cur_b, seg_b, chunk_b, a.n, seg_a, chunk_a);
  constexpr size_t kPartSmem = (size_t)kPartChunk * 12;
  for (auto kern : {partition64_kernel<false>, partition64_kernel<true>}) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPartSmem);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, partition64_kernel<true>, kPartThreads, kPartSmem);
  if (per_sm < 1) per_sm = 1;
  const uint64_t max_chunks = (a.n + kPartChunk - 1) / kPartChunk + n_seg;
  uint64_t grid = (uint64_t)sms * per_sm;
  if (grid > max_chunks) grid = max_chunks;
  const uint64_t* pb_desc = a.desc_in;
  const uint32_t* pb_bin = a.bin_in;
  if (n_seg > 1) {  // pass A by the high digit
    partition64_kernel<false><<<(unsigned)grid, kPartThreads, kPartSmem, st>>>(
        a.desc_in, a.bin_in, 1, seg_a, chunk_a, kGroupShift + 6, cur_a, a.tmp_desc, a.tmp_bin);
    pb_desc = a.tmp_desc;
    pb_bin = a.tmp_bin;
  }
  uint64_t* packed = n_seg > 1 ? a.desc_alt : a.tmp_desc;  // pass B output: never its own input
  partition64_kernel<true><<<(unsigned)grid, kPartThreads, kPartSmem, st>>>(pb_desc, pb_bin, n_seg, seg_b, chunk_b,
                                                                   kGroupShift, cur_b, packed, nullptr);
  // the 64-bit-counter instance is needed only when a fine bin could reach 2^32 windows;
  // GERBIL_REGROUP_WIDE=1 forces it (tests)
  const char* fw = getenv("GERBIL_REGROUP_WIDE");  // read per call (tests set it in-process)
  const bool force_wide = fw && atoi(fw) == 1;
  if (a.max_windows >= (1ull << 32) || force_wide)
    regroup_counted_kernel<true><<<G, kFineT, 0, st>>>(packed, goff, a.n_bins, a.off, a.win, a.desc_out);
  else
    regroup_counted_kernel<false><<<G, kFineT, 0, st>>>(packed, goff, a.n_bins, a.off, a.win, a.desc_out);
  return cudaGetLastError();
}

size_t group_shuffle_scratch_bytes(uint32_t n_bins) {
  const uint32_t G = group_shuffle_groups(n_bins), n_seg = (G + kDigits - 1) / kDigits;
  return ((size_t)G * 2 + n_seg * kDigits + 1 + kDigits + 4 + 2 * ((size_t)n_seg + 1)) * 8;
}

cudaError_t launch_regroup_fine_packed(const uint64_t* desc_in, const unsigned long long* off, uint32_t n_bins,
                                       uint32_t shift, uint64_t* desc_out, cudaStream_t st) {
  const uint32_t groups = (n_bins + (1u << shift) - 1) >> shift;
  if (groups == 0) return cudaSuccess;
  regroup_fine_packed_kernel<<<groups, kFineThreads, (size_t)4 << shift, st>>>(desc_in, off, n_bins, shift,
                                                                                desc_out);
  return cudaGetLastError();
}

cudaError_t launch_regroup_fine(const uint64_t* desc_in, const uint32_t* bin_in, const unsigned long long* off,
                                uint32_t n_bins, uint32_t shift, uint64_t* desc_out, cudaStream_t st) {
  const uint32_t groups = (n_bins + (1u << shift) - 1) >> shift;
  if (groups == 0) return cudaSuccess;
  regroup_fine_kernel<<<groups, kFineThreads, (size_t)4 << shift, st>>>(desc_in, bin_in, off, n_bins, shift,
                                                                         desc_out);
  return cudaGetLastError();
}

cudaError_t launch_pack(const PackArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  pack_kernel<<<sms * 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}

namespace {
__global__ void rebase_desc_kernel(uint64_t* desc, uint64_t n, uint64_t pos_add) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    desc[i] += pos_add << kNwinBits;
}
}  // namespace

// In-place position rebase of n descriptors (pos += pos_add mod 2^64 >> kNwinBits): spilled
// chunks of several batches placed side by side in one send segment (spill.cu, world > 1).
cudaError_t launch_rebase_desc(uint64_t* desc, uint64_t n, uint64_t pos_add, int sms, cudaStream_t st) {
  if (n == 0 || pos_add == 0) return cudaSuccess;
  const uint64_t want = (n + 255) / 256, cap = (uint64_t)sms * 8;
  const uint64_t blocks = want < cap ? want : cap;
  rebase_desc_kernel<<<(unsigned)blocks, 256, 0, st>>>(desc, n, pos_add);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const ScatterArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  const uint32_t nb = ((a.n_bins - 1) >> a.bin_shift) + 1;  // groups the kernel sees
  if (nb <= 16384) {
    const size_t dyn = (size_t)((nb + 1) & ~1u) * 4 + (size_t)nb * 8;
    auto run = [&](auto kern, int threads, int per) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return e;
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, dyn);
      if (per_sm < 1) per_sm = 1;
      const uint64_t chunk = (uint64_t)threads * per;
      const uint64_t n_chunks = (a.n + chunk - 1) / chunk;
      uint64_t grid = (uint64_t)sms * per_sm;
      if (grid > n_chunks) grid = n_chunks;
      kern<<<(unsigned)grid, threads, dyn, st>>>(a, n_chunks);
      return cudaSuccess;
    };
    cudaError_t e = nb <= 2048 ? run(scatter_smem_kernel<256, 8>, 256, 8) : run(scatter_smem_kernel<1024, 8>, 1024, 8);
    if (e != cudaSuccess) return e;
  } else {
    scatter_global_kernel<<<sms * 8, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace gerbil
