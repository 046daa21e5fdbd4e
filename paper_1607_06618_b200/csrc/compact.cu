// compact.cu — step (e): min-count compaction of a wave's table.
//
// PAPER.md:115 (§2.3.2 step 3): "After a temporary file has been completely
// processed, each hasher thread sends the content of its hash table to an
// output buffer"; PAPER.md:467 (`-l count`): "the minimal occurrence of a
// k-mer to be outputted" (reading Q5: output iff count >= min_count).
//
// Each CTA iteration covers 1024 slots (4 per thread). Keepers are ranked
// with warp ballots and one global atomic per CTA iteration reserves their
// output range; keys are converted from table chunks back to the W-word
// result layout (include/gerbil.h). The same pass sums every count (Σ-count
// invariant), counts distinct keys, and clears the slots it
// read, so the L2-resident table buffer is clean for the next wave.
#include "common.cuh"
#include "kernels.h"
#include "table.cuh"
#include "table_inline.cuh"

namespace gerbil {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPer = 4;

__global__ void __launch_bounds__(kThreads) compact_kernel(CompactArgs a) {
  __shared__ uint32_t s_cnt[kWarps * kPer];
  __shared__ unsigned long long s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t W = key_words(a.k);
  const bool inl = table_inline(a.k);
  const uint32_t WP = inl ? (a.k > 31 ? 2 : 1) : chunk_words(a.k);
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  uint64_t my_sum = 0, my_distinct = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kPer; base < n_slots;
       base += (uint64_t)gridDim.x * kThreads * kPer) {
    uint64_t c0[kPer], c1[kPer];
    uint32_t cnt[kPer], rank[kPer];
    bool keep[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint64_t slot = base + j * kThreads + tid;
      c0[j] = 0;
      c1[j] = 0;
      cnt[j] = 0;
      if (slot < n_slots) {
        if (inl) {  // 16-byte slot {chunk0, chunk1 | count}
          const uint64_t* p = reinterpret_cast<const uint64_t*>(a.table) + 2 * slot;
          c0[j] = p[0];
          c1[j] = p[1];
          cnt[j] = (uint32_t)c1[j];
        } else {
          const Bucket bk = bucket_at(a.table, slot >> 2, WP);
          c0[j] = bk.c0[slot & 3];
          if (c0[j]) cnt[j] = bk.cnt[slot & 3];
        }
      }
      keep[j] = c0[j] != 0 && cnt[j] >= a.min_count;
      const uint32_t m = __ballot_sync(0xffffffffu, keep[j]);
      rank[j] = __popc(m & ((1u << lane) - 1u));
      if (lane == 0) s_cnt[j * kWarps + warp] = __popc(m);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t run = 0;
      for (int i = 0; i < kWarps * kPer; ++i) {
        const uint32_t v = s_cnt[i];
        s_cnt[i] = run;
        run += v;
      }
      s_base = run ? atomicAdd(a.out_n, (unsigned long long)run) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (!c0[j]) continue;
      const uint64_t slot = base + j * kThreads + tid;
      const Bucket bk = bucket_at(a.table, slot >> 2, WP);
      const uint32_t s = slot & 3;
      if (keep[j]) {
        const uint64_t idx = s_base + s_cnt[j * kWarps + warp] + rank[j];
        if (idx < a.cap) {
          uint64_t ch[8], key[kMaxW];
          ch[0] = c0[j];
          if (inl) {
            ch[1] = c1[j] & 0xffffffff00000000ull;
          } else {
            for (uint32_t q = 1; q < WP; ++q) ch[q] = bk.rest[s * (WP - 1) + (q - 1)];
          }
          from_chunks(ch, WP, key, W);
          for (uint32_t w = 0; w < W; ++w) a.out_keys[idx * W + w] = key[w];
          a.out_counts[idx] = cnt[j];
        }
      }
      my_sum += cnt[j];
      ++my_distinct;
      if (inl) {
        uint64_t* p = reinterpret_cast<uint64_t*>(a.table) + 2 * slot;
        p[0] = 0ull;
        p[1] = 0ull;
      } else {
        bk.c0[s] = 0ull;
        bk.cnt[s] = 0u;
        for (uint32_t q = 1; q < WP; ++q) bk.rest[s * (WP - 1) + (q - 1)] = 0ull;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_sum += __shfl_down_sync(0xffffffffu, my_sum, o);
    my_distinct += __shfl_down_sync(0xffffffffu, my_distinct, o);
  }
  if (lane == 0 && my_distinct) {
    atomicAdd(a.sum_counts, (unsigned long long)my_sum);
    atomicAdd(a.distinct, (unsigned long long)my_distinct);
    if (a.wave_distinct) atomicAdd(a.wave_distinct, (unsigned long long)my_distinct);
  }
}

// Inline table kind (k <= 46): 16-byte slots read and cleared with one vector
// access each, W-word keys written with one vector store (W = 2) — every
// store covers whole 32-byte sectors across the warp.
constexpr int kPerI = 8;

template <int W, bool TWO>
__global__ void __launch_bounds__(kThreads) compact_inline_kernel(CompactArgs a) {
  __shared__ uint32_t s_cnt[kWarps * kPerI];
  __shared__ unsigned long long s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  ulonglong2* slots = reinterpret_cast<ulonglong2*>(a.table);
  uint64_t my_sum = 0, my_distinct = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kPerI; base < n_slots;
       base += (uint64_t)gridDim.x * kThreads * kPerI) {
    ulonglong2 v[kPerI];
    uint32_t rank[kPerI];
    uint32_t keepm = 0;
#pragma unroll
    for (int j = 0; j < kPerI; ++j) {
      const uint64_t slot = base + j * kThreads + tid;
      v[j] = slot < n_slots ? slots[slot] : make_ulonglong2(0ull, 0ull);
      const bool keep = v[j].x != 0ull && (uint32_t)v[j].y >= a.min_count;
      keepm |= (uint32_t)keep << j;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      rank[j] = __popc(m & ((1u << lane) - 1u));
      if (lane == 0) s_cnt[j * kWarps + warp] = __popc(m);
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the kWarps*kPerI counts (<= 64) by one warp
      const uint32_t x0 = tid < kWarps * kPerI ? s_cnt[tid] : 0u;
      const uint32_t x1 = tid + 32 < kWarps * kPerI ? s_cnt[tid + 32] : 0u;
      uint32_t i0 = x0, i1 = x1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= (uint32_t)o) { i0 += t0; i1 += t1; }
      }
      const uint32_t tot0 = __shfl_sync(0xffffffffu, i0, 31);
      if (tid < kWarps * kPerI) s_cnt[tid] = i0 - x0;
      if (tid + 32 < kWarps * kPerI) s_cnt[tid + 32] = tot0 + i1 - x1;
      const uint32_t run = tot0 + __shfl_sync(0xffffffffu, i1, 31);
      if (tid == 0) s_base = run ? atomicAdd(a.out_n, (unsigned long long)run) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPerI; ++j) {
      if (v[j].x == 0ull) continue;
      const uint64_t slot = base + j * kThreads + tid;
      const uint32_t cnt = (uint32_t)v[j].y;
      if ((keepm >> j) & 1u) {
        const uint64_t idx = s_base + s_cnt[j * kWarps + warp] + rank[j];
        if (idx < a.cap) {
          uint64_t ch[2] = {v[j].x, TWO ? (v[j].y & 0xffffffff00000000ull) : 0ull}, key[2];
          from_chunks(ch, TWO ? 2u : 1u, key, (uint32_t)W);
          if (W == 2) reinterpret_cast<ulonglong2*>(a.out_keys)[idx] = make_ulonglong2(key[0], key[1]);
          else a.out_keys[idx] = key[0];
          a.out_counts[idx] = cnt;
        }
      }
      my_sum += cnt;
      ++my_distinct;
      slots[slot] = make_ulonglong2(0ull, 0ull);
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_sum += __shfl_down_sync(0xffffffffu, my_sum, o);
    my_distinct += __shfl_down_sync(0xffffffffu, my_distinct, o);
  }
  if (lane == 0 && my_distinct) {
    atomicAdd(a.sum_counts, (unsigned long long)my_sum);
    atomicAdd(a.distinct, (unsigned long long)my_distinct);
    if (a.wave_distinct) atomicAdd(a.wave_distinct, (unsigned long long)my_distinct);
  }
}

}  // namespace

cudaError_t launch_compact(const CompactArgs& a, int sms, cudaStream_t st) {
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  if (n_slots == 0) return cudaSuccess;
  if (table_inline(a.k)) {
    uint64_t grid = (n_slots + kThreads * kPerI - 1) / (kThreads * kPerI);
    if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
    if (a.k <= 31) compact_inline_kernel<1, false><<<(unsigned)grid, kThreads, 0, st>>>(a);
    else if (a.k == 32) compact_inline_kernel<1, true><<<(unsigned)grid, kThreads, 0, st>>>(a);
    else compact_inline_kernel<2, true><<<(unsigned)grid, kThreads, 0, st>>>(a);
    return cudaGetLastError();
  }
  uint64_t grid = (n_slots + kThreads * kPer - 1) / (kThreads * kPer);
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  compact_kernel<<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_clear_table(unsigned char* table, uint64_t bytes, int, cudaStream_t st) {
  return cudaMemsetAsync(table, 0, bytes, st);
}

}  // namespace gerbil
