// compact.cu — step (e): min-count compaction of a wave's table.
//
// PAPER.md:115 (§2.3.2 step 3): "After a temporary file has been completely
// processed, each hasher thread sends the content of its hash table to an
// output buffer"; PAPER.md:467 (`-l count`): "the minimal occurrence of a
// k-mer to be outputted" (reading Q5: output iff count >= min_count).
//
// One thread per slot; keepers are appended to the SoA result with one
// atomic per warp (ballot + popc). The same pass sums every count (Σ-count
// invariant), counts distinct keys, and clears the slots it
// read, so the (L2-resident) table buffer is clean for the next wave without
// a separate memset.
#include "common.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) compact_kernel(CompactArgs a) {
  const uint32_t lane = lane_id();
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  const uint64_t bb = bucket_bytes(a.W);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint64_t my_sum = 0, my_distinct = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads + (threadIdx.x & ~31u); base < n_slots;
       base += stride) {
    const uint64_t slot = base + lane;
    uint32_t tag = 0, cnt = 0;
    uint32_t* tags = nullptr;
    if (slot < n_slots) {
      unsigned char* bucket = a.table + (slot >> 3) * bb;
      tags = reinterpret_cast<uint32_t*>(bucket) + (slot & 7);
      tag = *tags;
      if (tag) cnt = tags[kSlotsPerBucket];
    }
    const bool keep = tag != 0u && cnt >= a.min_count;
    const uint32_t mask = __ballot_sync(0xffffffffu, keep);
    unsigned long long out0 = 0;
    if (mask) {
      if (lane == 0) out0 = atomicAdd(a.out_n, (unsigned long long)__popc(mask));
      out0 = __shfl_sync(0xffffffffu, out0, 0);
    }
    if (keep) {
      const uint64_t idx = out0 + __popc(mask & ((1u << lane) - 1u));
      if (idx < a.cap) {
        const uint64_t* key = reinterpret_cast<const uint64_t*>(
            a.table + (slot >> 3) * bb + 64) + (slot & 7) * a.W;
        for (uint32_t w = 0; w < a.W; ++w) a.out_keys[idx * a.W + w] = key[w];
        a.out_counts[idx] = cnt;
      }
    }
    if (tag) {
      my_sum += cnt;
      ++my_distinct;
      tags[0] = 0u;
      tags[kSlotsPerBucket] = 0u;
    }
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
  uint64_t grid = (n_slots + kThreads - 1) / kThreads;
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  compact_kernel<<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_clear_table(unsigned char* table, uint64_t bytes, int, cudaStream_t st) {
  return cudaMemsetAsync(table, 0, bytes, st);
}

}  // namespace gerbil
