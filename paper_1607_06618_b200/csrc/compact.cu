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
//
// Optionally (streaming e2e path) the same pass encodes every kept k-mer as
// the paper's binary record (App. C: 1-byte counter, or
// 0xFF + 32-bit big-endian counter when >= 255, then ceil(k/4) bytes of 2-bit
// bases MSB-first): records are placed in shared memory by the same block
// scan (at the destination's 16-byte phase), one atomic per CTA iteration
// reserves their byte range in the lane's HBM staging buffer, and the CTA
// writes it with aligned 16-byte stores; the host then has the copy engine
// move each wave's records to page-locked host memory behind the counting of
// the next waves (api.cu, gerbil_count_host_stream).
#include "common.cuh"
#include "kernels.h"
#include "table.cuh"
#include "table_inline.cuh"

namespace gerbil {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPer = 4;

__device__ __forceinline__ uint32_t record_bytes(uint32_t kb, uint32_t cnt) { return (cnt < 255 ? 1u : 5u) + kb; }

// App. C record of (key, cnt) at s[o..): counter, then the key's big-endian bytes
__device__ __forceinline__ void put_record(uint8_t* s, uint32_t o, const uint64_t* key, uint32_t kb, uint32_t cnt) {
  if (cnt < 255) {
    s[o++] = (uint8_t)cnt;
  } else {
    s[o++] = 0xFF;
    s[o++] = (uint8_t)(cnt >> 24);
    s[o++] = (uint8_t)(cnt >> 16);
    s[o++] = (uint8_t)(cnt >> 8);
    s[o++] = (uint8_t)cnt;
  }
  for (uint32_t b = 0; b < kb; ++b) s[o++] = (uint8_t)(key[b >> 3] >> (56 - 8 * (b & 7)));
}

// all threads: copy the staged range to out[dst0, dst0 + tot), unless it passes
// cap. The records were staged at smem offset dst0 % 16, so smem and the
// destination share their alignment: whole 16-byte blocks move with one vector
// load/store each, the (at most two) partial edge blocks byte by byte.
__device__ __forceinline__ void flush_records(const uint8_t* s, uint32_t tot, uint64_t dst0, uint8_t* out,
                                              uint64_t cap) {
  if (tot == 0 || dst0 + tot > cap) return;
  const uint32_t a0 = (uint32_t)(dst0 & 15), end = a0 + tot;
  uint8_t* base = out + (dst0 - a0);
  const uint32_t nblk = (end + 15) >> 4;
  for (uint32_t b = threadIdx.x; b < nblk; b += blockDim.x) {
    const uint32_t lo = b << 4, hi = lo + 16;
    if (lo >= a0 && hi <= end) {
      *reinterpret_cast<uint4*>(base + lo) = *reinterpret_cast<const uint4*>(s + lo);
    } else {
      for (uint32_t i = max(lo, a0); i < min(hi, end); ++i) base[i] = s[i];
    }
  }
}

__global__ void __launch_bounds__(kThreads) compact_kernel(CompactArgs a) {
  __shared__ uint32_t s_cnt[kWarps * kPer], s_big[kWarps * kPer];
  __shared__ unsigned long long s_base, s_rbase;
  __shared__ uint32_t s_rtot;
  extern __shared__ __align__(16) uint8_t s_rec[];  // [16 + kThreads * kPer * (5 + kb)] when a.rec_out
  const uint32_t kb = (a.k + 3) / 4;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t W = key_words(a.k);
  const bool inl = table_inline(a.k);
  const uint32_t WP = inl ? (a.k > 31 ? 2 : 1) : chunk_words(a.k);
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  uint64_t my_sum = 0, my_distinct = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kPer; base < n_slots;
       base += (uint64_t)gridDim.x * kThreads * kPer) {
    uint64_t c0[kPer], c1[kPer];
    uint32_t cnt[kPer], rank[kPer], brank[kPer];
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
      const uint32_t mb = __ballot_sync(0xffffffffu, keep[j] && cnt[j] >= 255);
      brank[j] = __popc(mb & ((1u << lane) - 1u));
      if (lane == 0) {
        s_cnt[j * kWarps + warp] = __popc(m);
        s_big[j * kWarps + warp] = __popc(mb);
      }
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t run = 0, runb = 0;
      for (int i = 0; i < kWarps * kPer; ++i) {
        const uint32_t v = s_cnt[i], vb = s_big[i];
        s_cnt[i] = run;
        s_big[i] = runb;
        run += v;
        runb += vb;
      }
      s_base = run ? atomicAdd(a.out_n, (unsigned long long)run) : 0ull;
      if (a.rec_out) {
        s_rtot = run * (1 + kb) + 4 * runb;
        s_rbase = s_rtot ? atomicAdd(a.rec_n, (unsigned long long)s_rtot) : 0ull;
      }
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
          uint64_t ch[kMaxW + 1], key[kMaxW];
          ch[0] = c0[j];
          if (inl) {
            ch[1] = c1[j] & 0xffffffff00000000ull;
          } else {
            for (uint32_t q = 1; q < WP; ++q) ch[q] = bk.rest[s * (WP - 1) + (q - 1)];
          }
          from_chunks(ch, WP, key, W);
          for (uint32_t w = 0; w < W; ++w) a.out_keys[idx * W + w] = key[w];
          a.out_counts[idx] = cnt[j];
          if (a.rec_out) {
            const uint32_t r = s_cnt[j * kWarps + warp] + rank[j], rb = s_big[j * kWarps + warp] + brank[j];
            put_record(s_rec, (uint32_t)(s_rbase & 15) + r * (1 + kb) + 4 * rb, key, kb, cnt[j]);
          }
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
    if (a.rec_out) {
      flush_records(s_rec, s_rtot, s_rbase, a.rec_out, a.rec_cap);
      __syncthreads();
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

// Inline table kind (k <= 46): 16-byte slots read and cleared with one vector
// access each, W-word keys written with one vector store (W = 2) — every
// store covers whole 32-byte sectors across the warp.
constexpr int kPerI = 8;

// one warp: exclusive scan in place of c[0..n) (n <= 64, two entries per lane); returns the total
__device__ __forceinline__ uint32_t excl_scan64(uint32_t* c, uint32_t n) {
  const uint32_t lane = lane_id();
  const uint32_t x0 = lane < n ? c[lane] : 0u;
  const uint32_t x1 = lane + 32 < n ? c[lane + 32] : 0u;
  uint32_t i0 = x0, i1 = x1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o);
    if (lane >= (uint32_t)o) {
      i0 += t0;
      i1 += t1;
    }
  }
  const uint32_t tot0 = __shfl_sync(0xffffffffu, i0, 31);
  if (lane < n) c[lane] = i0 - x0;
  if (lane + 32 < n) c[lane + 32] = tot0 + i1 - x1;
  return tot0 + __shfl_sync(0xffffffffu, i1, 31);
}

template <int W, bool TWO>
__global__ void __launch_bounds__(kThreads) compact_inline_kernel(CompactArgs a) {
  __shared__ uint32_t s_cnt[kWarps * kPerI], s_big[kWarps * kPerI];
  __shared__ unsigned long long s_base, s_rbase;
  __shared__ uint32_t s_rtot;
  extern __shared__ __align__(16) uint8_t s_rec[];  // [16 + kThreads * kPerI * (5 + kb)] when a.rec_out
  const uint32_t kb = (a.k + 3) / 4;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  ulonglong2* slots = reinterpret_cast<ulonglong2*>(a.table);
  uint64_t my_sum = 0, my_distinct = 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kPerI; base < n_slots;
       base += (uint64_t)gridDim.x * kThreads * kPerI) {
    ulonglong2 v[kPerI];
    uint32_t rank[kPerI], brank[kPerI];
    uint32_t keepm = 0;
#pragma unroll
    for (int j = 0; j < kPerI; ++j) {
      const uint64_t slot = base + j * kThreads + tid;
      v[j] = slot < n_slots ? slots[slot] : make_ulonglong2(0ull, 0ull);
      const bool keep = v[j].x != 0ull && (uint32_t)v[j].y >= a.min_count;
      keepm |= (uint32_t)keep << j;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      rank[j] = __popc(m & ((1u << lane) - 1u));
      const uint32_t mb = __ballot_sync(0xffffffffu, keep && (uint32_t)v[j].y >= 255);
      brank[j] = __popc(mb & ((1u << lane) - 1u));
      if (lane == 0) {
        s_cnt[j * kWarps + warp] = __popc(m);
        s_big[j * kWarps + warp] = __popc(mb);
      }
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scans of the kWarps*kPerI (<= 64) keep / big counts by one warp
      const uint32_t run = excl_scan64(s_cnt, kWarps * kPerI);
      const uint32_t runb = excl_scan64(s_big, kWarps * kPerI);
      if (tid == 0) {
        s_base = run ? atomicAdd(a.out_n, (unsigned long long)run) : 0ull;
        if (a.rec_out) {
          s_rtot = run * (1 + kb) + 4 * runb;
          s_rbase = s_rtot ? atomicAdd(a.rec_n, (unsigned long long)s_rtot) : 0ull;
        }
      }
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
          if (a.rec_out) {
            const uint32_t r = s_cnt[j * kWarps + warp] + rank[j], rb = s_big[j * kWarps + warp] + brank[j];
            put_record(s_rec, (uint32_t)(s_rbase & 15) + r * (1 + kb) + 4 * rb, key, kb, cnt);
          }
        }
      }
      my_sum += cnt;
      ++my_distinct;
      slots[slot] = make_ulonglong2(0ull, 0ull);
    }
    __syncthreads();
    if (a.rec_out) {
      flush_records(s_rec, s_rtot, s_rbase, a.rec_out, a.rec_cap);
      __syncthreads();
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

// App. C records of results [*lo, *hi) of a result array (shared-memory / reference passes
// write (key, count) arrays; the streaming call turns each slice of them into records here):
// per CTA iteration the records are sized, block-scanned, reserved with one atomic on
// *rec_n and written through shared memory with aligned 16-byte stores (flush_records).
__global__ void __launch_bounds__(kThreads) encode_records_kernel(const uint64_t* __restrict__ keys,
                                                                  const uint32_t* __restrict__ counts,
                                                                  const unsigned long long* lo,
                                                                  const unsigned long long* hi, uint32_t k,
                                                                  uint8_t* rec, uint64_t rec_cap,
                                                                  unsigned long long* rec_n) {
  __shared__ uint32_t s_w[kWarps];
  __shared__ unsigned long long s_rbase;
  __shared__ uint32_t s_rtot;
  extern __shared__ __align__(16) uint8_t s_rec[];  // [16 + kThreads * kPer * (5 + kb)]
  const uint32_t kb = (k + 3) / 4, W = key_words(k);
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const unsigned long long e0 = *lo, e1 = *hi;
  for (unsigned long long base = e0 + (uint64_t)blockIdx.x * kThreads * kPer; base < e1;
       base += (uint64_t)gridDim.x * kThreads * kPer) {
    // thread tid owns entries base + tid*kPer .. +kPer (contiguous: one scan value per thread)
    uint32_t sz = 0, cnt[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const unsigned long long e = base + (uint64_t)tid * kPer + j;
      cnt[j] = e < e1 ? counts[e] : 0u;
      if (e < e1) sz += record_bytes(kb, cnt[j]);
    }
    uint32_t incl = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (tid == 0) {
      uint32_t run = 0;
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t v = s_w[w];
        s_w[w] = run;
        run += v;
      }
      s_rtot = run;
      s_rbase = run ? atomicAdd(rec_n, (unsigned long long)run) : 0ull;
    }
    __syncthreads();
    uint32_t o = (uint32_t)(s_rbase & 15) + s_w[warp] + incl - sz;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const unsigned long long e = base + (uint64_t)tid * kPer + j;
      if (e < e1) {
        put_record(s_rec, o, keys + e * W, kb, cnt[j]);
        o += record_bytes(kb, cnt[j]);
      }
    }
    __syncthreads();
    flush_records(s_rec, s_rtot, s_rbase, rec, rec_cap);
    __syncthreads();
  }
}

}  // namespace

// *dst = *src, dst in page-locked (mapped) host memory: a counter snapshot that does not queue
// behind the large record copies on the copy engine
__global__ void store_u64_kernel(unsigned long long* dst, const unsigned long long* src) {
  *reinterpret_cast<volatile unsigned long long*>(dst) = *reinterpret_cast<const volatile unsigned long long*>(src);
  __threadfence_system();
}
cudaError_t launch_store_u64(unsigned long long* dst_mapped, const unsigned long long* src, cudaStream_t st) {
  store_u64_kernel<<<1, 1, 0, st>>>(dst_mapped, src);
  return cudaGetLastError();
}

__global__ void copy_words_kernel(unsigned long long* dst, const unsigned long long* src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    reinterpret_cast<volatile unsigned long long*>(dst)[i] = src[i];
  __threadfence_system();
}
cudaError_t launch_copy_words_mapped(unsigned long long* dst_mapped, const unsigned long long* src, uint64_t n,
                                     cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint64_t g = (n + 255) / 256;
  copy_words_kernel<<<(unsigned)(g < 64 ? g : 64), 256, 0, st>>>(dst_mapped, src, n);
  return cudaGetLastError();
}

cudaError_t launch_encode_records(const uint64_t* keys, const uint32_t* counts, const unsigned long long* lo,
                                  const unsigned long long* hi, uint64_t max_n, uint32_t k, uint8_t* rec,
                                  uint64_t rec_cap, unsigned long long* rec_n, int sms, cudaStream_t st) {
  if (max_n == 0) return cudaSuccess;
  const uint32_t rec_max = 5 + (k + 3) / 4;
  const size_t dyn = 16 + (size_t)kThreads * kPer * rec_max;
  cudaError_t e = cudaFuncSetAttribute(encode_records_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  uint64_t grid = (max_n + kThreads * kPer - 1) / (kThreads * kPer);
  if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
  encode_records_kernel<<<(unsigned)grid, kThreads, dyn, st>>>(keys, counts, lo, hi, k, rec, rec_cap, rec_n);
  return cudaGetLastError();
}

cudaError_t launch_compact(const CompactArgs& a, int sms, cudaStream_t st) {
  const uint64_t n_slots = a.nb * kSlotsPerBucket;
  if (n_slots == 0) return cudaSuccess;
  const uint32_t rec_max = 5 + (a.k + 3) / 4;  // largest App. C record
  if (table_inline(a.k)) {
    uint64_t grid = (n_slots + kThreads * kPerI - 1) / (kThreads * kPerI);
    if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
    const size_t dyn = a.rec_out ? 16 + (size_t)kThreads * kPerI * rec_max : 0;
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return e;
      kern<<<(unsigned)grid, kThreads, dyn, st>>>(a);
      return cudaGetLastError();
    };
    if (a.k <= 31) return go(compact_inline_kernel<1, false>);
    if (a.k == 32) return go(compact_inline_kernel<1, true>);
    return go(compact_inline_kernel<2, true>);
  }
  uint64_t grid = (n_slots + kThreads * kPer - 1) / (kThreads * kPer);
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  const size_t dyn = a.rec_out ? 16 + (size_t)kThreads * kPer * rec_max : 0;
  cudaError_t e = cudaFuncSetAttribute(compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  compact_kernel<<<(unsigned)grid, kThreads, dyn, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_clear_table(unsigned char* table, uint64_t bytes, int, cudaStream_t st) {
  return cudaMemsetAsync(table, 0, bytes, st);
}

}  // namespace gerbil
