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

}  // namespace

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
