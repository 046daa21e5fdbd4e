// sort.cu — device LSD radix sort of the (k-mer, count) results for gerbil_fetch(sorted) and
// the sorted encodings (sorted CSV; include/gerbil.h key layout: W left-aligned
// words, numeric order of the word array = A<C<G<T string order).
//
// Only the 2k meaningful bits are sorted, in 8-bit digits from the least significant one up
// (the last word's pad bits are zero and skipped). Each pass:
//   1. tile histograms: a CTA counts the digits of its tile of kSortTile elements;
//   2. an exclusive scan over (digit, tile) gives every (digit, tile) its output offset;
//   3. stable scatter: the CTA ranks its elements in input order — per row of 256 elements,
//      lanes of equal digit find each other with __match_any_sync, warps' per-digit counts are
//      prefix-summed in shared memory, rows accumulate — and writes the keys and counts.
// Not on the counting path (steps b-e); it runs once per sorted fetch.
#include "common.cuh"
#include "kernels.h"

#include <utility>

namespace gerbil {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kRows = 8;                         // elements per thread
constexpr int kSortTile = kSortThreads * kRows;     // 2048 elements per tile

// digit of element i: 8 bits at bit offset `bit` (from the LSB) of word `w`
__device__ __forceinline__ uint32_t digit_of(const uint64_t* keys, uint64_t i, uint32_t W, uint32_t w, uint32_t bit) {
  return (uint32_t)(__ldg(keys + i * W + w) >> bit) & 0xffu;
}

__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                                 uint32_t W, uint32_t w, uint32_t bit,
                                                                 uint32_t* __restrict__ hist, uint64_t n_tiles) {
  __shared__ uint32_t s_h[256];
  const uint64_t tile = blockIdx.x;
  s_h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t t0 = tile * kSortTile;
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const uint64_t i = t0 + (uint64_t)j * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_h[digit_of(keys, i, W, w, bit)], 1u);
  }
  __syncthreads();
  hist[(uint64_t)threadIdx.x * n_tiles + tile] = s_h[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(kSortThreads) sort_scatter_kernel(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ cnt, uint64_t n, uint32_t W, uint32_t w,
    uint32_t bit, const uint64_t* __restrict__ off, uint64_t n_tiles, uint64_t* __restrict__ keys_out,
    uint32_t* __restrict__ cnt_out) {
  __shared__ uint32_t s_wc[kSortWarps][256];  // per-warp digit counts of the current row
  __shared__ uint32_t s_base[256];            // elements of each digit in earlier rows
  const uint64_t tile = blockIdx.x;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  s_base[tid] = 0;
  for (int q = 0; q < kSortWarps; ++q) s_wc[q][tid] = 0;
  const uint64_t gbase = off[(uint64_t)tid * n_tiles + tile];  // this tile's first slot for digit tid
  __shared__ uint64_t s_gbase[256];
  s_gbase[tid] = gbase;
  __syncthreads();
  const uint64_t t0 = tile * kSortTile;
  for (int j = 0; j < kRows; ++j) {
    const uint64_t i = t0 + (uint64_t)j * kSortThreads + tid;
    const bool act = i < n;
    const uint32_t d = act ? digit_of(keys, i, W, w, bit) : 256u + lane;  // inactive lanes stay alone
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = __popc(peers & ((1u << lane) - 1u));
    if (act && before == 0) s_wc[warp][d] = __popc(peers);
    __syncthreads();
    if (act) {
      uint32_t r = s_base[d] + before;
      for (uint32_t q = 0; q < warp; ++q) r += s_wc[q][d];
      const uint64_t o = s_gbase[d] + r;
      for (uint32_t v = 0; v < W; ++v) keys_out[o * W + v] = __ldg(keys + i * W + v);
      cnt_out[o] = __ldg(cnt + i);
    }
    __syncthreads();
    uint32_t tot = 0;
    for (int q = 0; q < kSortWarps; ++q) {
      tot += s_wc[q][tid];
      s_wc[q][tid] = 0;
    }
    s_base[tid] += tot;
    __syncthreads();
  }
}

}  // namespace

uint64_t sort_scratch_words(uint64_t n) {
  const uint64_t m = 256 * ((n + kSortTile - 1) / kSortTile);
  return m / 2 + 1 + 2 * m + 1 + scan_tmp_words(m);
}

// keys/cnt sorted in place (ping-pong through keys_tmp/cnt_tmp). scratch: sort_scratch_words(n) u64.
cudaError_t launch_sort_results(uint64_t* keys, uint32_t* cnt, uint64_t n, uint32_t W, uint32_t k, uint64_t* keys_tmp,
                                uint32_t* cnt_tmp, uint64_t* scratch, int sms, cudaStream_t st) {
  if (n < 2) return cudaSuccess;
  const uint64_t n_tiles = (n + kSortTile - 1) / kSortTile;
  const uint64_t m = 256 * n_tiles;
  uint32_t* hist = reinterpret_cast<uint32_t*>(scratch);  // [m] u32, digit-major
  uint64_t* hist64 = scratch + m / 2 + 1;                  // [m]
  uint64_t* off = hist64 + m;                              // [m] exclusive scan
  uint64_t* total = off + m;                               // [1]
  uint64_t* tmp = total + 1;                               // scan_tmp_words(m)
  // digits from the least significant meaningful bit: last word first
  const uint32_t bits_last = 2 * k - 64 * (W - 1);  // meaningful bits of word W-1 (1..64)
  uint64_t *ka = keys, *kb = keys_tmp;
  uint32_t *ca = cnt, *cb = cnt_tmp;
  int passes = 0;
  for (int w = (int)W - 1; w >= 0; --w) {
    const uint32_t lo = (uint32_t)w == W - 1 ? 64 - bits_last : 0;  // lowest meaningful bit of the word
    for (uint32_t bit = lo & ~7u; bit < 64; bit += 8) {
      sort_hist_kernel<<<(unsigned)n_tiles, kSortThreads, 0, st>>>(ka, n, W, (uint32_t)w, bit, hist, n_tiles);
      cudaError_t e = launch_widen(hist, hist64, m, sms, st);
      if (e != cudaSuccess) return e;
      e = launch_scan_u64(hist64, off, m, tmp, total, st);
      if (e != cudaSuccess) return e;
      sort_scatter_kernel<<<(unsigned)n_tiles, kSortThreads, 0, st>>>(ka, ca, n, W, (uint32_t)w, bit, off, n_tiles,
                                                                      kb, cb);
      std::swap(ka, kb);
      std::swap(ca, cb);
      ++passes;
    }
  }
  if (passes & 1) {  // result in the temporaries: copy back
    cudaError_t e = cudaMemcpyAsync(keys, ka, n * W * 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(cnt, ca, n * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace gerbil
