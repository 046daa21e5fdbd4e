// supermer.cu — step (b): strand-symmetric minimizers, super-mers, bins.
//
// PAPER.md:50-53 (§2.1): "A genome sequence can be decomposed into a number
// of overlapping super-mers. Each super-mer is a substring of maximal length
// such that all k-mers on that substring share the same minimizer" and
// "It suffices to partition the set of super-mers into different temporary
// files to achieve a partitioning of all different k-mers". The paper did
// this on the CPU and names a GPU phase one as future work
// (PAPER.md:426).
//
// B200 design: the read batch is one packed base
// stream; each CTA owns a tile of kTile = 2048 window start positions,
// independent of read length (100-bp and 10-kbp reads balance the same way).
//   1. stage the tile's packed codes, N-mask and read-start bitmap in smem;
//   2. per position j: m-mer value f_j, rc(f_j), ordering key
//      c_j = min(ord f_j, ord rc f_j)  (strand-symmetric minimizer, Q7);
//   3. sliding minimum over w = k-m+1 keys by log2(w) doubling passes in smem
//      (sparse-table: min[p,p+w) = min(M_a[p], M_a[p+w-a]));
//   4. window p valid iff its k bases are N-free and inside one read
//      (PAPER.md:121-122); a super-mer is a maximal run of valid windows with
//      equal μ (value-based runs, Q8), cut at tile boundaries;
//   5. bin = fastrange(fmix32(μ), B); descriptors are appended with one
//      global atomic per tile; per-bin window / super-mer counts are
//      accumulated in smem and flushed once per persistent CTA.
#include "common.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr int kThreads = 256;
constexpr int kPer = kTile / kThreads;  // 8 window positions per thread
constexpr int kMaxK = 200;
constexpr int kCodeWords = (kTile + kMaxK + 31) / 32 + 2;
constexpr int kMaskWords = (kTile + kMaxK + 63) / 64 + 2;
constexpr int kKeyLen = kTile + kMaxK;

// MSB-first bitmaps: position i is bit (63 - i%64) of word i/64.
__device__ __forceinline__ bool bit_get(const uint64_t* bm, uint32_t i) {
  return (bm[i >> 6] >> (63 - (i & 63))) & 1ull;
}
__device__ __forceinline__ void bit_set(uint64_t* bm, uint32_t i) {
  atomicOr((unsigned long long*)&bm[i >> 6], 1ull << (63 - (i & 63)));
}
// any set bit in [lo, hi)
__device__ __forceinline__ bool bits_any(const uint64_t* bm, uint32_t lo, uint32_t hi) {
  if (lo >= hi) return false;
  const uint32_t wl = lo >> 6, wh = (hi - 1) >> 6;
  for (uint32_t w = wl; w <= wh; ++w) {
    uint64_t v = bm[w];
    if (w == wl) v &= ~0ull >> (lo & 63);
    if (w == wh) {
      const uint32_t e = ((hi - 1) & 63) + 1;
      if (e < 64) v &= ~(~0ull >> e);
    }
    if (v) return true;
  }
  return false;
}
// smallest set position in [from, limit), or limit
__device__ __forceinline__ uint32_t next_bit(const uint64_t* bm, uint32_t from, uint32_t limit) {
  for (uint32_t w = from >> 6; (w << 6) < limit; ++w) {
    uint64_t v = bm[w];
    if (w == (from >> 6)) v &= ~0ull >> (from & 63);
    if (v) {
      const uint32_t i = (w << 6) + __clzll(v);
      return i < limit ? i : limit;
    }
  }
  return limit;
}

// Ordering key of an m-mer value (right-aligned 2m bits). KMC2
// (reading Q9): A<C<G<T, m-mers starting with AAA or ACA after
// all others. LEX: plain A<C<G<T (Fig. 1).
__device__ __forceinline__ uint32_t order_key(uint32_t v, uint32_t m, uint32_t ordering) {
  if (ordering == 0 && m >= 3) {
    const uint32_t pre = v >> (2 * m - 6);
    if (pre == 0u || pre == 4u) return v | (1u << (2 * m));
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (uint32_t)o) v += t;
  }
  return v;
}

__global__ void __launch_bounds__(kThreads)
supermer_kernel(SupermerArgs a, uint64_t n_tiles, int hist_smem) {
  __shared__ uint64_t s_codes[kCodeWords];
  __shared__ uint64_t s_nm[kMaskWords];
  __shared__ uint64_t s_rs[kMaskWords];
  __shared__ uint64_t s_valid[kTile / 64];
  __shared__ uint64_t s_brk[kTile / 64];
  __shared__ uint32_t s_buf[2][kKeyLen];
  __shared__ uint32_t s_warp[kThreads / 32];
  __shared__ uint64_t s_r0;
  __shared__ unsigned long long s_base;
  extern __shared__ uint32_t s_hist[];  // [3 * n_bins] when hist_smem

  const uint32_t tid = threadIdx.x, k = a.k, m = a.m, B = a.n_bins;
  const uint32_t w = k - m + 1;
  const uint32_t n_keys = kTile + k - m;  // m-mers needed by the tile's windows
  const uint64_t n_code_words = (a.n_bases + 31) / 32, n_mask_words = (a.n_bases + 63) / 64;
  uint32_t* h_win = s_hist;
  uint32_t* h_cnt = s_hist + B;
  uint32_t* h_wrd = s_hist + 2 * B;
  if (hist_smem) {
    for (uint32_t b = tid; b < 3 * B; b += kThreads) s_hist[b] = 0;
  }
  uint64_t my_windows = 0;

  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t p0 = tile * kTile;
    // 1. stage codes, N-mask, clear bitmaps
    const uint64_t wb = p0 >> 5, mb = p0 >> 6;
    for (uint32_t i = tid; i < (uint32_t)kCodeWords; i += kThreads)
      s_codes[i] = (wb + i < n_code_words) ? __ldg(a.codes + wb + i) : 0ull;
    for (uint32_t i = tid; i < (uint32_t)kMaskWords; i += kThreads) {
      s_nm[i] = (a.nmask && mb + i < n_mask_words) ? __ldg(a.nmask + mb + i) : 0ull;
      s_rs[i] = 0ull;
    }
    for (uint32_t i = tid; i < kTile / 64; i += kThreads) {
      s_valid[i] = 0ull;
      s_brk[i] = 0ull;
    }
    if (tid == 0) {  // first read whose start lies after p0
      uint64_t lo = 0, hi = a.n_reads + 1;
      while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (a.read_start[mid] > p0) hi = mid; else lo = mid + 1;
      }
      s_r0 = lo;
    }
    __syncthreads();
    // read boundaries inside (p0, p0 + kTile + k); read_start[n_reads] marks the end
    const uint64_t lim = p0 + kTile + k;
    for (uint64_t r = s_r0 + tid; r <= a.n_reads; r += kThreads) {
      const uint64_t v = __ldg(a.read_start + r);
      if (v >= lim) break;
      bit_set(s_rs, (uint32_t)(v - p0));
    }
    // 2. ordering keys of the strand-symmetric m-mers
    const uint32_t sh_r = 64 - 2 * m;
    for (uint32_t j = tid; j < n_keys; j += kThreads) {
      const uint32_t wi = j >> 5, sh = (j & 31) * 2;
      uint64_t v = sh ? ((s_codes[wi] << sh) | (s_codes[wi + 1] >> (64 - sh))) : s_codes[wi];
      const uint32_t f = (uint32_t)(v >> sh_r);
      const uint32_t rc = (uint32_t)(rev_pairs(~v & (~0ull << sh_r)) & ((1ull << (2 * m)) - 1));
      const uint32_t kf = order_key(f, m, a.ordering), kr = order_key(rc, m, a.ordering);
      s_buf[0][j] = kf < kr ? kf : kr;
    }
    __syncthreads();
    // 3. sliding minimum by doubling: after the loop M_s[i] = min c[i, i+s)
    uint32_t len = n_keys, s = 1, cur = 0;
    while (2 * s <= w) {
      const uint32_t nl = len - s;
      const uint32_t* src = s_buf[cur];
      uint32_t* dst = s_buf[cur ^ 1];
      for (uint32_t i = tid; i < nl; i += kThreads) {
        const uint32_t x = src[i], y = src[i + s];
        dst[i] = x < y ? x : y;
      }
      __syncthreads();
      cur ^= 1;
      len = nl;
      s <<= 1;
    }
    // μ_p = min(M_s[p], M_s[p+w-s]); validity of window p
    {
      const uint32_t* src = s_buf[cur];
      uint32_t* dst = s_buf[cur ^ 1];
      for (uint32_t p = tid; p < kTile; p += kThreads) {
        const uint32_t x = src[p], y = src[p + w - s];
        dst[p] = x < y ? x : y;
        const uint64_t g = p0 + p;
        const bool valid = g < a.n_bases && !bits_any(s_nm, p, p + k) && !bits_any(s_rs, p + 1, p + k);
        if (valid) bit_set(s_valid, p);
      }
    }
    __syncthreads();
    const uint32_t* mu = s_buf[cur ^ 1];
    // 4. super-mer starts: valid and (first, or previous invalid, or μ changed)
    uint32_t starts = 0, nst = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t p = tid * kPer + i;
      const bool v = bit_get(s_valid, p);
      const bool pv = p > 0 && bit_get(s_valid, p - 1);
      const bool st = v && (!pv || mu[p] != mu[p - 1]);
      if (st) { starts |= 1u << i; ++nst; }
      if (!v || st) bit_set(s_brk, p);
    }
    const uint32_t incl = warp_incl_scan(nst);
    if (lane_id() == 31) s_warp[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
      uint32_t v = tid < kThreads / 32 ? s_warp[tid] : 0;
      uint32_t t = warp_incl_scan(v);
      if (tid < kThreads / 32) s_warp[tid] = t - v;  // exclusive
      if (tid == kThreads / 32 - 1) s_base = atomicAdd(a.n_supermers, (unsigned long long)t);
    }
    __syncthreads();
    uint64_t idx = s_base + s_warp[tid >> 5] + (incl - nst);
    // 5. emit descriptors and histogram
    while (starts) {
      const int i = __ffs(starts) - 1;
      starts &= starts - 1;
      const uint32_t p = tid * kPer + i;
      const uint32_t e = next_bit(s_brk, p + 1, kTile);
      const uint32_t nwin = e - p;
      const uint32_t key = mu[p];
      const uint32_t b = (uint32_t)(((uint64_t)fmix32(key) * B) >> 32);
      if (idx < a.cap) {
        a.desc[idx] = ((p0 + p) << kNwinBits) | (nwin - 1);
        a.bin[idx] = b;
        if (a.mu) a.mu[idx] = key;
      }
      ++idx;
      my_windows += nwin;
      const uint32_t words = (nwin + k - 1 + 31) / 32;
      if (hist_smem) {
        atomicAdd(&h_win[b], nwin);
        atomicAdd(&h_cnt[b], 1u);
        if (a.bin_words) atomicAdd(&h_wrd[b], words);
      } else {
        atomicAdd(&a.bin_windows[b], (unsigned long long)nwin);
        atomicAdd(&a.bin_supermers[b], 1ull);
        if (a.bin_words) atomicAdd(&a.bin_words[b], (unsigned long long)words);
      }
    }
    __syncthreads();
  }
  // flush per-CTA counters
  for (int o = 16; o > 0; o >>= 1) my_windows += __shfl_down_sync(0xffffffffu, my_windows, o);
  if (lane_id() == 0 && my_windows) atomicAdd(a.n_windows, (unsigned long long)my_windows);
  if (hist_smem) {
    __syncthreads();
    for (uint32_t b = tid; b < B; b += kThreads) {
      if (h_win[b]) atomicAdd(&a.bin_windows[b], (unsigned long long)h_win[b]);
      if (h_cnt[b]) atomicAdd(&a.bin_supermers[b], (unsigned long long)h_cnt[b]);
      if (a.bin_words && h_wrd[b]) atomicAdd(&a.bin_words[b], (unsigned long long)h_wrd[b]);
    }
  }
}

}  // namespace

cudaError_t launch_supermer(const SupermerArgs& a, int sms, cudaStream_t st) {
  const uint64_t n_tiles = (a.n_bases + kTile - 1) / kTile;
  if (n_tiles == 0) return cudaSuccess;
  const int hist_smem = a.n_bins <= 8192;
  const size_t dyn = hist_smem ? 3ull * a.n_bins * sizeof(uint32_t) : 0;
  cudaError_t e = cudaFuncSetAttribute(supermer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, supermer_kernel, kThreads, dyn);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sms * per_sm;
  if (grid > n_tiles) grid = n_tiles;
  supermer_kernel<<<(unsigned)grid, kThreads, dyn, st>>>(a, n_tiles, hist_smem);
  return cudaGetLastError();
}

}  // namespace gerbil
