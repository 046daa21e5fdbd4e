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
// stream; a persistent CTA takes tiles of kTile = 2048 window start positions,
// independent of read length (100-bp and 10-kbp reads balance the same way).
//   0. tile_reads_kernel: first read of every tile (one pass over read_start);
//   1. stage the tile's packed codes, N-mask and read starts in smem
//      (bitmaps are LSB-first u32 words: position i = bit i%32 of word i/32);
//   2. per position j: m-mer f_j, rc(f_j), ordering key
//      c_j = min(ord f_j, ord rc f_j) (strand-symmetric minimizer, Q7);
//   3. sliding minimum over w = k-m+1 keys by log2(w) doubling passes in smem
//      (sparse table: min[p, p+w) = min(M_a[p], M_a[p+w-a]));
//   4. window p valid iff its k bases are N-free and inside one read
//      (PAPER.md:121-122): X = N | (read-start shifted by one); valid iff
//      no X bit in [p, p+k-2] and base p+k-1 is not N — one next-set-bit scan;
//   5. positions are strided over threads (p = i*256 + tid) so the valid and
//      start bitmaps come straight out of warp ballots; a super-mer is a
//      maximal run of valid windows with equal μ (value-based runs, DESIGN.md
//      Q8), cut at tile boundaries; its length is the distance to the next
//      break bit;
//   6. bin = fastrange(fmix32(μ), B); descriptors are appended with one global
//      atomic per tile; per-bin counts accumulate in smem and are flushed once
//      per persistent CTA.
#include "common.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPer = kTile / kThreads;  // 8 window positions per thread
constexpr int kMaxK = 200;
constexpr int kCodeWords = (kTile + kMaxK + 31) / 32 + 2;  // u64 words of 32 bases
constexpr int kBitWords = ((kTile + kMaxK + 31) / 32 + 3) & ~1;  // u32 bitmap words (even)
constexpr int kKeyLen = kTile + kMaxK;

__device__ __forceinline__ bool bget(const uint32_t* bm, uint32_t i) { return (bm[i >> 5] >> (i & 31)) & 1u; }

// smallest set position in [from, limit), or limit
__device__ __forceinline__ uint32_t next_set(const uint32_t* bm, uint32_t from, uint32_t limit) {
  uint32_t w = from >> 5;
  uint32_t v = bm[w] & (~0u << (from & 31));
  while (!v) {
    if (((++w) << 5) >= limit) return limit;
    v = bm[w];
  }
  const uint32_t i = (w << 5) + __ffs(v) - 1;
  return i < limit ? i : limit;
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

__global__ void tile_reads_kernel(const uint64_t* __restrict__ read_start, uint64_t n_reads,
                                  uint64_t n_tiles, uint64_t* __restrict__ tile_first) {
  // tile t starts at p0 = t*kTile; its first read is the last r with read_start[r] <= p0
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n_reads;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = read_start[r], b = read_start[r + 1];
    if (a == b) continue;  // empty read owns no position
    for (uint64_t t = (a + kTile - 1) / kTile; t * kTile < b && t < n_tiles; ++t) tile_first[t] = r;
  }
}

__global__ void __launch_bounds__(kThreads)
supermer_kernel(SupermerArgs a, const uint64_t* __restrict__ tile_first, uint64_t n_tiles, int hist_smem) {
  __shared__ uint64_t s_codes[kCodeWords];
  __shared__ uint32_t s_n[kBitWords];    // N bits
  __shared__ uint32_t s_rs[kBitWords];   // read-start bits
  __shared__ uint32_t s_x[kBitWords];    // N(q) | RS(q+1)
  __shared__ uint32_t s_valid[kTile / 32];
  __shared__ uint32_t s_brk[kTile / 32 + 1];
  __shared__ uint32_t s_buf[2][kKeyLen];
  __shared__ uint32_t s_warp[kWarps];
  __shared__ unsigned long long s_base;
  extern __shared__ uint32_t s_hist[];  // [2 or 3][n_bins] when hist_smem

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t k = a.k, m = a.m, B = a.n_bins;
  const uint32_t w = k - m + 1;
  const uint32_t n_keys = kTile + k - m;  // m-mers needed by the tile's windows
  const uint32_t n_bits = kTile + k;      // staged base positions
  const uint64_t n_code_words = (a.n_bases + 31) / 32, n_mask_words = (a.n_bases + 63) / 64;
  const int nh = a.bin_words ? 3 : 2;
  uint32_t* h_win = s_hist;
  uint32_t* h_cnt = s_hist + B;
  uint32_t* h_wrd = s_hist + 2 * B;
  if (hist_smem)
    for (uint32_t b = tid; b < nh * B; b += kThreads) s_hist[b] = 0;
  uint64_t my_windows = 0;

  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t p0 = tile * kTile;
    // 1. stage codes and N bits (u64 MSB-first → u32 LSB-first via bit reversal)
    const uint64_t wb = p0 >> 5;
    for (uint32_t i = tid; i < (uint32_t)kCodeWords; i += kThreads)
      s_codes[i] = (wb + i < n_code_words) ? __ldg(a.codes + wb + i) : 0ull;
    const uint64_t mb = p0 >> 6;
    for (uint32_t i = tid; i < (uint32_t)(kBitWords / 2); i += kThreads) {
      uint64_t v = (a.nmask && mb + i < n_mask_words) ? __ldg(a.nmask + mb + i) : 0ull;
      v = __brevll(v);
      s_n[2 * i] = (uint32_t)v;
      s_n[2 * i + 1] = (uint32_t)(v >> 32);
      s_rs[2 * i] = 0u;
      s_rs[2 * i + 1] = 0u;
    }
    __syncthreads();
    // read boundaries inside (p0, p0 + n_bits); read_start[n_reads] marks the end
    const uint64_t lim = p0 + n_bits;
    for (uint64_t r = tile_first[tile] + 1 + tid; r <= a.n_reads; r += kThreads) {
      const uint64_t v = __ldg(a.read_start + r);
      if (v >= lim) break;
      if (v > p0) atomicOr(&s_rs[(uint32_t)(v - p0) >> 5], 1u << ((uint32_t)(v - p0) & 31));
    }
    // 2. ordering keys of the strand-symmetric m-mers
    const uint32_t sh_r = 64 - 2 * m;
    const uint64_t mmask = (1ull << (2 * m)) - 1;
    for (uint32_t j = tid; j < n_keys; j += kThreads) {
      const uint32_t wi = j >> 5, sh = (j & 31) * 2;
      const uint64_t v = sh ? ((s_codes[wi] << sh) | (s_codes[wi + 1] >> (64 - sh))) : s_codes[wi];
      const uint32_t f = (uint32_t)(v >> sh_r);
      const uint32_t rc = (uint32_t)(rev_pairs(~v & (~0ull << sh_r)) & mmask);
      const uint32_t kf = order_key(f, m, a.ordering), kr = order_key(rc, m, a.ordering);
      s_buf[0][j] = kf < kr ? kf : kr;
    }
    __syncthreads();
    // X = N | RS shifted down by one position
    for (uint32_t i = tid; i < (uint32_t)kBitWords - 1; i += kThreads)
      s_x[i] = s_n[i] | (s_rs[i] >> 1) | (s_rs[i + 1] << 31);
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
    // 4. μ_p = min(M_s[p], M_s[p+w-s]) and validity (strided positions → ballots)
    const uint32_t* src = s_buf[cur];
    uint32_t* mu = s_buf[cur ^ 1];
    const uint64_t end_p = a.n_bases >= k ? a.n_bases - k + 1 : 0;  // windows start below this
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t p = i * kThreads + tid;
      const uint32_t x = src[p], y = src[p + w - s];
      mu[p] = x < y ? x : y;
      const bool valid = p0 + p < end_p && next_set(s_x, p, p + k - 1) == p + k - 1 && !bget(s_n, p + k - 1);
      const uint32_t bal = __ballot_sync(0xffffffffu, valid);
      if (lane == 0) s_valid[(i * kThreads + warp * 32) >> 5] = bal;
    }
    __syncthreads();
    // 5. starts: valid and (tile start, or previous invalid, or μ changed); breaks = !valid | start
    uint32_t nst = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t p = i * kThreads + tid;
      const bool v = bget(s_valid, p);
      const bool st = v && (p == 0 || !bget(s_valid, p - 1) || mu[p] != mu[p - 1]);
      const uint32_t bal = __ballot_sync(0xffffffffu, !v || st);
      if (lane == 0) s_brk[(i * kThreads + warp * 32) >> 5] = bal;
      nst += st;
    }
    if (tid == 0) s_brk[kTile / 32] = 1u;  // tile end
    const uint32_t incl = warp_incl_scan(nst);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (tid < 32) {
      const uint32_t v = tid < kWarps ? s_warp[tid] : 0;
      const uint32_t t = warp_incl_scan(v);
      if (tid < kWarps) s_warp[tid] = t - v;  // exclusive
      if (tid == kWarps - 1) s_base = atomicAdd(a.n_supermers, (unsigned long long)t);
    }
    __syncthreads();
    uint64_t idx = s_base + s_warp[warp] + (incl - nst);
    // 6. emit descriptors and histogram
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t p = i * kThreads + tid;
      if (!bget(s_brk, p) || !bget(s_valid, p)) continue;  // not a start
      const uint32_t e = next_set(s_brk, p + 1, kTile);
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
      if (hist_smem) {
        atomicAdd(&h_win[b], nwin);
        atomicAdd(&h_cnt[b], 1u);
        if (a.bin_words) atomicAdd(&h_wrd[b], (nwin + k - 1 + 31) / 32);
      } else {
        atomicAdd(&a.bin_windows[b], (unsigned long long)nwin);
        atomicAdd(&a.bin_supermers[b], 1ull);
        if (a.bin_words) atomicAdd(&a.bin_words[b], (unsigned long long)((nwin + k - 1 + 31) / 32));
      }
    }
    __syncthreads();
  }
  // flush per-CTA counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_windows += __shfl_down_sync(0xffffffffu, my_windows, o);
  if (lane == 0 && my_windows) atomicAdd(a.n_windows, (unsigned long long)my_windows);
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

cudaError_t launch_supermer(const SupermerArgs& a, uint64_t* tile_first, int sms, cudaStream_t st) {
  const uint64_t n_tiles = (a.n_bases + kTile - 1) / kTile;
  if (n_tiles == 0) return cudaSuccess;
  if (a.n_reads) {
    uint64_t g = (a.n_reads + 255) / 256;
    if (g > (uint64_t)sms * 16) g = (uint64_t)sms * 16;
    tile_reads_kernel<<<(unsigned)g, 256, 0, st>>>(a.read_start, a.n_reads, n_tiles, tile_first);
  }
  const int nh = a.bin_words ? 3 : 2;
  const int hist_smem = (size_t)nh * a.n_bins * 4 <= 96 * 1024;
  const size_t dyn = hist_smem ? (size_t)nh * a.n_bins * sizeof(uint32_t) : 0;
  cudaError_t e = cudaFuncSetAttribute(supermer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, supermer_kernel, kThreads, dyn);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sms * per_sm;
  if (grid > n_tiles) grid = n_tiles;
  supermer_kernel<<<(unsigned)grid, kThreads, dyn, st>>>(a, tile_first, n_tiles, hist_smem);
  return cudaGetLastError();
}

uint64_t supermer_tiles(uint64_t n_bases) { return (n_bases + kTile - 1) / kTile; }

}  // namespace gerbil
