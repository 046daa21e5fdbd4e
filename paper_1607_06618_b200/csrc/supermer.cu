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
// stream; a persistent CTA takes tiles of kSTile = 1024 window start positions,
// independent of read length (100-bp and 10-kbp reads balance the same way).
//   0. rs_bits_kernel: read-start bitmap of the batch (one bit per base, laid
//      out like the N-mask), so a tile stages read boundaries like N bits;
//   1. stage the tile's packed codes, N bits and read-start bits in smem
//      (bitmaps are LSB-first u32 words: position i = bit i%32 of word i/32);
//      every thread holds at most one u64 of the NEXT tile in a register,
//      loaded while the current tile is processed;
//   2. keys: thread t rolls the m-mers of key block t (kKB = 10 consecutive
//      positions: one extraction, then 2-bit shifts of f and rc(f)); ordering
//      key c_j = min(ord f_j, ord rc f_j) (strand-symmetric minimizer,
//      DESIGN.md Q7); it publishes the block's prefix minima, suffix minima
//      and minimum;
//   3. thread t owns windows p = 8t..8t+7: μ_p = min over c[p, p+w) =
//      min(suffix[p], min of the whole key blocks in between, prefix[p+w-1]);
//      validity: no X = N | RS(q+1) bit in [p, p+k-2] and
//      base p+k-1 not N — one amortised next-set-bit scan per thread;
//   4. a super-mer starts at a valid window whose predecessor is invalid or has
//      another μ (value-based runs, Q8); the break bitmap is built
//      with 4-lane shuffles; a super-mer's length is the distance to the next
//      break (tile boundaries cut super-mers);
//   5. bin = fastrange(fmix32(μ), B); descriptors are appended with one global
//      atomic per tile; per-bin counts accumulate in smem and are flushed once
//      per persistent CTA.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "ordering.cuh"

namespace gerbil {
namespace {

constexpr int kThreads = 128;
constexpr uint32_t kSTile = 1024;  // window positions per tile (also caps super-mer length)
constexpr int kWarps = kThreads / 32;
constexpr int kPer = kSTile / kThreads;  // 8 window positions per thread
constexpr int kKeyBlocks = kThreads;
// Tile geometry for k <= KMAX (two instances: k <= 200 and k <= 479):
// KB keys per key block (one block per thread), KB * 128 >= kSTile + k - m keys per tile.
template <int KMAX>
struct Geo {
  static constexpr int kMaxK = KMAX;
  static constexpr int kKB = KMAX <= 200 ? 10 : 12;
  static constexpr int kKeyLen = kThreads * kKB;
  static constexpr int kCodeWords = (kKeyLen + 16 + 31) / 32 + 2;          // u64 words of 32 bases
  static constexpr int kBitWords = ((kSTile + kMaxK + 31) / 32 + 3) & ~1;  // u32 bitmap words (even)
  static constexpr int kBitWords64 = kBitWords / 2;
  static_assert(kKeyLen >= (int)kSTile + kMaxK - 1, "key blocks must cover every window");
  static_assert(kCodeWords + 2 * kBitWords64 <= kThreads, "one staged u64 per thread");
  static_assert(kKB + 15 - 1 <= 32, "a key block's bases (kKB + m - 1, m <= 15) sit in one u64");
};
constexpr int kMaxKSmall = 200, kMaxKAll = 479;

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

// smallest position q in [from, limit) with X(q) = N(q) | RS(q+1) set, or limit
__device__ __forceinline__ uint32_t next_x(const uint32_t* n, const uint32_t* rs, uint32_t from, uint32_t limit) {
  uint32_t w = from >> 5;
  uint32_t v = (n[w] | (rs[w] >> 1) | (rs[w + 1] << 31)) & (~0u << (from & 31));
  while (!v) {
    if (((++w) << 5) >= limit) return limit;
    v = n[w] | (rs[w] >> 1) | (rs[w + 1] << 31);
  }
  const uint32_t i = (w << 5) + __ffs(v) - 1;
  return i < limit ? i : limit;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (uint32_t)o) v += t;
  }
  return v;
}

// bit (63 - v%64) of word v/64 is set for every read start v (PAPER.md:121:
// k-mers never span two reads)
__global__ void rs_bits_kernel(const uint64_t* __restrict__ read_start, uint64_t n_reads, uint64_t* rs) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n_reads;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = read_start[r];
    if (v < read_start[r + 1]) atomicOr(reinterpret_cast<unsigned long long*>(rs + (v >> 6)), 1ull << (63 - (v & 63)));
  }
}

#ifndef GERBIL_SM_MINB
#define GERBIL_SM_MINB 8  // CTAs per SM the register budget is sized for (8: 64 regs; occupancy beats the small L1-resident spill)
#endif
// A8 (w = k-m+1 <= 193, the KMAX = 200 geometry): key blocks of 8 aligned with the thread's 8
// windows, so a window's minimum is the suffix of the thread's OWN block (registers) + whole
// blocks + the prefix of one later block (shared memory); the keys past the tile's 1024
// positions (up to 192) are computed one or two per thread (prefix minima by 8-lane shuffle scans).
#ifndef GERBIL_SM_MINB_A8
#define GERBIL_SM_MINB_A8 16  // A8: 32 registers (no spill), 16 CTAs (64 warps) per SM — more warps hide the tile barriers
#endif                        // (C1: 8 CTAs 22.4 ms, 12: 20.7 ms, 16: 19.8 ms)
template <uint32_t ORD, int KMAX, uint32_t MT, bool A8 = false>  // MT: m fixed at compile time (0 = runtime a.m)
__global__ void __launch_bounds__(kThreads, A8 ? GERBIL_SM_MINB_A8 : GERBIL_SM_MINB)
supermer_kernel(SupermerArgs a, const uint64_t* __restrict__ rs_bits, uint64_t tile_begin, uint64_t tile_end,
                int hist_smem) {
  using G = Geo<KMAX>;
  constexpr int kKB = G::kKB, kKeyLen = G::kKeyLen, kCodeWords = G::kCodeWords, kBitWords = G::kBitWords,
                kBitWords64 = G::kBitWords64;
  __shared__ uint64_t s_codes[kCodeWords];
  __shared__ uint32_t s_n[kBitWords];    // N bits
  __shared__ uint32_t s_rs[kBitWords];   // read-start bits
  __shared__ uint32_t s_key[kKeyLen];    // c_j
  __shared__ uint32_t s_pre[kKeyLen];    // min over c[8b .. j] (j in block b)
  __shared__ uint32_t s_suf[kKeyLen];    // min over c[j .. 8b+7]
  __shared__ uint32_t s_blk[kKeyBlocks + 24]; // min over block b (A8: 24 more blocks past the tile)
  __shared__ uint32_t s_brk[kSTile / 32 + 1];
  __shared__ uint32_t s_last[kThreads];  // μ of window 8t+7, or ~0 if invalid
  __shared__ uint16_t s_sp[kSTile];      // the tile's super-mer start positions
  __shared__ uint32_t s_smu[kSTile];     // and their minimizer keys
  __shared__ uint32_t s_nst;
  __shared__ uint32_t s_warp[kWarps];
  __shared__ unsigned long long s_base;
  extern __shared__ uint32_t s_hist[];   // [2 or 3][n_bins] when hist_smem

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t k = a.k, m = MT ? MT : a.m, B = a.n_bins;
  const uint32_t w = k - m + 1;
  const uint32_t n_keys = kSTile + k - m;  // m-mers needed by the tile's windows
  const uint64_t n_code_words = (a.n_bases + 31) / 32, n_mask_words = (a.n_bases + 63) / 64;
  // rs_bits has n_mask_words + 2 words (the end marker read_start[n_reads] may
  // sit past the N-mask's last word); words past either end stage as 0
  const int nh = a.bin_words ? 3 : 2;
  const uint32_t mmask = (uint32_t)((1ull << (2 * m)) - 1);
  const OrderCtx ord = make_order(a.ordering, m, a.order_rank);
  const uint64_t end_p = a.n_bases >= k ? a.n_bases - k + 1 : 0;  // windows start below this
  uint32_t* h_win = s_hist;
  uint32_t* h_cnt = s_hist + B;
  uint32_t* h_wrd = s_hist + 2 * B;
  if (hist_smem)
    for (uint32_t b = tid; b < nh * B; b += kThreads) s_hist[b] = 0;
  uint64_t my_windows = 0;
  // 1. staging: thread t owns one u64 of a tile — code word t, or N word
  //    t - kCodeWords, or read-start word t - kCodeWords - kBitWords64
  auto stage_load = [&](uint64_t tile) -> uint64_t {
    if (tile >= tile_end) return 0ull;
    const uint64_t p0 = tile * kSTile;
    if (tid < (uint32_t)kCodeWords) {
      const uint64_t i = (p0 >> 5) + tid;
      return i < n_code_words ? __ldg(a.codes + i) : 0ull;
    }
    if (tid < (uint32_t)(kCodeWords + 2 * kBitWords64)) {
      const bool is_n = tid < (uint32_t)(kCodeWords + kBitWords64);
      const uint64_t i = (p0 >> 6) + tid - kCodeWords - (is_n ? 0 : kBitWords64);
      const uint64_t* src = is_n ? a.nmask : rs_bits;
      return (src && i < n_mask_words + (is_n ? 0 : 2)) ? __ldg(src + i) : 0ull;
    }
    return 0ull;
  };
  auto stage_store = [&](uint64_t v) {  // bitmaps: u64 MSB-first → u32 LSB-first
    if (tid < (uint32_t)kCodeWords) {
      s_codes[tid] = v;
    } else if (tid < (uint32_t)(kCodeWords + kBitWords64)) {
      const uint32_t i = tid - kCodeWords;
      v = __brevll(v);
      s_n[2 * i] = (uint32_t)v;
      s_n[2 * i + 1] = (uint32_t)(v >> 32);
    } else if (tid < (uint32_t)(kCodeWords + 2 * kBitWords64)) {
      const uint32_t i = tid - kCodeWords - kBitWords64;
      v = __brevll(v);
      s_rs[2 * i] = (uint32_t)v;
      s_rs[2 * i + 1] = (uint32_t)(v >> 32);
    }
  };
  uint64_t staged = stage_load(tile_begin + blockIdx.x);

  for (uint64_t tile = tile_begin + blockIdx.x; tile < tile_end; tile += gridDim.x) {
    const uint64_t p0 = tile * kSTile;
    stage_store(staged);
    __syncthreads();
    staged = stage_load(tile + gridDim.x);  // in flight while this tile is processed
    uint32_t mu[kPer];
    if constexpr (A8) {
      // 2'. keys of the thread's own block 8t .. 8t+7 (one u64 of bases, independent extractions)
      static_assert(kPer == 8 && KMAX <= 200, "aligned blocks of 8");
      const uint32_t j0 = kPer * tid;
      uint32_t c[kPer];
      {
        const uint32_t wi = j0 >> 5, sh = (j0 & 31) * 2;
        const uint64_t v = sh ? ((s_codes[wi] << sh) | (s_codes[wi + 1] >> (64 - sh))) : s_codes[wi];
        const uint64_t R = rev_pairs(~v);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const uint32_t f = (uint32_t)(v >> (64 - 2 * (i + m))) & mmask;
          const uint32_t rc = (uint32_t)(R >> (2 * i)) & mmask;
          const uint32_t kf = order_key<ORD>(f, ord), kr = order_key<ORD>(rc, ord);
          c[i] = kf < kr ? kf : kr;
        }
        uint32_t pre = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          pre = min(pre, c[i]);
          s_pre[j0 + i] = pre;
        }
        s_blk[tid] = pre;
      }
      // the keys past the tile (positions 1024 .. 1024+w-2 <= 1215): position 1024+i by thread i,
      // 1152+i by thread i of warps 0-1; only the warps whose positions some window reaches
      // (warp-uniform conditions)
      auto extra_key = [&](uint32_t j) {
        const uint32_t wi = j >> 5, sh = (j & 31) * 2;
        const uint64_t v = sh ? ((s_codes[wi] << sh) | (s_codes[wi + 1] >> (64 - sh))) : s_codes[wi];
        const uint32_t f = (uint32_t)(v >> (64 - 2 * m)) & mmask;
        const uint32_t rc = (uint32_t)(rev_pairs(~v) & mmask);
        const uint32_t kf = order_key<ORD>(f, ord), kr = order_key<ORD>(rc, ord);
        uint32_t x = kf < kr ? kf : kr;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {  // prefix minima within blocks of 8 lanes
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o, 8);
          if ((lane & 7) >= (uint32_t)o) x = min(x, y);
        }
        s_pre[j] = x;
        if ((lane & 7) == 7) s_blk[j >> 3] = x;
      };
      if (tid < 64 || w > 65) extra_key(kSTile + tid);
      if (tid < 64 && w > 129) extra_key(kSTile + 128 + tid);
      __syncthreads();
      // 3'. minimizers of windows 8t+i = min(suffix of c from i, whole blocks, prefix at the end)
      uint32_t suf[kPer];
      suf[kPer - 1] = c[kPer - 1];
#pragma unroll
      for (int i = kPer - 2; i >= 0; --i) suf[i] = min(c[i], suf[i + 1]);
      if (w <= kPer) {  // short windows may end inside the own block
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          uint32_t x = 0xffffffffu;
#pragma unroll
          for (int j = i; j < kPer; ++j)
            if ((uint32_t)(j - i) < w) x = min(x, c[j]);
          if ((uint32_t)i + w > (uint32_t)kPer) x = min(x, s_pre[j0 + i + w - 1]);
          mu[i] = x;
        }
      } else {
        const uint32_t qa = (w - 1) >> 3, ra = (w - 1) & 7;  // window 0 ends at block t+qa, offset ra
        uint32_t midA = 0xffffffffu;
        for (uint32_t b = 1; b < qa; ++b) midA = min(midA, s_blk[tid + b]);
        const uint32_t midB = min(midA, s_blk[tid + qa]);  // windows ending in block t+qa+1
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const uint32_t mid = (uint32_t)i + ra >= (uint32_t)kPer ? midB : midA;
          mu[i] = min(min(suf[i], mid), s_pre[j0 + i + w - 1]);
        }
      }
    } else {
      // 2. rolling strand-symmetric m-mer keys of key block t (kKB keys, exactly
      //    one block per thread), block prefix/suffix minima
      {
        const uint32_t j0 = kKB * tid;
        // initial m-mer at j0
        const uint32_t wi = j0 >> 5, sh = (j0 & 31) * 2;
        const uint64_t v = sh ? ((s_codes[wi] << sh) | (s_codes[wi + 1] >> (64 - sh))) : s_codes[wi];
        // the block's bases j0 .. j0+kKB-1+m-1 (<= 26) all sit in v; R = reverse complement of v's
        // 32 bases, so the m-mer at i is bits [64-2(i+m), 64-2i) of v and its reverse complement
        // bits [2i, 2i+2m) of R — independent extractions (no rolling dependency chain)
        const uint64_t R = rev_pairs(~v);
        uint32_t c[kKB];
  #pragma unroll
        for (int i = 0; i < kKB; ++i) {
          const uint32_t f = (uint32_t)(v >> (64 - 2 * (i + m))) & mmask;
          const uint32_t rc = (uint32_t)(R >> (2 * i)) & mmask;
          const uint32_t kf = order_key<ORD>(f, ord), kr = order_key<ORD>(rc, ord);
          c[i] = kf < kr ? kf : kr;
        }
        uint32_t pre = 0xffffffffu;
  #pragma unroll
        for (int i = 0; i < kKB; ++i) {
          pre = min(pre, c[i]);
          if (w < 2 * kKB) s_key[j0 + i] = c[i];
          s_pre[j0 + i] = pre;
        }
        uint32_t suf = 0xffffffffu;
  #pragma unroll
        for (int i = kKB - 1; i >= 0; --i) {
          suf = min(suf, c[i]);
          s_suf[j0 + i] = suf;
        }
        s_blk[tid] = suf;
      }
      __syncthreads();
      // 3. minimizers and validity of windows 8t .. 8t+7
      {
        const uint32_t s0 = tid * kPer;
        if (w >= 2 * kKB) {
          // window [s, e] (e = s+w-1) = suffix of block s/kKB, the whole blocks in
          // between, prefix of block e/kKB. The 8 windows share every whole block
          // strictly between bsL = (s0+7)/kKB and beF = (s0+w-1)/kKB.
          const uint32_t bsL = (s0 + kPer - 1) / kKB, beF = (s0 + w - 1) / kKB;
          uint32_t mid = 0xffffffffu;
          for (uint32_t b = bsL + 1; b < beF; ++b) mid = min(mid, s_blk[b]);
          const uint32_t xa = s_blk[bsL], xb = s_blk[beF];
  #pragma unroll
          for (int i = 0; i < kPer; ++i) {
            const uint32_t s = s0 + i, e = s + w - 1;
            uint32_t m2 = mid;
            if (s / kKB < bsL) m2 = min(m2, xa);
            if (e / kKB > beF) m2 = min(m2, xb);
            mu[i] = min(min(s_suf[s], s_pre[e]), m2);
          }
        } else {
  #pragma unroll
          for (int i = 0; i < kPer; ++i) {
            uint32_t x = 0xffffffffu;
            for (uint32_t j = s0 + i; j < s0 + i + w; ++j) x = min(x, s_key[j]);
            mu[i] = x;
          }
        }
      }
    }
    uint32_t vmask = 0;
    {
      const uint32_t s0 = tid * kPer;
      // window s0+i is valid iff the next X position >= s0+i lies beyond s0+i+k-2
      // and base s0+i+k-1 is not N. x8 = X bits of the thread's own 8 positions
      // (s0 is 8-aligned), ns2 = next X at or after s0+8, n8 = N bits of the
      // 8 window ends.
      const uint32_t lim = s0 + k - 1 + kPer;
      const uint32_t s0w = s0 >> 5, s0b = s0 & 31;  // s0b in {0, 8, 16, 24}
      uint32_t rs8 = s_rs[s0w] >> (s0b + 1);         // RS bits s0+1 .. s0+8
      if (s0b == 24) rs8 |= s_rs[s0w + 1] << 7;
      const uint32_t x8 = ((s_n[s0w] >> s0b) | rs8) & 0xffu;
      const uint32_t ns2 = next_x(s_n, s_rs, s0 + kPer, lim);
      const uint32_t q = s0 + k - 1, qs = q & 31;
      uint32_t n8 = s_n[q >> 5] >> qs;
      if (qs > 24) n8 |= s_n[(q >> 5) + 1] << (32 - qs);
      if (k > kPer) {
        // bit masks over the 8 windows: an X among the thread's own positions at or after
        // s0+i lies closer than k-1 (< kPer <= k-2), so window i needs none (A); the next X
        // from s0+8 on must be >= s0+i+k-1 (B); base s0+i+k-1 not N (~n8); window in range (D)
        const uint32_t A = x8 ? (0xffu & ~((2u << (31 - __clz(x8))) - 1u)) : 0xffu;
        const int t = (int)ns2 - (int)(s0 + k - 1);  // windows i <= t pass B
        const uint32_t B = t >= kPer - 1 ? 0xffu : (t < 0 ? 0u : (2u << t) - 1u);
        const uint64_t base = p0 + s0;
        const uint32_t D = base >= end_p ? 0u : (end_p - base >= (uint64_t)kPer ? 0xffu
                                                                             : (1u << (uint32_t)(end_p - base)) - 1u);
        vmask = A & B & ~n8 & D & 0xffu;
      } else {
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const uint32_t xi = x8 >> i;
          const uint32_t nxt = xi ? s0 + i + __ffs(xi) - 1 : ns2;
          const bool valid = p0 + s0 + i < end_p && nxt >= s0 + i + k - 1 && !((n8 >> i) & 1u);
          vmask |= (uint32_t)valid << i;
        }
      }
      s_last[tid] = (vmask >> (kPer - 1)) & 1u ? mu[kPer - 1] : 0xffffffffu;
    }
    __syncthreads();
    // 4. starts and breaks
    uint32_t smask = 0;
    {
      uint32_t prev = tid ? s_last[tid - 1] : 0xffffffffu;  // ~0: invalid or tile start
      bool pv = prev != 0xffffffffu;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const bool v = (vmask >> i) & 1u;
        const bool st = v && (!pv || mu[i] != prev);
        smask |= (uint32_t)st << i;
        pv = v;
        prev = mu[i];
      }
      // break = !valid | start; 4 threads (32 positions) per bitmap word
      uint32_t bw = ((~vmask | smask) & 0xffu) << (8 * (tid & 3));
      bw |= __shfl_xor_sync(0xffffffffu, bw, 1);
      bw |= __shfl_xor_sync(0xffffffffu, bw, 2);
      if ((tid & 3) == 0) s_brk[tid >> 2] = bw;
      if (tid == 0) s_brk[kSTile / 32] = 1u;  // tile end
    }
    const uint32_t nst = __popc(smask);
    const uint32_t incl = warp_incl_scan(nst);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (tid < 32) {
      const uint32_t v = tid < kWarps ? s_warp[tid] : 0;
      const uint32_t t = warp_incl_scan(v);
      if (tid < kWarps) s_warp[tid] = t - v;  // exclusive
      if (tid == kWarps - 1) {
        s_base = atomicAdd(a.n_supermers, (unsigned long long)t);
        s_nst = t;
      }
    }
    __syncthreads();
    // 5. the tile's starts go to a shared list at their scan offsets, then all
    //    threads emit them together (full lanes, coalesced descriptor writes)
    {
      uint32_t o = s_warp[warp] + (incl - nst);
#pragma unroll
      for (int i = 0; i < kPer; ++i) {  // unrolled: mu stays in registers (no local-memory array)
        if ((smask >> i) & 1u) {
          s_sp[o] = (uint16_t)(tid * kPer + i);
          s_smu[o] = mu[i];
          ++o;
        }
      }
    }
    __syncthreads();
    const uint32_t n_st_tile = s_nst;
    for (uint32_t e = tid; e < n_st_tile; e += kThreads) {
      const uint32_t p = s_sp[e];
      const uint32_t nwin = next_set(s_brk, p + 1, kSTile) - p;
      const uint32_t key = s_smu[e];
      const uint32_t b = (uint32_t)(((uint64_t)fmix32(key) * B) >> 32);
      const uint64_t idx = s_base + e;
      if (idx < a.cap) {
        a.desc[idx] = ((p0 + p) << kNwinBits) | (nwin - 1);
        a.bin[idx] = b;
        if (a.mu) a.mu[idx] = key;
      }
      my_windows += nwin;
      if (hist_smem) {
        atomicAdd(&h_win[b], nwin);
        atomicAdd(&h_cnt[b], 1u);
        if (a.bin_words) atomicAdd(&h_wrd[b], (nwin + k - 1 + 31) / 32);
      } else if (a.bin_windows) {  // null: the bin shuffle derives the histogram (launch_group_shuffle)
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

cudaError_t supermer_prepare(const SupermerArgs& a, uint64_t* rs_bits, cudaStream_t st) {
  return cudaMemsetAsync(rs_bits, 0, supermer_scratch_words(a.n_bases) * 8, st);
}

cudaError_t supermer_mark_reads(const SupermerArgs& a, uint64_t* rs_bits, uint64_t r0, uint64_t r1, int sms,
                                cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  uint64_t g = (r1 - r0 + 255) / 256;
  if (g > (uint64_t)sms * 16) g = (uint64_t)sms * 16;
  rs_bits_kernel<<<(unsigned)g, 256, 0, st>>>(a.read_start + r0, r1 - r0, rs_bits);
  return cudaGetLastError();
}

cudaError_t supermer_run_tiles(const SupermerArgs& a, const uint64_t* rs_bits, uint64_t t0, uint64_t t1, int sms,
                               cudaStream_t st) {
  if (t1 <= t0) return cudaSuccess;
  const int nh = a.bin_words ? 3 : 2;
  // per-CTA smem histograms only while small: a large one would cap occupancy,
  // and spread global REDs are cheap next to this kernel's arithmetic
  const int hist_smem = a.n_bins <= 2048 && a.bin_windows != nullptr;
  const size_t dyn = hist_smem ? (size_t)nh * a.n_bins * sizeof(uint32_t) : 0;
  const bool wide = a.k > kMaxKSmall;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, dyn);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (grid > t1 - t0) grid = t1 - t0;
    kern<<<(unsigned)grid, kThreads, dyn, st>>>(a, rs_bits, t0, t1, hist_smem);
    return cudaGetLastError();
  };
#define GERBIL_SM_ORD(O) \
  case O: return wide ? go(supermer_kernel<O, kMaxKAll, 0>) : go(supermer_kernel<O, kMaxKSmall, 0>)
  // the default ordering with the common minimizer lengths: shifts and masks as constants
  static const bool a8_on = [] {
    const char* e = getenv("GERBIL_SM_A8");
    return !(e && atoi(e) == 0);
  }();
  if (a.ordering == kOrdKMC2 && !wide && a.k - a.m + 1 <= 193 && a8_on) {
    if (a.m == 15) return go(supermer_kernel<kOrdKMC2, kMaxKSmall, 15, true>);
    if (a.m == 11) return go(supermer_kernel<kOrdKMC2, kMaxKSmall, 11, true>);
    if (a.m == 7) return go(supermer_kernel<kOrdKMC2, kMaxKSmall, 7, true>);
  }
  if (a.ordering == kOrdKMC2 && !wide) {
    if (a.m == 15) return go(supermer_kernel<kOrdKMC2, kMaxKSmall, 15>);
    if (a.m == 11) return go(supermer_kernel<kOrdKMC2, kMaxKSmall, 11>);
    if (a.m == 7) return go(supermer_kernel<kOrdKMC2, kMaxKSmall, 7>);
  }
  if (a.ordering == kOrdKMC2 && wide && a.m == 15) return go(supermer_kernel<kOrdKMC2, kMaxKAll, 15>);
  switch (a.ordering) {
    GERBIL_SM_ORD(kOrdKMC2);
    GERBIL_SM_ORD(kOrdLEX);
    GERBIL_SM_ORD(kOrdCGAT);
    GERBIL_SM_ORD(kOrdROBERTS);
    GERBIL_SM_ORD(kOrdRANDOM);
    GERBIL_SM_ORD(kOrdDFP);
    default: return cudaErrorInvalidValue;
  }
#undef GERBIL_SM_ORD
}

cudaError_t launch_supermer(const SupermerArgs& a, uint64_t* rs_bits, int sms, cudaStream_t st) {
  const uint64_t n_tiles = supermer_tile_count(a.n_bases);
  if (n_tiles == 0) return cudaSuccess;
  cudaError_t e = supermer_prepare(a, rs_bits, st);
  if (e == cudaSuccess) e = supermer_mark_reads(a, rs_bits, 0, a.n_reads, sms, st);
  if (e == cudaSuccess) e = supermer_run_tiles(a, rs_bits, 0, n_tiles, sms, st);
  return e;
}

uint64_t supermer_tile_count(uint64_t n_bases) { return (n_bases + kSTile - 1) / kSTile; }

// a tile is complete once bases [0, t*kSTile + reach) are resident: its staged
// code words and bitmap words end below that (kernel step 1)
uint64_t supermer_tile_reach() { return (uint64_t)Geo<kMaxKAll>::kCodeWords * 32 + 64; }  // the larger geometry

uint64_t supermer_scratch_words(uint64_t n_bases) { return (n_bases + 63) / 64 + 2; }

}  // namespace gerbil
