// count_ref.cu — steps (d)+(e) for long k-mers (W >= 4 key words, k > 96 up to 479): one
// shared-memory hash table per bin, owned by one CTA, whose slots hold a REFERENCE to an
// occurrence of the k-mer instead of the k-mer itself.
//
// The paper counts each temporary file in its own hash table (§2.3.2;
// Alg. 1) and notes that for long k the GPU advantage vanishes (PAPER.md:314:
// a probe window holds ever fewer entries). With W-word keys a slot of the wave tables costs
// 8W+8 bytes, and k = 200 reads are mostly singletons (1 % errors: distinct ≈ 0.9 windows),
// so the tables are written almost once per window. Here a slot is 14 bytes whatever k is:
//
//   ref  u64 = 1 (occupied) | fp (23 bits of the key hash) | pos (39 bits) | rc (1 bit)
//   cnt  u32   occurrences so far - 1 (a claim publishes the reference and writes nothing else)
//   list u16   (the bin's occupied slots, in claim order)
//
// where pos is the stream position of the window that inserted the k-mer and rc says whether
// its canonical form is the reverse complement. A lane probes linearly from the
// key's hash: an empty slot is claimed with one 64-bit atomicCAS that publishes the whole
// reference; a slot with the same fingerprint is VERIFIED by re-extracting the referenced
// occurrence from the packed stream (global memory, L1/L2) and comparing all W words — so the
// count is exact, fingerprints only spare most comparisons. Counts are shared-memory atomicAdds.
// With 16 warps per CTA the whole 227 KB of shared memory is one table (~16K slots), i.e. bins
// of up to ~12K distinct k-mers; a bin that fills past max_fill is abandoned and recounted in
// the L2 wave tables (api.cu), as in count_smem.cu.
//
// Work inside a bin: warps take units of `dpc` consecutive descriptors (few for long
// super-mers, so every warp has work), lanes take consecutive windows of the unit, the window
// → super-mer map comes from one OR-reduction per round (count_smem.cu). Output: the CTA walks
// the occupied-slot list, re-extracts every kept k-mer from its reference and writes (W key
// words, u32 count) into a range reserved with one global atomic per bin (PAPER.md:467,
// reading Q5); Σcount and distinct are accumulated for the invariant.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
// Threads per CTA (the kernel's template parameter NT): one CTA of 512 per SM (one bin in flight,
// the whole shared memory its table), or two CTAs per SM (two bins in flight, half tables) of
// GERBIL_REF_T1_NT threads each — 384 (80 registers, a small L1-resident spill) beat 256 at C4
// by 20 ms: the kernel is latency-bound, more warps hide more of it.
constexpr int kRefSmThreads = 512;
#ifndef GERBIL_REF_T1_NT
#define GERBIL_REF_T1_NT 384
#endif
constexpr int kRefT1Threads = GERBIL_REF_T1_NT;
template <int NT>
constexpr int ref_ctas_per_sm() { return NT == kRefSmThreads ? 1 : 2; }
constexpr uint32_t kLongSm = 32;                 // mean windows per super-mer from which a bin is cut in pieces
constexpr uint64_t kOcc = 1ull << 63;
constexpr int kFpShift = 40;
constexpr uint64_t kPosMask = (1ull << 39) - 1;

// canonical key of the window at stream position q, and whether it is the reverse complement
template <int W>
__device__ __forceinline__ bool canon_at(const uint64_t* codes, uint64_t q, uint32_t k, bool canonical,
                                         uint64_t (&c)[W]) {
  extract_kmer<W>(codes, q, k, c);
  if (!canonical) return false;
  uint64_t r[W];
  reverse_complement<W>(c, k, r);
  if (!key_less<W>(r, c)) return false;
#pragma unroll
  for (int v = 0; v < W; ++v) c[v] = r[v];
  return true;
}

template <int W>
__device__ __forceinline__ void key_of_ref(const uint64_t* codes, uint64_t ref, uint32_t k, uint64_t (&c)[W]) {
  extract_kmer<W>(codes, (ref >> 1) & kPosMask, k, c);
  if (ref & 1ull) {
    uint64_t r[W];
    reverse_complement<W>(c, k, r);
#pragma unroll
    for (int v = 0; v < W; ++v) c[v] = r[v];
  }
}

// ---- rolling hashes for long super-mers (k >= 32) -------------------------------------------
// Extracting, reverse-complementing and hashing all W words of every window costs ~740 lane
// instructions per window at k = 200 (C4, ncu). Consecutive windows share k-1 bases, so a warp
// whose lanes take consecutive windows can instead carry two 32-bit polynomial hashes of the
// forward k-mer and of its reverse complement from window to window:
//   F(p) = sum_j c[p+j] B^(k-1-j),  R(p) = sum_j (3 - c[p+j]) B^j   (mod 2^32, B odd)
// R(p) is the same polynomial evaluated on the string rc(x), so a k-mer hashes alike on both
// strands. F(p) = B F(p-1) - B^k c[p-1] + c[p+k-1] and R(p) = B^-1 (R(p-1) - (3 - c[p-1])) +
// (3 - c[p+k-1]) B^(k-1) are affine recurrences with a constant multiplier: one warp scan per
// round of 32 windows. The canonical orientation is decided on the first 32
// bases of x and of rc(x) (a full comparison only when they tie). The hash only places a k-mer
// and gives its fingerprint; equality is still decided by comparing the k-mers (exact counts).
constexpr uint32_t kRB1 = 0x9E3779B1u, kRB2 = 0x85EBCA77u;  // odd multipliers
__host__ __device__ constexpr uint32_t inv_mod32(uint32_t b) {
  uint32_t x = b;  // Newton: each step doubles the correct low bits (b odd: b*b = 1 mod 8)
  for (int i = 0; i < 5; ++i) x *= 2u - b * x;
  return x;
}
constexpr uint32_t kRI1 = inv_mod32(kRB1), kRI2 = inv_mod32(kRB2);
static_assert(kRB1 * kRI1 == 1u && kRB2 * kRI2 == 1u, "inverse multipliers");
#ifndef GERBIL_REF_DEFER
#define GERBIL_REF_DEFER 1
#endif
#ifndef GERBIL_REF_DEFER_SHORT
#define GERBIL_REF_DEFER_SHORT 1  // the short-super-mer path defers its verifications too
#endif
#ifndef GERBIL_REF_ROLL
#define GERBIL_REF_ROLL 2
#endif
constexpr uint32_t kRollRounds = GERBIL_REF_ROLL;  // rounds of 32 windows per unit (one hash init)
constexpr uint32_t kPiece = 32 * kRollRounds;

__device__ __forceinline__ uint32_t pow32(uint32_t b, uint32_t e) {
  uint32_t r = 1u;
  for (; e; e >>= 1, b *= b)
    if (e & 1u) r *= b;
  return r;
}

// 32 bases [q, q+32) left-aligned; both words lie inside the k-mer at q when k >= 32
__device__ __forceinline__ uint64_t word_at(const uint64_t* __restrict__ codes, uint64_t q) {
  const uint64_t i = q >> 5;
  const uint32_t s = (uint32_t)(q & 31) * 2;
  const uint64_t a = __ldg(codes + i);
  return s ? ((a << s) | (__ldg(codes + i + 1) >> (64 - s))) : a;
}

// inclusive scan of v_l = sum_{j<=l} M^(l-j) e_j over the warp (M constant)
template <uint32_t M>
__device__ __forceinline__ uint32_t affine_scan(uint32_t v, uint32_t lane) {
  uint32_t m = M;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, o);
    if (lane >= (uint32_t)o) v += m * t;
    m *= m;
  }
  return v;
}

// the canonical k-mers of the occurrences (q1, rc1) and (q2, rc2) are equal
template <int W>
__device__ __noinline__ bool same_kmer(const uint64_t* codes, uint32_t k, uint64_t q1, bool rc1, uint64_t q2,
                                       bool rc2) {
  uint64_t x[W], y[W];
  extract_kmer<W>(codes, q1, k, x);
  extract_kmer<W>(codes, q2, k, y);
  if (rc1 != rc2) {  // x == rc(y)
    uint64_t r[W];
    reverse_complement<W>(y, k, r);
#pragma unroll
    for (int w = 0; w < W; ++w) y[w] = r[w];
  }
  bool eq = true;
#pragma unroll
  for (int w = 0; w < W; ++w) eq = eq && x[w] == y[w];
  return eq;
}

// F or R of the window at q computed from scratch (the rolling path's hash of one k-mer; used
// only when a deferred verification finds another k-mer under the same fingerprint)
__device__ __noinline__ uint64_t direct_roll_hash(const uint64_t* codes, uint64_t q, uint32_t k, bool rc) {
  uint32_t h1 = 0, h2 = 0;
  for (uint32_t j = 0; j < k; ++j) {
    const uint64_t p = rc ? q + k - 1 - j : q + j;  // R(q) = F of rc(x): bases from the end, complemented
    uint32_t b = (uint32_t)(__ldg(codes + (p >> 5)) >> (62 - 2 * (p & 31))) & 3u;
    if (rc) b = 3u - b;
    h1 = h1 * kRB1 + b;
    h2 = h2 * kRB2 + b;
  }
  return fmix64((uint64_t)h1 << 32 | h2);
}

// the short path's hash of the occurrence (q, rc): key_hash of its canonical k-mer (used when a
// deferred verification finds another k-mer under the same fingerprint)
template <int W>
__device__ __noinline__ uint64_t direct_key_hash(const uint64_t* codes, uint64_t q, uint32_t k, bool rc) {
  uint64_t c[W];
  extract_kmer<W>(codes, q, k, c);
  if (rc) {
    uint64_t r[W];
    reverse_complement<W>(c, k, r);
#pragma unroll
    for (int w = 0; w < W; ++w) c[w] = r[w];
  }
  return key_hash<W>(c);
}

template <int W>
__device__ __noinline__ bool rc_is_less(const uint64_t* codes, uint64_t q, uint32_t k) {
  uint64_t c[W];
  return canon_at<W>(codes, q, k, true, c);
}

template <int W, int NT>
__global__ void __launch_bounds__(NT, ref_ctas_per_sm<NT>()) count_ref_kernel(SmemCountArgs a) {
  constexpr int kRefThreads = NT;  // warps per bin = kRefThreads / 32
  constexpr int kRefWarps = kRefThreads / 32;
  extern __shared__ __align__(16) unsigned char s_raw[];
  const uint32_t cap = a.cap;
  uint64_t* s_ref = reinterpret_cast<uint64_t*>(s_raw);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_ref + cap);
  uint16_t* s_list = reinterpret_cast<uint16_t*>(s_cnt + cap);
  __shared__ uint32_t s_nd, s_unit, s_keep, s_ocur;
  __shared__ uint64_t s_dsc[kRefThreads];   // long super-mers: a batch of descriptors
  __shared__ uint32_t s_pfx[kRefThreads];   // and the first piece of each
  __shared__ uint32_t s_wsum[kRefWarps];
  __shared__ int s_abandon;
  __shared__ unsigned long long s_obase;
#if GERBIL_REF_DEFER
  // rolling path: per-warp queue of fingerprint matches awaiting verification, drained 32 at a
  // time (a verification re-extracts two k-mers; inline it would stall the whole warp for the
  // ~11 % of C4 windows that repeat a k-mer). Entry: slot << 48 | 1 << 40 | pos << 1 | rc.
  __shared__ uint64_t s_vq[kRefWarps][2 * 32];
  uint32_t vq_n = 0;  // warp-uniform
#endif
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const bool canonical = a.canonical != 0;
  // rolling-hash constants (long super-mers, k >= 32): B^(lane+1), B^-(lane+1), B^k, B^(k-1), and
  // the weights of the 8-base chunks lane and lane+32 of a window in F and R
  const bool roll = a.k >= 32;
  // diagnostics (GERBIL_REF_DBG=16): zero fingerprints, so every occupied slot a probe meets is
  // verified by comparing k-mers (exercises the verification and re-probe paths)
  const uint64_t fpm = (a.dbg & 16u) ? 0ull : ~0ull;
  const uint32_t k = a.k;
  const uint32_t pw1 = pow32(kRB1, lane + 1), pw2 = pow32(kRB2, lane + 1);
  const uint32_t pi1 = pow32(kRI1, lane + 1), pi2 = pow32(kRI2, lane + 1);
  const uint32_t bk1 = pow32(kRB1, k), bk2 = pow32(kRB2, k);
  const uint32_t bkm1 = pow32(kRB1, k - 1), bkm2 = pow32(kRB2, k - 1);
  uint32_t wf1[2], wf2[2], wr1[2], wr2[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint32_t j = lane + 32u * c, t = 8 * j < k ? (k - 8 * j < 8 ? k - 8 * j : 8u) : 0u;
    wf1[c] = t ? pow32(kRB1, k - 8 * j - t) : 0u;
    wf2[c] = t ? pow32(kRB2, k - 8 * j - t) : 0u;
    wr1[c] = t ? pow32(kRB1, 8 * j) : 0u;
    wr2[c] = t ? pow32(kRB2, 8 * j) : 0u;
  }
  for (uint32_t s = tid; s < cap; s += kRefThreads) {
    s_ref[s] = 0ull;
    s_cnt[s] = 0u;
  }
  unsigned long long acc_sum = 0, acc_dist = 0;
  for (uint32_t bi = blockIdx.x; bi < a.n_list; bi += gridDim.x) {
    const uint64_t d0 = __ldg(a.range + 2 * (size_t)bi), e1 = __ldg(a.range + 2 * (size_t)bi + 1);
    const uint64_t d1 = e1 & kRangeEndMask, win = e1 >> kRangeWinShift;
    const float avg = (float)win / (float)(d1 > d0 ? d1 - d0 : 1);
    if (tid == 0) {
      s_nd = 0;
      s_abandon = 0;
      s_unit = kRefWarps;
      s_keep = 0;
      s_ocur = 0;
    }
    __syncthreads();
    const bool roll_bin = roll && avg >= (float)kLongSm;  // this bin's windows use the rolling hashes
    // one window per lane: probe / claim / verify (eqf compares the slot's k-mer with ours),
    // then (warp-wide) the occupied-slot list
    auto probe = [&](bool act, uint64_t q, uint64_t hv, bool rc, auto&& eqf) {
      bool won = false;
      uint32_t h = 0;
      if (act) {
        const uint64_t ref = kOcc | (((hv >> 41) & fpm) << kFpShift) | ((q & kPosMask) << 1) | (rc ? 1ull : 0ull);
        h = (uint32_t)(((hv & 0xffffffffull) * cap) >> 32);
        // a bin too large for one table is counted in `parts` passes, each taking the k-mers of
        // one hash class (every occurrence of a k-mer is in the same class)
        const bool mine = a.parts <= 1 || ((uint32_t)(hv >> 32) & (a.parts - 1u)) == a.part;
        for (; mine;) {
          // claim first: the CAS returns the occupant when the slot is taken (one shared-memory
          // round trip per probe instead of a load and then a CAS)
          const uint64_t v = atomicCAS(reinterpret_cast<unsigned long long*>(s_ref + h), 0ull, (unsigned long long)ref);
          if (v == 0ull) {
            won = true;
            break;
          }
          if ((v >> kFpShift) == (ref >> kFpShift) && eqf(v)) {  // same fingerprint: compare the k-mers
            atomicAdd(s_cnt + h, 1u);
            break;
          }
          h = (h + 1 == cap) ? 0u : h + 1;
        }
      }
      const uint32_t wm = __ballot_sync(kFull, won);
      if (wm) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&s_nd, (uint32_t)__popc(wm));
        b = __shfl_sync(kFull, b, 0);
        if (won) s_list[b + __popc(wm & ((1u << lane) - 1u))] = (uint16_t)h;
        if (lane == 0 && b + __popc(wm) > a.max_fill) s_abandon = 1;
      }
    };
    // short super-mers: every window's key extracted, canonicalised and hashed whole
    auto process = [&](bool act, uint64_t q) {
      uint64_t c[W];
      bool rc = false;
      uint64_t hv = 0;
      if (act) {
        rc = canon_at<W>(a.codes, q, k, canonical, c);
        hv = key_hash<W>(c);
      }
      probe(act, q, hv, rc, [&](uint64_t v) {
        uint64_t o[W];
        key_of_ref<W>(a.codes, v, k, o);
        bool eq = true;
#pragma unroll
        for (int w = 0; w < W; ++w) eq = eq && o[w] == c[w];
        return eq;
      });
    };
#if GERBIL_REF_DEFER
    // verify the warp's queued fingerprint matches, one per lane: equal k-mers are counted in
    // their slot, a different k-mer under the same fingerprint re-probes from the next slot
    auto drain = [&]() {
      for (uint32_t i0 = 0; i0 < vq_n; i0 += 32) {
        const bool act = i0 + lane < vq_n;
        const uint64_t e = act ? s_vq[warp][i0 + lane] : 0ull;
        bool won = false;
        uint32_t h = (uint32_t)(e >> 48);
        if (act) {
          const uint64_t q = (e >> 1) & kPosMask;
          const bool rc = (e & 1ull) != 0;
          uint64_t v = *(volatile uint64_t*)(s_ref + h);
          if (same_kmer<W>(a.codes, k, q, rc, (v >> 1) & kPosMask, (v & 1ull) != 0)) {
            atomicAdd(s_cnt + h, 1u);
          } else {
            const uint64_t hv = roll_bin ? direct_roll_hash(a.codes, q, k, rc) : direct_key_hash<W>(a.codes, q, k, rc);
            const uint64_t ref = kOcc | (((hv >> 41) & fpm) << kFpShift) | (q << 1) | (rc ? 1ull : 0ull);
            for (;;) {
              h = (h + 1 == cap) ? 0u : h + 1;
              v = *(volatile uint64_t*)(s_ref + h);
              if (v == 0ull) {
                v = atomicCAS(reinterpret_cast<unsigned long long*>(s_ref + h), 0ull, (unsigned long long)ref);
                if (v == 0ull) {
                  won = true;
                  break;
                }
              }
              if ((v >> kFpShift) == (ref >> kFpShift) &&
                  same_kmer<W>(a.codes, k, q, rc, (v >> 1) & kPosMask, (v & 1ull) != 0)) {
                atomicAdd(s_cnt + h, 1u);
                break;
              }
            }
          }
        }
        const uint32_t wm = __ballot_sync(kFull, won);
        if (wm) {
          uint32_t b = 0;
          if (lane == 0) b = atomicAdd(&s_nd, (uint32_t)__popc(wm));
          b = __shfl_sync(kFull, b, 0);
          if (won) s_list[b + __popc(wm & ((1u << lane) - 1u))] = (uint16_t)h;
          if (lane == 0 && b + __popc(wm) > a.max_fill) s_abandon = 1;
        }
      }
      vq_n = 0;
      __syncwarp();
    };
    // the rolling path's probe: a fingerprint match is queued instead of verified in place
    auto probe_defer = [&](bool act, uint64_t q, uint64_t hv, bool rc) {
      bool won = false, defer = false;
      uint32_t h = 0;
      if (act) {
        const uint64_t ref = kOcc | (((hv >> 41) & fpm) << kFpShift) | ((q & kPosMask) << 1) | (rc ? 1ull : 0ull);
        h = (uint32_t)(((hv & 0xffffffffull) * cap) >> 32);
        const bool mine = a.parts <= 1 || ((uint32_t)(hv >> 32) & (a.parts - 1u)) == a.part;
        for (; mine;) {
          // claim first: the CAS returns the occupant when the slot is taken (one shared-memory
          // round trip per probe instead of a load and then a CAS)
          const uint64_t v = atomicCAS(reinterpret_cast<unsigned long long*>(s_ref + h), 0ull, (unsigned long long)ref);
          if (v == 0ull) {
            won = true;
            break;
          }
          if ((v >> kFpShift) == (ref >> kFpShift)) {
            defer = true;
            break;
          }
          h = (h + 1 == cap) ? 0u : h + 1;
        }
      }
      const uint32_t wm = __ballot_sync(kFull, won);
      if (wm) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&s_nd, (uint32_t)__popc(wm));
        b = __shfl_sync(kFull, b, 0);
        if (won) s_list[b + __popc(wm & ((1u << lane) - 1u))] = (uint16_t)h;
        if (lane == 0 && b + __popc(wm) > a.max_fill) s_abandon = 1;
      }
      const uint32_t dm = __ballot_sync(kFull, defer);
      if (defer)
        s_vq[warp][vq_n + __popc(dm & ((1u << lane) - 1u))] =
            ((uint64_t)h << 48) | (1ull << 40) | ((q & kPosMask) << 1) | (rc ? 1ull : 0ull);
      vq_n += __popc(dm);
      __syncwarp();
      if (vq_n >= 32) drain();
    };
    // short super-mers with the deferred verification: the canonical key is extracted and hashed
    // whole; a fingerprint match is queued like on the rolling path
    auto process_defer = [&](bool act, uint64_t q) {
      bool rc = false;
      uint64_t hv = 0;
      if (act) {
        uint64_t c[W];
        rc = canon_at<W>(a.codes, q, k, canonical, c);
        hv = key_hash<W>(c);
      }
      probe_defer(act, q, hv, rc);
    };
#endif
    // long super-mers (k >= 32): n <= kPiece consecutive windows from q0, lanes = consecutive
    // windows, F and R carried by the affine recurrences (one warp scan per hash per round)
    auto roll_unit = [&](uint64_t q0, uint32_t n) {
      uint32_t f1 = 0, f2 = 0, r1 = 0, r2 = 0;  // F(q0), R(q0): 8-base chunks lane, lane+32
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t j = lane + 32u * c;
        if (8 * j >= k) continue;
        const uint32_t t = k - 8 * j < 8 ? k - 8 * j : 8u;
        const uint64_t pos = q0 + 8 * j;
        const uint32_t s = (uint32_t)(pos & 31) * 2;
        uint64_t v = __ldg(a.codes + (pos >> 5)) << s;
        if (s + 2 * t > 64) v |= __ldg(a.codes + (pos >> 5) + 1) >> (64 - s);
        const uint32_t b16 = (uint32_t)(v >> 48);
        uint32_t pf1 = 0, pf2 = 0, pr1 = 0, pr2 = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if ((uint32_t)i < t) {
            const uint32_t b = (b16 >> (14 - 2 * i)) & 3u;
            pf1 = pf1 * kRB1 + b;
            pf2 = pf2 * kRB2 + b;
          }
#pragma unroll
        for (int i = 7; i >= 0; --i)
          if ((uint32_t)i < t) {
            const uint32_t b = 3u - ((b16 >> (14 - 2 * i)) & 3u);
            pr1 = pr1 * kRB1 + b;
            pr2 = pr2 * kRB2 + b;
          }
        f1 += wf1[c] * pf1;
        f2 += wf2[c] * pf2;
        r1 += wr1[c] * pr1;
        r2 += wr2[c] * pr2;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        f1 += __shfl_xor_sync(kFull, f1, o);
        f2 += __shfl_xor_sync(kFull, f2, o);
        r1 += __shfl_xor_sync(kFull, r1, o);
        r2 += __shfl_xor_sync(kFull, r2, o);
      }
      uint32_t gf1 = 0, gf2 = 0, gr1 = 0, gr2 = 0, carry = 0;  // state at the window before the round
      for (uint32_t base = 0; base < n; base += 32) {
        if (__any_sync(kFull, *(volatile int*)&s_abandon != 0)) break;  // warp-uniform
        const bool act = base + lane < n;
        const uint64_t p = q0 + base + lane;
        const uint64_t x0 = act ? word_at(a.codes, p) : 0ull;          // bases [p, p+32)
        const uint64_t y = act ? word_at(a.codes, p + k - 32) : 0ull;  // bases [p+k-32, p+k)
        const uint32_t cp = (uint32_t)(x0 >> 62), cl = (uint32_t)y & 3u;
        uint32_t cprev = __shfl_up_sync(kFull, cp, 1);
        if (lane == 0) cprev = carry;
        uint32_t e1 = cl - bk1 * cprev, e2 = cl - bk2 * cprev;
        uint32_t g1 = (3u - cl) * bkm1 - kRI1 * (3u - cprev), g2 = (3u - cl) * bkm2 - kRI2 * (3u - cprev);
        if (base == 0 && lane == 0) {
          e1 = f1;
          e2 = f2;
          g1 = r1;
          g2 = r2;
        }
        const uint32_t F1 = pw1 * gf1 + affine_scan<kRB1>(e1, lane);
        const uint32_t F2 = pw2 * gf2 + affine_scan<kRB2>(e2, lane);
        const uint32_t R1 = pi1 * gr1 + affine_scan<kRI1>(g1, lane);
        const uint32_t R2 = pi2 * gr2 + affine_scan<kRI2>(g2, lane);
        gf1 = __shfl_sync(kFull, F1, 31);
        gf2 = __shfl_sync(kFull, F2, 31);
        gr1 = __shfl_sync(kFull, R1, 31);
        gr2 = __shfl_sync(kFull, R2, 31);
        carry = __shfl_sync(kFull, cp, 31);
        bool rc = false;
        if (canonical && act) {
          const uint64_t rc0 = rev_pairs(~y);  // bases [0, 32) of rc(x)
          rc = x0 != rc0 ? rc0 < x0 : rc_is_less<W>(a.codes, p, k);
        }
        const uint64_t hv = fmix64(rc ? ((uint64_t)R1 << 32 | R2) : ((uint64_t)F1 << 32 | F2));
#if GERBIL_REF_DEFER
        probe_defer(act, p, hv, rc);
#else
        probe(act, p, hv, rc, [&](uint64_t v) {
          return same_kmer<W>(a.codes, k, p, rc, (v >> 1) & kPosMask, (v & 1ull) != 0);
        });
#endif
      }
    };
    if (avg < (float)kLongSm) {
      // short super-mers: a unit = dpc consecutive descriptors, lanes = consecutive windows
      // across them (the window → super-mer map from one OR-reduction per round)
      const float want = 24.0f / (avg > 1.0f ? avg : 1.0f);
      const uint32_t dpc = want >= 32.0f ? 32u : (want <= 1.0f ? 1u : (uint32_t)want);
      const uint64_t n_units = (d1 - d0 + dpc - 1) / dpc;
      for (uint64_t u = warp; u < n_units;) {
        const uint64_t di = d0 + u * dpc + lane;
        uint64_t pos = 0;
        uint32_t nw = 0;
        if (lane < dpc && di < d1) {
          const uint64_t d = __ldg(a.desc + di);
          pos = d >> kNwinBits;
          nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
        }
        uint32_t incl = nw;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, incl, o);
          if (lane >= (uint32_t)o) incl += t;
        }
        const uint32_t excl = incl - nw, total = __shfl_sync(kFull, incl, 31);
        uint32_t n_before = 0;
        for (uint32_t base = 0; base < total; base += 32) {
          if (__any_sync(kFull, *(volatile int*)&s_abandon != 0)) break;  // warp-uniform
          const uint32_t i = base + lane;
          const bool act = i < total;
          const uint32_t rel = excl - base;
          const uint32_t starts = __reduce_or_sync(kFull, (nw && rel < 32u) ? 1u << rel : 0u);
          int j = (int)(n_before + __popc(starts & ((2u << lane) - 1u))) - 1;
          n_before += __popc(starts);
          if (!act) j = 0;
          const uint64_t pj = __shfl_sync(kFull, pos, j);
          const uint32_t ej = __shfl_sync(kFull, excl, j);
#if GERBIL_REF_DEFER && GERBIL_REF_DEFER_SHORT
          process_defer(act, pj + (i - ej));
#else
          process(act, pj + (i - ej));
#endif
        }
        uint32_t nu = 0;  // next unit: a dynamic counter per bin (units differ in length)
        if (lane == 0) nu = atomicAdd(&s_unit, 1u);
        u = __shfl_sync(kFull, nu, 0);
      }
#if GERBIL_REF_DEFER && GERBIL_REF_DEFER_SHORT
      if (vq_n) {
        if (*(volatile int*)&s_abandon == 0) drain();  // the block-wide barrier below orders it
        vq_n = 0;
      }
#endif
    } else {
      // long super-mers (long reads): a unit = one piece of <= 32 (k < 32) or kPiece (rolling
      // hashes) consecutive windows of one super-mer, numbered over the bin's descriptors (a block
      // scan per batch of kRefThreads descriptors), so the warps of the CTA end a bin close together
      const uint32_t piece = roll ? kPiece : 32u;
      for (uint64_t b0 = d0; b0 < d1; b0 += kRefThreads) {
        const uint64_t di = b0 + tid;
        uint64_t dd = 0;
        uint32_t np = 0;
        if (di < d1) {
          dd = __ldg(a.desc + di);
          np = ((uint32_t)(dd & ((1u << kNwinBits) - 1)) + 1 + piece - 1) / piece;
        }
        uint32_t incl = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, incl, o);
          if (lane >= (uint32_t)o) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        s_dsc[tid] = dd;
        __syncthreads();
        uint32_t wex = 0, tot = 0;
        for (int q = 0; q < kRefWarps; ++q) {
          if (q < (int)warp) wex += s_wsum[q];
          tot += s_wsum[q];
        }
        s_pfx[tid] = wex + incl - np;
        if (tid == 0) s_unit = kRefWarps;
        __syncthreads();
        const uint32_t nb = d1 - b0 < (uint64_t)kRefThreads ? (uint32_t)(d1 - b0) : (uint32_t)kRefThreads;
        // unit u -> (first window, windows): the last descriptor t with s_pfx[t] <= u, found by
        // the warp in two ballots (every 16th entry, then the 16 entries of that stretch)
        auto locate = [&](uint32_t u, uint64_t& q0, uint32_t& n) {
          static_assert(kRefThreads <= 32 * 16, "two-level unit search");
          const uint32_t i1 = lane * 16;
          const uint32_t m1 = __ballot_sync(kFull, i1 < nb && s_pfx[i1] <= u);
          const uint32_t j = (31 - __clz(m1)) * 16, i2 = j + (lane & 15);
          const uint32_t m2 = __ballot_sync(kFull, lane < 16 && i2 < nb && s_pfx[i2] <= u);
          const uint32_t t = j + 31 - __clz(m2);
          const uint64_t d = s_dsc[t];
          const uint32_t nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
          const uint32_t off = (u - s_pfx[t]) * piece;
          q0 = (d >> kNwinBits) + off;
          n = nw - off < piece ? nw - off : piece;
        };
        uint32_t u = warp, n = 0;
        uint64_t q0 = 0;
        if (u < tot) locate(u, q0, n);
        while (u < tot) {
          if (__any_sync(kFull, *(volatile int*)&s_abandon != 0)) break;  // warp-uniform
          // claim the next unit now: its lookup and the first touch of its bases (a miss to
          // HBM — the packed reads are far larger than L2) overlap this unit's rounds
          uint32_t nu = 0, nn = 0;
          uint64_t nq0 = 0;
          if (lane == 0) nu = atomicAdd(&s_unit, 1u);
          nu = __shfl_sync(kFull, nu, 0);
          if (nu < tot) {
            locate(nu, nq0, nn);
            const uint64_t w0 = nq0 >> 5, w1 = (nq0 + nn + k - 2) >> 5;
            if (w0 + lane <= w1) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.codes + w0 + lane));
          }
          if (roll)
            roll_unit(q0, n);
          else
            process(lane < n, q0 + lane);
          u = nu;
          q0 = nq0;
          n = nn;
        }
#if GERBIL_REF_DEFER
        if (vq_n) {
          if (*(volatile int*)&s_abandon == 0) drain();  // the block-wide barrier below orders it
          vq_n = 0;
        }
#endif
        __syncthreads();  // the batch's staging is reused
      }
    }
    __syncthreads();
    const uint32_t nd = s_nd;
    const bool abandoned = s_abandon != 0;
    if (!abandoned && a.min_count > 1) {  // keepers first (min_count 1 keeps every k-mer)
      uint32_t my_keep = 0;
      for (uint32_t i = tid; i < nd; i += kRefThreads) my_keep += s_cnt[s_list[i]] + 1u >= a.min_count ? 1u : 0u;
      for (int o = 16; o > 0; o >>= 1) my_keep += __shfl_xor_sync(kFull, my_keep, o);
      if (lane == 0 && my_keep) atomicAdd(&s_keep, my_keep);
      __syncthreads();
    }
    if (tid == 0) {
      if (abandoned) {
        const unsigned long long e = atomicAdd(a.n_failed, 1ull);
        a.failed[2 * e] = d0;  // the bin's range entry, for the L2 recount
        a.failed[2 * e + 1] = e1;
      } else {
        const uint32_t keep = a.min_count > 1 ? s_keep : nd;
        s_obase = keep ? atomicAdd(a.out_n, (unsigned long long)keep) : 0ull;
      }
    }
    __syncthreads();
    // output (re-extract every kept k-mer from its reference) and clear the occupied slots
    for (uint32_t i0 = 0; i0 < nd; i0 += kRefThreads) {
      const uint32_t i = i0 + tid;
      uint32_t s = 0, n = 0;
      uint64_t ref = 0;
      if (i < nd) {
        s = s_list[i];
        n = s_cnt[s] + 1u;  // the count array holds occurrences - 1 (a claim writes nothing)
        ref = s_ref[s];
        s_ref[s] = 0ull;
        s_cnt[s] = 0u;
      }
      if (abandoned) continue;  // block-uniform
      acc_sum += n;
      const bool kp = i < nd && n >= a.min_count;
      const uint32_t km = __ballot_sync(kFull, kp);
      uint32_t b = 0;
      if (lane == 0 && km) b = atomicAdd(&s_ocur, (uint32_t)__popc(km));
      b = __shfl_sync(kFull, b, 0);
      if (kp) {
        const unsigned long long oi = s_obase + b + __popc(km & ((1u << lane) - 1u));
        if (oi < a.out_cap) {
          uint64_t c[W];
          key_of_ref<W>(a.codes, ref, a.k, c);
#pragma unroll
          for (int v = 0; v < W; ++v) a.out_keys[oi * W + v] = c[v];
          a.out_counts[oi] = n;
        }
      }
    }
    if (!abandoned) acc_dist += tid == 0 ? nd : 0u;
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    acc_sum += __shfl_xor_sync(kFull, acc_sum, o);
    acc_dist += __shfl_xor_sync(kFull, acc_dist, o);
  }
  if (lane == 0) {
    if (acc_sum) atomicAdd(a.sum_counts, acc_sum);
    if (acc_dist) atomicAdd(a.distinct, acc_dist);
  }
}

template <int W, int NT>
cudaError_t launch_ref_nt(const SmemCountArgs& a, int sms, cudaStream_t st) {
  const size_t dyn = ref_table_bytes(a.cap);
  SmemCountArgs b = a;
  if (const char* ev = getenv("GERBIL_REF_DBG")) b.dbg = (uint32_t)atoi(ev);
  cudaError_t e = cudaFuncSetAttribute(count_ref_kernel<W, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  uint64_t grid = (uint64_t)sms * ref_ctas_per_sm<NT>();
  if (grid > a.n_list) grid = a.n_list;
  if (grid == 0) return cudaSuccess;
  count_ref_kernel<W, NT><<<(unsigned)grid, NT, dyn, st>>>(b);
  return cudaGetLastError();
}

// a.warps = -2: two 256-thread CTAs per SM (a.cap = ref_table_slots(.., 2)); else one of 512
template <int W>
cudaError_t launch_ref_w(const SmemCountArgs& a, int sms, cudaStream_t st) {
  return a.warps == -2 ? launch_ref_nt<W, kRefT1Threads>(a, sms, st) : launch_ref_nt<W, kRefSmThreads>(a, sms, st);
}

}  // namespace

size_t ref_table_bytes(uint32_t cap) { return (size_t)cap * 14 + 16; }

uint32_t ref_table_slots(size_t smem_per_block, int ctas_per_sm) {
  // CTAs sharing an SM each get their share of its shared memory (the opt-in per-block maximum
  // + the 1 KB the runtime reserves per block), minus that reserve and the static arrays
  const int ctas = ctas_per_sm == 2 ? 2 : 1;
  const size_t nt = ctas == 2 ? (size_t)kRefT1Threads : (size_t)kRefSmThreads;
  const size_t share = (smem_per_block + 1024) / ctas;
  const size_t stat = nt * 13 + 256 + (GERBIL_REF_DEFER ? nt / 32 * 64 * 8 : 0);  // static shared arrays
  const size_t avail = share > 1024 + stat ? share - 1024 - stat : 0;
  uint32_t cap = (uint32_t)(avail / 14) & ~31u;
  if (cap > 65504) cap = 65504;  // u16 list entries
  return cap;
}

uint32_t ref_max_fill(uint32_t cap) {
  // a margin for the claims in flight (every lane of the bin's warps plus queued re-probes)
  const uint32_t margin = cap / 4 > 2u * kRefSmThreads ? cap / 4 : 2u * kRefSmThreads;
  return cap > margin ? cap - margin : 0u;
}

cudaError_t launch_count_ref(const SmemCountArgs& a, int sms, cudaStream_t st) {
  if (a.n_list == 0) return cudaSuccess;
  switch (key_words(a.k)) {
    case 1: return launch_ref_w<1>(a, sms, st);
    case 2: return launch_ref_w<2>(a, sms, st);
    case 3: return launch_ref_w<3>(a, sms, st);
    case 4: return launch_ref_w<4>(a, sms, st);
    case 5: return launch_ref_w<5>(a, sms, st);
    case 6: return launch_ref_w<6>(a, sms, st);
    case 7: return launch_ref_w<7>(a, sms, st);
    case 8: return launch_ref_w<8>(a, sms, st);
    case 9: return launch_ref_w<9>(a, sms, st);
    case 10: return launch_ref_w<10>(a, sms, st);
    case 11: return launch_ref_w<11>(a, sms, st);
    case 12: return launch_ref_w<12>(a, sms, st);
    case 13: return launch_ref_w<13>(a, sms, st);
    case 14: return launch_ref_w<14>(a, sms, st);
    case 15: return launch_ref_w<15>(a, sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace gerbil
