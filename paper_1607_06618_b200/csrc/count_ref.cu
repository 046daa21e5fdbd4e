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
//   cnt  u32   occurrences so far
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
#include "common.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
#ifndef GERBIL_REF_THREADS
#define GERBIL_REF_THREADS 512
#endif
#ifndef GERBIL_REF_CTAS
#define GERBIL_REF_CTAS 1
#endif
constexpr int kRefThreads = GERBIL_REF_THREADS;  // warps per bin = kRefThreads / 32
constexpr int kRefWarps = kRefThreads / 32;
constexpr int kRefCtasPerSm = GERBIL_REF_CTAS;   // bins in flight per SM
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

template <int W>
__global__ void __launch_bounds__(kRefThreads, kRefCtasPerSm) count_ref_kernel(SmemCountArgs a) {
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
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const bool canonical = a.canonical != 0;
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
    // one window per lane: canonical key, probe / claim / verify, then (warp-wide) the list
    auto process = [&](bool act, uint64_t q) {
      bool won = false;
      uint32_t h = 0;
      if (act) {
        uint64_t c[W];
        const bool rc = canon_at<W>(a.codes, q, a.k, canonical, c);
        const uint64_t hv = key_hash<W>(c);
        const uint64_t ref = kOcc | ((hv >> 41) << kFpShift) | ((q & kPosMask) << 1) | (rc ? 1ull : 0ull);
        h = (uint32_t)(((hv & 0xffffffffull) * cap) >> 32);
        // a bin too large for one table is counted in `parts` passes, each taking the k-mers of
        // one hash class (every occurrence of a k-mer is in the same class)
        const bool mine = a.parts <= 1 || (uint32_t)((hv >> 32) % a.parts) == a.part;
        for (; mine;) {
          uint64_t v = *(volatile uint64_t*)(s_ref + h);
          if (v == 0ull) {
            v = atomicCAS(reinterpret_cast<unsigned long long*>(s_ref + h), 0ull, (unsigned long long)ref);
            if (v == 0ull) {
              atomicAdd(s_cnt + h, 1u);
              won = true;
              break;
            }
          }
          if ((v >> kFpShift) == (ref >> kFpShift)) {  // same fingerprint: compare the k-mers
            uint64_t o[W];
            key_of_ref<W>(a.codes, v, a.k, o);
            bool eq = true;
#pragma unroll
            for (int w = 0; w < W; ++w) eq = eq && o[w] == c[w];
            if (eq) {
              atomicAdd(s_cnt + h, 1u);
              break;
            }
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
          process(act, pj + (i - ej));
        }
        uint32_t nu = 0;  // next unit: a dynamic counter per bin (units differ in length)
        if (lane == 0) nu = atomicAdd(&s_unit, 1u);
        u = __shfl_sync(kFull, nu, 0);
      }
    } else {
      // long super-mers (long reads): a unit = one piece of <= 32 consecutive windows of one
      // super-mer, numbered over the bin's descriptors (a block scan per batch of kRefThreads
      // descriptors), so the warps of the CTA end a bin within one round of each other
      for (uint64_t b0 = d0; b0 < d1; b0 += kRefThreads) {
        const uint64_t di = b0 + tid;
        uint64_t dd = 0;
        uint32_t np = 0;
        if (di < d1) {
          dd = __ldg(a.desc + di);
          np = ((uint32_t)(dd & ((1u << kNwinBits) - 1)) + 1 + 31) / 32;
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
        for (uint32_t u = warp; u < tot;) {
          if (__any_sync(kFull, *(volatile int*)&s_abandon != 0)) break;  // warp-uniform
          uint32_t t = 0;  // last descriptor with s_pfx[t] <= u
          for (uint32_t step = kRefThreads / 2; step >= 1; step >>= 1)
            if (t + step < nb && s_pfx[t + step] <= u) t += step;
          const uint64_t d = s_dsc[t];
          const uint32_t nw = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
          const uint32_t off = (u - s_pfx[t]) * 32 + lane;
          process(off < nw, (d >> kNwinBits) + off);
          uint32_t nu = 0;
          if (lane == 0) nu = atomicAdd(&s_unit, 1u);
          u = __shfl_sync(kFull, nu, 0);
        }
        __syncthreads();  // the batch's staging is reused
      }
    }
    __syncthreads();
    const uint32_t nd = s_nd;
    const bool abandoned = s_abandon != 0;
    if (!abandoned && a.min_count > 1) {  // keepers first (min_count 1 keeps every k-mer)
      uint32_t my_keep = 0;
      for (uint32_t i = tid; i < nd; i += kRefThreads) my_keep += s_cnt[s_list[i]] >= a.min_count ? 1u : 0u;
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
        n = s_cnt[s];
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

template <int W>
cudaError_t launch_ref_w(const SmemCountArgs& a, int sms, cudaStream_t st) {
  const size_t dyn = ref_table_bytes(a.cap);
  cudaError_t e = cudaFuncSetAttribute(count_ref_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  uint64_t grid = (uint64_t)sms * kRefCtasPerSm;
  if (grid > a.n_list) grid = a.n_list;
  if (grid == 0) return cudaSuccess;
  count_ref_kernel<W><<<(unsigned)grid, kRefThreads, dyn, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t ref_table_bytes(uint32_t cap) { return (size_t)cap * 14 + 16; }

uint32_t ref_table_slots(size_t smem_per_block) {
  // two CTAs share an SM: each gets half of the SM's shared memory (the opt-in per-block
  // maximum + the 1 KB the runtime reserves per block), minus that reserve and the statics
  const size_t half = (smem_per_block + 1024) / kRefCtasPerSm;
  const size_t avail = half > 1024 + 6656 ? half - 1024 - 6656 : 0;  // minus the static shared arrays (6.2 KB)
  uint32_t cap = (uint32_t)(avail / 14) & ~31u;
  if (cap > 65504) cap = 65504;  // u16 list entries
  return cap;
}

uint32_t ref_max_fill(uint32_t cap) {
  const uint32_t margin = cap / 4 > (uint32_t)kRefThreads * 2 ? cap / 4 : (uint32_t)kRefThreads * 2;
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
