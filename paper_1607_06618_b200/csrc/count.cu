// count.cu — step (d): split super-mers into canonical k-mers and count them.
//
// PAPER.md:113-115 (§2.3.2 steps 2-3): "split the super-mers into k-mers" and
// "insert the k-mers into their thread-own hash tables"; Alg. 1
// with the emergency mechanism after θ trials
// (PAPER.md:255-259). Table layout and claim protocol: table.cuh.
//
// Work distribution: a warp grabs 32 super-mer
// descriptors at a time (dynamic counter), prefix-sums their window counts,
// and its lanes walk the union of windows 32·U at a time (lane ↔ U windows),
// so long and short super-mers balance the same way. For its U windows a lane
// first issues every packed-stream gather (read-only path; neighbouring lanes
// share words), then computes rc, c = min(x, rc x), the hash
// and bucket, then issues all U bucket-sector loads, and only then probes —
// U independent L2 round trips in flight per lane instead of one.
#include "count_kernels.cuh"

namespace gerbil {
namespace {

// (W, WP) pairs: W = ceil(k/32) u64 words, WP = ceil(k/31) table chunks ∈ {W, W+1}; W > 7
// (k > 224) is instantiated in count_wide.cu
#define GERBIL_DISPATCH(FN, WIDE, ARGS)                               \
  do {                                                                \
    const uint32_t W_ = key_words(k), P_ = chunk_words(k);            \
    const bool x_ = P_ != W_;                                         \
    switch (W_) {                                                     \
      case 1: return x_ ? FN<1, 2> ARGS : FN<1, 1> ARGS;              \
      case 2: return x_ ? FN<2, 3> ARGS : FN<2, 2> ARGS;              \
      case 3: return x_ ? FN<3, 4> ARGS : FN<3, 3> ARGS;              \
      case 4: return x_ ? FN<4, 5> ARGS : FN<4, 4> ARGS;              \
      case 5: return x_ ? FN<5, 6> ARGS : FN<5, 5> ARGS;              \
      case 6: return x_ ? FN<6, 7> ARGS : FN<6, 6> ARGS;              \
      case 7: return x_ ? FN<7, 8> ARGS : FN<7, 7> ARGS;              \
      default: return WIDE ARGS;                                      \
    }                                                                 \
  } while (0)

// One window per lane per step (the B200 sweep in profiles/r01_sweep.txt: more
// resident warps beat more windows per lane).
template <int W, bool TWO>
cudaError_t launch_inline(const CountArgs& a, int sms, cudaStream_t st) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_inline_kernel<W, TWO>, 128, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t dpc = a.dpc ? a.dpc : 32u;
  const uint64_t chunks = (a.d1 - a.d0 + dpc - 1) / dpc;
  uint64_t grid = (uint64_t)sms * per_sm;
  const uint64_t need = (chunks + 3) / 4;
  if (grid > need) grid = need;
  if (grid == 0) return cudaSuccess;
  count_inline_kernel<W, TWO><<<(unsigned)grid, 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <int W, bool TWO>
cudaError_t launch_keys_inline(const CountKeysArgs& a, int sms, cudaStream_t st) {
  uint64_t grid = (a.n + kThreads - 1) / kThreads;
  if (grid > (uint64_t)sms * 8) grid = (uint64_t)sms * 8;
  if (grid == 0) return cudaSuccess;
  count_keys_inline_kernel<W, TWO><<<(unsigned)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_count(const CountArgs& a, uint32_t, int sms, cudaStream_t st) {
  if (a.d1 <= a.d0) return cudaSuccess;
  const uint32_t k = a.k;
  if (table_inline(k)) {
    if (k <= 31) return launch_inline<1, false>(a, sms, st);
    if (k == 32) return launch_inline<1, true>(a, sms, st);
    return launch_inline<2, true>(a, sms, st);
  }
  GERBIL_DISPATCH(launch_count_w, launch_count_wide, (a, sms, st));
}

cudaError_t launch_count_keys(const CountKeysArgs& a, uint32_t, int sms, cudaStream_t st) {
  const uint32_t k = a.k;
  if (table_inline(k)) {
    if (k <= 31) return launch_keys_inline<1, false>(a, sms, st);
    if (k == 32) return launch_keys_inline<1, true>(a, sms, st);
    return launch_keys_inline<2, true>(a, sms, st);
  }
  GERBIL_DISPATCH(launch_count_keys_w, launch_count_keys_wide, (a, sms, st));
}

}  // namespace gerbil
