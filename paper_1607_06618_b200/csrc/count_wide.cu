// count_wide.cu — step (d) for 224 < k <= 479 (W = 8..15 key words, PAPER.md:447:
// "Supported k range from 8 to 479"): the count.cu kernels instantiated for the wide keys
// in their own translation unit (they compile in parallel with count.cu).
#include "count_kernels.cuh"

namespace gerbil {

#define GERBIL_WIDE_CASE(W, FN, ARGS)                                                                \
  case W:                                                                                    \
    return x_ ? FN<W, W + 1> ARGS : FN<W, W> ARGS

#define GERBIL_DISPATCH_WIDE(FN, ARGS)                  \
  do {                                                  \
    const uint32_t W_ = key_words(k), P_ = chunk_words(k); \
    const bool x_ = P_ != W_;                           \
    switch (W_) {                                       \
      GERBIL_WIDE_CASE(8, FN, ARGS);                              \
      GERBIL_WIDE_CASE(9, FN, ARGS);                              \
      GERBIL_WIDE_CASE(10, FN, ARGS);                             \
      GERBIL_WIDE_CASE(11, FN, ARGS);                             \
      GERBIL_WIDE_CASE(12, FN, ARGS);                             \
      GERBIL_WIDE_CASE(13, FN, ARGS);                             \
      GERBIL_WIDE_CASE(14, FN, ARGS);                             \
      GERBIL_WIDE_CASE(15, FN, ARGS);                             \
    }                                                   \
    return cudaErrorInvalidValue;                       \
  } while (0)

cudaError_t launch_count_wide(const CountArgs& a, int sms, cudaStream_t st) {
  const uint32_t k = a.k;
  GERBIL_DISPATCH_WIDE(launch_count_w, (a, sms, st));
}

cudaError_t launch_count_keys_wide(const CountKeysArgs& a, int sms, cudaStream_t st) {
  const uint32_t k = a.k;
  GERBIL_DISPATCH_WIDE(launch_count_keys_w, (a, sms, st));
}

}  // namespace gerbil
