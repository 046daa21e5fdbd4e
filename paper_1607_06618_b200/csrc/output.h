// output.h — result encodings (App. C binary, CSV); internal.
#pragma once
#include <stdint.h>

namespace gerbil {

// Encodes n results (keys[n*W] in the include/gerbil.h layout, counts[n]);
// format 0 = App. C binary, 1 = CSV. Returns the byte count; writes only if
// out != nullptr.
uint64_t encode_results(int format, const uint64_t* keys, const uint32_t* counts, uint64_t n, uint32_t k,
                        uint32_t W, uint8_t* out, int threads);

// k-way merge of L sorted result lists (keys[l][n[l]*W], counts[l][n[l]]) into one sorted list;
// equal keys across lists become one entry with the summed count. Returns the entry count;
// writes only if out_keys and out_counts are non-null (two-call pattern).
uint64_t merge_sorted(uint32_t L, const uint64_t* const* keys, const uint32_t* const* counts, const uint64_t* n,
                      uint32_t W, uint64_t* out_keys, uint32_t* out_counts, int threads);

}  // namespace gerbil
