// output.h — result encodings (App. C binary, CSV); internal.
#pragma once
#include <stdint.h>

namespace gerbil {

// Encodes n results (keys[n*W] in the include/gerbil.h layout, counts[n]);
// format 0 = App. C binary, 1 = CSV. Returns the byte count; writes only if
// out != nullptr.
uint64_t encode_results(int format, const uint64_t* keys, const uint32_t* counts, uint64_t n, uint32_t k,
                        uint32_t W, uint8_t* out, int threads);

}  // namespace gerbil
