// ordering.cuh — total orderings on m-mers as integer keys (§3.1).
//
// An m-mer is its 2m-bit value v (A=00, C=01, G=10, T=11, first base in the
// most significant digit). Every ordering is a key function: x < y in the
// ordering iff key(x) < key(y); keys are < 2^(2m+1). DESIGN.md "Orderings":
//   KMC2    (Gerbil's choice, reading Q9): A<C<G<T, m-mers
//           starting with AAA or ACA after all others → v | demoted << 2m;
//   LEX     A<C<G<T (Fig. 1) → v;
//   CGAT    lexicographic with C<G<A<T → every digit mapped
//           A→2, C→0, G→1, T→3 (bitwise: hi' = ~(hi ^ lo), lo' = hi);
//   ROBERTS C<A<T<G after complementing the bases at even positions
//           (reading Q22: counted from 1 — the 2nd, 4th, ...
//           base — so that "rare minimizers like CGCGCG are preferred":
//           CGCGCG → CCCCCC) → plain positions A→1, C→0, G→3, T→2
//           (hi' = hi, lo' = ~lo), complemented ones (hi' = ~hi, lo' = lo);
//   RANDOM  a fixed random order: a bijection of the 2m-bit
//           values, x = v·0x9E3779B1, x ^= x >> m, x = x·0x85EBCA6B,
//           x ^= x >> m (all mod 2^2m);
//   DFP     distance from pivot: key = rank[v] from a table
//           the host builds from sampled m-mer frequencies (api.cu).
#pragma once
#include "common.cuh"

namespace gerbil {

enum : uint32_t { kOrdKMC2 = 0, kOrdLEX = 1, kOrdCGAT = 2, kOrdROBERTS = 3, kOrdRANDOM = 4, kOrdDFP = 5 };

struct OrderCtx {
  uint32_t ordering, m, mask;
  uint32_t comp_digits;  // 01-pattern of the digits ROBERTS complements (2nd, 4th, ... base)
  const uint32_t* rank;  // DFP key table [4^m], else null
};

__host__ __device__ inline OrderCtx make_order(uint32_t ordering, uint32_t m, const uint32_t* rank) {
  OrderCtx o;
  o.ordering = ordering;
  o.m = m;
  o.mask = (uint32_t)((1ull << (2 * m)) - 1);
  o.comp_digits = 0;
  for (uint32_t i = 1; i < m; i += 2) o.comp_digits |= 1u << (2 * (m - 1 - i));
  o.rank = rank;
  return o;
}

// ORD = one ordering fixed at compile time (hot kernels), or kOrdRuntime
constexpr uint32_t kOrdRuntime = 0xffffffffu;

template <uint32_t ORD = kOrdRuntime>
__device__ __forceinline__ uint32_t order_key(uint32_t v, const OrderCtx& o) {
  const uint32_t lo = v & 0x55555555u, hi = (v >> 1) & 0x55555555u, dig = o.mask & 0x55555555u;
  switch (ORD == kOrdRuntime ? o.ordering : ORD) {
    case kOrdKMC2:
      if (o.m >= 3) {  // prefix AAA (000000) or ACA (000100): demoted
        const uint32_t pre = v >> (2 * o.m - 6);
        return v | ((uint32_t)((pre & ~4u) == 0u) << (2 * o.m));
      }
      return v;
    case kOrdCGAT:
      return (((~(hi ^ lo)) & dig) << 1) | hi;
    case kOrdROBERTS:
      return ((hi ^ o.comp_digits) << 1) | (lo ^ (dig & ~o.comp_digits));
    case kOrdRANDOM: {
      uint32_t x = (v * 0x9E3779B1u) & o.mask;
      x ^= x >> o.m;
      x = (x * 0x85EBCA6Bu) & o.mask;
      x ^= x >> o.m;
      return x;
    }
    case kOrdDFP:
      return __ldg(o.rank + v);
    default:
      return v;
  }
}

}  // namespace gerbil
