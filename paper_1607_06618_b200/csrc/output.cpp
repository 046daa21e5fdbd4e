// output.cpp — result encodings (App. C).
//
// Binary: "The counter of each occurring k-mer is stored in binary form,
// followed by the corresponding byte-encoded k-mer. Each four bases of a k-mer
// are encoded in one single byte. We encode A with 00, C with 01, G with 10 and
// T with 11 ... only one byte for counters less than 255. A counter greater than
// or equal to 255 is encoded in five bytes. In the latter case, all bits of the
// first byte are set to 1. The remaining four bytes contain the counter in a
// conventional 32-bit unsigned integer" — big-endian, as the worked example
// "345 TGGATC ⇒ 11111111 00000000 00000000 00000001 01011001 ..." shows; pad
// bits ("X") are written as 0.
// CSV (`-x h`): one "KMER,COUNT" line per k-mer.
//
// Both encoders split the entries into ranges, size each range, prefix-sum
// the sizes and fill the ranges on host threads.
#include "output.h"

#include <algorithm>
#include <queue>
#include <thread>
#include <vector>

namespace gerbil {
namespace {

inline uint64_t kmer_bytes(uint32_t k) { return (k + 3) / 4; }

inline uint64_t digits(uint32_t v) {
  uint64_t d = 1;
  while (v >= 10) { v /= 10; ++d; }
  return d;
}

inline uint64_t record_size(int format, uint32_t k, uint32_t count) {
  if (format == 0) return (count < 255 ? 1 : 5) + kmer_bytes(k);
  return k + 1 + digits(count) + 1;
}

inline uint8_t* put_record(int format, uint8_t* o, const uint64_t* key, uint32_t k, uint32_t count) {
  if (format == 0) {
    if (count < 255) {
      *o++ = (uint8_t)count;
    } else {
      *o++ = 0xFF;
      *o++ = (uint8_t)(count >> 24);
      *o++ = (uint8_t)(count >> 16);
      *o++ = (uint8_t)(count >> 8);
      *o++ = (uint8_t)count;
    }
    // big-endian dump of the key words, truncated to ceil(k/4) bytes (include/gerbil.h layout)
    const uint64_t nb = kmer_bytes(k);
    for (uint64_t b = 0; b < nb; ++b) *o++ = (uint8_t)(key[b / 8] >> (56 - 8 * (b % 8)));
    return o;
  }
  static const char kL[4] = {'A', 'C', 'G', 'T'};
  for (uint32_t i = 0; i < k; ++i) *o++ = (uint8_t)kL[(key[i / 32] >> (62 - 2 * (i % 32))) & 3];
  *o++ = ',';
  char buf[12];
  int n = 0;
  uint32_t v = count;
  do { buf[n++] = (char)('0' + v % 10); v /= 10; } while (v);
  while (n) *o++ = (uint8_t)buf[--n];
  *o++ = '\n';
  return o;
}

}  // namespace

uint64_t encode_results(int format, const uint64_t* keys, const uint32_t* counts, uint64_t n, uint32_t k,
                        uint32_t W, uint8_t* out, int threads) {
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  if (n < 65536) threads = 1;
  const uint64_t per = (n + threads - 1) / std::max(threads, 1);
  std::vector<uint64_t> sizes(threads + 1, 0);
  auto size_range = [&](int t) {
    uint64_t s = 0;
    for (uint64_t i = t * per; i < std::min(n, (t + 1) * per); ++i) s += record_size(format, k, counts[i]);
    sizes[t + 1] = s;
  };
  {
    std::vector<std::thread> ts;
    for (int t = 1; t < threads; ++t) ts.emplace_back(size_range, t);
    size_range(0);
    for (auto& t : ts) t.join();
  }
  for (int t = 0; t < threads; ++t) sizes[t + 1] += sizes[t];
  if (!out) return sizes[threads];
  auto fill = [&](int t) {
    uint8_t* o = out + sizes[t];
    for (uint64_t i = t * per; i < std::min(n, (t + 1) * per); ++i) o = put_record(format, o, keys + i * W, k, counts[i]);
  };
  std::vector<std::thread> ts;
  for (int t = 1; t < threads; ++t) ts.emplace_back(fill, t);
  fill(0);
  for (auto& t : ts) t.join();
  return sizes[threads];
}

// ---- k-way merge of sorted result lists (one per rank) ------------------
namespace {
inline bool key_lt(const uint64_t* a, const uint64_t* b, uint32_t W) {
  for (uint32_t i = 0; i < W; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}
inline bool key_eq(const uint64_t* a, const uint64_t* b, uint32_t W) {
  for (uint32_t i = 0; i < W; ++i)
    if (a[i] != b[i]) return false;
  return true;
}
// first index of list l whose key is not below `key`
uint64_t lower(const uint64_t* keys, uint64_t n, uint32_t W, const uint64_t* key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (key_lt(keys + mid * W, key, W)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// heap merge of the sub-ranges [b[l], e[l]) of every list; equal keys across lists are one
// entry with the summed count. out == nullptr → only the entry count.
uint64_t merge_range(uint32_t L, const uint64_t* const* keys, const uint32_t* const* counts, uint32_t W,
                     const uint64_t* b, const uint64_t* e, uint64_t* out_keys, uint32_t* out_counts) {
  struct Head {
    const uint64_t* key;
    uint32_t list;
  };
  auto gt = [W](const Head& x, const Head& y) {
    if (key_lt(y.key, x.key, W)) return true;
    if (key_lt(x.key, y.key, W)) return false;
    return x.list > y.list;
  };
  std::priority_queue<Head, std::vector<Head>, decltype(gt)> pq(gt);
  std::vector<uint64_t> pos(b, b + L);
  for (uint32_t l = 0; l < L; ++l)
    if (pos[l] < e[l]) pq.push({keys[l] + pos[l] * W, l});
  uint64_t n = 0;
  const uint64_t* last = nullptr;
  while (!pq.empty()) {
    const Head h = pq.top();
    pq.pop();
    const uint64_t i = pos[h.list]++;
    const uint32_t c = counts[h.list][i];
    if (last && key_eq(last, h.key, W)) {
      if (out_counts) out_counts[n - 1] += c;
    } else {
      if (out_keys) {
        for (uint32_t v = 0; v < W; ++v) out_keys[n * W + v] = h.key[v];
        out_counts[n] = c;
      }
      ++n;
    }
    last = h.key;
    if (pos[h.list] < e[h.list]) pq.push({keys[h.list] + pos[h.list] * W, h.list});
  }
  return n;
}
}  // namespace

uint64_t merge_sorted(uint32_t L, const uint64_t* const* keys, const uint32_t* const* counts, const uint64_t* n,
                      uint32_t W, uint64_t* out_keys, uint32_t* out_counts, int threads) {
  uint64_t total = 0;
  uint32_t big = 0;
  for (uint32_t l = 0; l < L; ++l) {
    total += n[l];
    if (n[l] > n[big]) big = l;
  }
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  if (total < (1u << 16) || L == 0) threads = 1;
  // key-space ranges: splitters at quantiles of the largest list; every list is cut at the
  // same keys, so the ranges merge independently
  std::vector<std::vector<uint64_t>> cut(threads + 1, std::vector<uint64_t>(L, 0));
  for (uint32_t l = 0; l < L; ++l) cut[threads][l] = n[l];
  for (int t = 1; t < threads; ++t) {
    const uint64_t* sk = keys[big] + (n[big] * t / threads) * W;
    for (uint32_t l = 0; l < L; ++l) cut[t][l] = lower(keys[l], n[l], W, sk);
  }
  std::vector<uint64_t> sizes(threads + 1, 0);
  auto run = [&](int t, bool write) {
    uint64_t* ok = write ? out_keys + sizes[t] * W : nullptr;
    uint32_t* oc = write ? out_counts + sizes[t] : nullptr;
    const uint64_t m = merge_range(L, keys, counts, W, cut[t].data(), cut[t + 1].data(), ok, oc);
    if (!write) sizes[t + 1] = m;
  };
  auto par = [&](bool write) {
    std::vector<std::thread> ts;
    for (int t = 1; t < threads; ++t) ts.emplace_back(run, t, write);
    run(0, write);
    for (auto& th : ts) th.join();
  };
  par(false);
  for (int t = 0; t < threads; ++t) sizes[t + 1] += sizes[t];
  if (out_keys && out_counts) par(true);
  return sizes[threads];
}

}  // namespace gerbil
