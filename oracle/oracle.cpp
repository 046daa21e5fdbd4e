/*
 * oracle.cpp — the CPU ORACLE for the Gerbil counting phase.
 *
 *   *** TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and
 *   *** bench.py's cpu_baseline / --impl reference leg may load this library.
 *   *** The product path (paper_1607_06618_b200/) never imports, links or
 *   *** executes anything under oracle/.
 *
 * A plain, slow, obviously correct implementation of what the path computes,
 * written from PAPER.md and sharing no code with the CUDA path (its own
 * parser, its own reverse complement, its own ordering, std::string keys in a
 * std::map). Every function cites the passage it follows.
 *
 *  - oracle_count: the k-mer histogram (Abstract: "build a
 *    histogram of all substrings of length k"), canonical = lexicographically
 *    smaller of x and rc(x) (§2.4.2), ignoring k-mers with
 *    an undetermined base (§2.4.1), output iff
 *    count >= min_count (`-l`). Pinned by tests/test_oracle.py
 *    (brute force, `sort | uniq -c`, de Bruijn closed forms, planted
 *    multiplicities, Σ-count identity, rc invariance).
 *  - oracle_minimizer / oracle_supermers: minimizer = smallest m-substring
 *    under a total order (§2.1); super-mers = maximal substrings
 *    whose k-mers share one minimizer (Fig. 1);
 *    orderings LEX (A<C<G<T, Fig. 1) and KMC2 (A<C<G<T with the AAA/ACA
 *    prefixes demoted; reading Q9 in DESIGN.md), and the other
 *    orderings the paper evaluates: CGAT, Roberts, Random,
 *    dfp(p) with its sampled frequency table (oracle_dfp_table). Pinned by the
 *    Fig. 1 example, SPEC.md:81-82 minimizer examples, hand-ranked alphabet
 *    examples, bijectivity and the planted-frequency dfp fixture.
 *  - oracle_minimizer_stats: the Fig. Minimizer metric (max distinct k-mers
 *    per minimizer), by brute force over the histogram.
 *  - oracle_count_sampled: the same histogram restricted to canonical k-mers
 *    whose FNV-1a-64 hash of the ASCII string is ≡ 0 (mod `mod`) — the
 *    full-scale parity check of SURVEY.md §8(c) "Scale strategy". Pinned by
 *    equality with oracle_count filtered by the same predicate.
 *
 * Input parsing (reading Q3/Q4 in DESIGN.md): FASTA ('>' header, multi-line
 * sequence concatenated), FASTQ ('@' header, sequence, '+' [header],
 * quality of equal length), or raw (one read per line) when the first
 * non-empty byte is neither '>' nor '@'. CR bytes are dropped, empty lines
 * skipped; lowercase is folded; every other byte outside ACGT breaks the read.
 */
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <thread>
#include <vector>

namespace {

struct Result {
  std::vector<std::string> kmers;
  std::vector<uint64_t> counts;
  uint64_t windows = 0;   /* valid windows seen (Σ counts before threshold) */
  uint64_t distinct = 0;  /* distinct canonical k-mers before threshold */
  std::string error;
};

/* ---- parsing (App. B; Q3/Q4) ------------------- */

/* Splits text into lines without CR; returns false + message on malformed. */
static void split_lines(const char* text, size_t len, std::vector<std::string>& lines) {
  size_t i = 0;
  while (i < len) {
    size_t j = i;
    while (j < len && text[j] != '\n') ++j;
    std::string line(text + i, j - i);
    line.erase(std::remove(line.begin(), line.end(), '\r'), line.end());
    lines.push_back(line);
    i = j + 1;
  }
}

static bool parse_reads(const char* text, size_t len, std::vector<std::string>& reads,
                        std::string& err) {
  std::vector<std::string> lines;
  split_lines(text, len, lines);
  size_t first = 0;
  while (first < lines.size() && lines[first].empty()) ++first;
  if (first == lines.size()) return true; /* empty input: no reads */
  char kind = lines[first][0];
  if (kind == '>') {
    std::string cur;
    bool have = false;
    for (size_t i = first; i < lines.size(); ++i) {
      const std::string& l = lines[i];
      if (l.empty()) continue;
      if (l[0] == '>') {
        if (have) reads.push_back(cur);
        cur.clear();
        have = true;
      } else {
        cur += l;
      }
    }
    if (have) reads.push_back(cur);
    return true;
  }
  if (kind == '@') {
    size_t i = first;
    while (i < lines.size()) {
      if (lines[i].empty()) { ++i; continue; }
      if (lines[i][0] != '@') {
        err = "FASTQ: expected '@' at line " + std::to_string(i + 1);
        return false;
      }
      if (i + 3 >= lines.size()) {
        err = "FASTQ: truncated record at line " + std::to_string(i + 1);
        return false;
      }
      const std::string& seq = lines[i + 1];
      const std::string& plus = lines[i + 2];
      const std::string& qual = lines[i + 3];
      if (plus.empty() || plus[0] != '+') {
        err = "FASTQ: expected '+' at line " + std::to_string(i + 3);
        return false;
      }
      if (qual.size() != seq.size()) {
        err = "FASTQ: quality length mismatch at line " + std::to_string(i + 4);
        return false;
      }
      reads.push_back(seq);
      i += 4;
    }
    return true;
  }
  for (size_t i = first; i < lines.size(); ++i)
    if (!lines[i].empty()) reads.push_back(lines[i]);
  return true;
}

/* Case-fold, then break at every byte outside {A,C,G,T}. */
static void fragments_of(const std::string& read, std::vector<std::string>& out) {
  std::string cur;
  for (char ch : read) {
    char u = (ch >= 'a' && ch <= 'z') ? (char)(ch - 'a' + 'A') : ch;
    if (u == 'A' || u == 'C' || u == 'G' || u == 'T') {
      cur.push_back(u);
    } else {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    }
  }
  if (!cur.empty()) out.push_back(cur);
}

/* ---- k-mer definitions (§2.4.2) ----------------------- */

static char complement(char c) {
  switch (c) {
    case 'A': return 'T';
    case 'T': return 'A';
    case 'C': return 'G';
    case 'G': return 'C';
  }
  return c;
}

/* "reversing x and replacing A⇔T and C⇔G" */
static std::string reverse_complement(const std::string& x) {
  std::string r(x.rbegin(), x.rend());
  for (char& c : r) c = complement(c);
  return r;
}

/* "the lexicographically smaller k-mer as canonical representation";
 * ASCII 'A'<'C'<'G'<'T' is the paper's A<C<G<T order (reading Q1). */
static std::string canonical(const std::string& x) {
  std::string r = reverse_complement(x);
  return r < x ? r : x;
}

static uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (char c : s) {
    h ^= (unsigned char)c;
    h *= 1099511628211ull;
  }
  return h;
}

/* Count every window of every fragment into the map. */
static void count_reads(const std::vector<std::string>& reads, size_t r0, size_t r1,
                        uint32_t k, int canon, uint64_t mod,
                        std::map<std::string, uint64_t>& hist, uint64_t& windows) {
  std::vector<std::string> frags;
  for (size_t r = r0; r < r1; ++r) {
    frags.clear();
    fragments_of(reads[r], frags);
    for (const std::string& f : frags) {
      if (f.size() < k) continue;
      for (size_t i = 0; i + k <= f.size(); ++i) {
        std::string w = f.substr(i, k);
        std::string c = canon ? canonical(w) : w;
        ++windows;
        if (mod > 1 && fnv1a(c) % mod != 0) continue;
        ++hist[c];
      }
    }
  }
}

static Result* finish(std::map<std::string, uint64_t>& hist, uint64_t windows,
                      uint32_t min_count) {
  Result* res = new Result();
  res->windows = windows;
  res->distinct = hist.size();
  for (auto& kv : hist)
    if (kv.second >= min_count) {
      res->kmers.push_back(kv.first);
      res->counts.push_back(kv.second);
    }
  return res;
}

/* ---- minimizers and super-mers (§2.1; §3.1) ------------- */

/* ---- orderings (§3.1) -------- */

/* base-4 number of an m-mer string over a given letter ranking */
static uint32_t number_in(const std::string& s, const char* alphabet) {
  uint32_t v = 0;
  for (char c : s) v = v * 4 + (uint32_t)(strchr(alphabet, c) - alphabet);
  return v;
}

/* Ordering key of an m-mer (readings Q9, Q22, Q23 in DESIGN.md):
 *  0 KMC2    A<C<G<T, m-mers starting with AAA or ACA after all others;
 *  1 LEX     A<C<G<T (Fig. 1);
 *  2 CGAT    lexicographic with C<G<A<T;
 *  3 ROBERTS bases at even positions — counted from 1, i.e. the 2nd, 4th, ...
 *            base, the reading under which "rare minimizers like CGCGCG are
 *            preferred" holds (CGCGCG → CCCCCC) — replaced by their
 *            complement, then lexicographic with C<A<T<G;
 *  4 RANDOM  a fixed bijection of the A<C<G<T number v of the m-mer:
 *            x = v*0x9E3779B1, x ^= x >> m, x = x*0x85EBCA6B, x ^= x >> m,
 *            every product taken mod 4^m;
 *  5 DFP     table[v] (oracle_dfp_table). */
static uint32_t order_key_of(const std::string& mm, int ordering, const uint32_t* table) {
  const uint32_t m = (uint32_t)mm.size();
  const uint32_t lex = number_in(mm, "ACGT");
  switch (ordering) {
    case 0: {
      const bool demoted = m >= 3 && (mm.compare(0, 3, "AAA") == 0 || mm.compare(0, 3, "ACA") == 0);
      return lex + (demoted ? (uint32_t)(1ull << (2 * m)) : 0u);
    }
    case 2:
      return number_in(mm, "CGAT");
    case 3: {
      std::string t = mm;
      for (size_t i = 1; i < t.size(); i += 2) t[i] = complement(t[i]);
      return number_in(t, "CATG");
    }
    case 4: {
      const uint64_t mod = 1ull << (2 * m);
      uint64_t x = ((uint64_t)lex * 0x9E3779B1ull) % mod;
      x ^= x >> m;
      x = (x * 0x85EBCA6Bull) % mod;
      x ^= x >> m;
      return (uint32_t)x;
    }
    case 5:
      return table[lex];
    default:
      return lex;
  }
}

/* Ordering "less than" on two m-mers. LEX: A<C<G<T. KMC2: the same, except
 * that m-mers starting with AAA or ACA come after all others,
 * lexicographic inside each group (reading Q9). Others: by order_key_of. */
static bool order_less(const std::string& a, const std::string& b, int ordering,
                       const uint32_t* table = nullptr) {
  if (ordering >= 2) return order_key_of(a, ordering, table) < order_key_of(b, ordering, table);
  if (ordering == 0 && a.size() >= 3) {
    bool da = a.compare(0, 3, "AAA") == 0 || a.compare(0, 3, "ACA") == 0;
    bool db = b.compare(0, 3, "AAA") == 0 || b.compare(0, 3, "ACA") == 0;
    if (da != db) return db; /* non-demoted < demoted */
  }
  return a < b;
}

/* "a minimizer of a k-mer is defined as its lexicographically smallest
 * substring of a fixed length m < k with respect to some total ordering"
 * (PAPER.md:51). symmetric = minimum over the m-mers of x and of rc(x)
 * (reading Q7: required for canonical bins). */
static std::string minimizer_of(const std::string& x, uint32_t m, int ordering,
                                int symmetric, const uint32_t* table = nullptr) {
  std::string best;
  bool have = false;
  std::string rx = reverse_complement(x);
  for (size_t j = 0; j + m <= x.size(); ++j) {
    std::string f = x.substr(j, m);
    if (!have || order_less(f, best, ordering, table)) { best = f; have = true; }
    if (symmetric) {
      std::string g = rx.substr(j, m);
      if (order_less(g, best, ordering, table)) best = g;
    }
  }
  return best;
}

}  // namespace

extern "C" {

typedef struct oracle_result oracle_result;

/* Full histogram of a FASTA/FASTQ/raw document. Returns NULL on parse error
 * (message copied into err). canon=0 counts k-mers as they occur (-d,
 * PAPER.md:483). */
oracle_result* oracle_count(const char* text, uint64_t len, uint32_t k,
                            uint32_t min_count, int canon, char* err, uint64_t err_len) {
  std::vector<std::string> reads;
  std::string e;
  if (!parse_reads(text, len, reads, e)) {
    if (err && err_len) { strncpy(err, e.c_str(), err_len - 1); err[err_len - 1] = 0; }
    return nullptr;
  }
  std::map<std::string, uint64_t> hist;
  uint64_t windows = 0;
  count_reads(reads, 0, reads.size(), k, canon, 1, hist, windows);
  return (oracle_result*)finish(hist, windows, min_count);
}

/* Hash-sampled histogram on `threads` host threads: only canonical k-mers
 * with fnv1a(string) % mod == 0 are kept; windows counts all valid windows. */
oracle_result* oracle_count_sampled(const char* text, uint64_t len, uint32_t k,
                                    uint32_t min_count, uint64_t mod, int threads,
                                    char* err, uint64_t err_len) {
  std::vector<std::string> reads;
  std::string e;
  if (!parse_reads(text, len, reads, e)) {
    if (err && err_len) { strncpy(err, e.c_str(), err_len - 1); err[err_len - 1] = 0; }
    return nullptr;
  }
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::map<std::string, uint64_t>> parts(threads);
  std::vector<uint64_t> wins(threads, 0);
  std::vector<std::thread> ts;
  size_t per = (reads.size() + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    size_t a = std::min(reads.size(), t * per), b = std::min(reads.size(), a + per);
    ts.emplace_back([&, t, a, b] { count_reads(reads, a, b, k, 1, mod, parts[t], wins[t]); });
  }
  for (auto& t : ts) t.join();
  std::map<std::string, uint64_t> hist;
  uint64_t windows = 0;
  for (int t = 0; t < threads; ++t) {
    windows += wins[t];
    for (auto& kv : parts[t]) hist[kv.first] += kv.second;
  }
  return (oracle_result*)finish(hist, windows, min_count);
}

uint64_t oracle_result_n(const oracle_result* r) { return ((const Result*)r)->kmers.size(); }
uint64_t oracle_result_windows(const oracle_result* r) { return ((const Result*)r)->windows; }
uint64_t oracle_result_distinct(const oracle_result* r) { return ((const Result*)r)->distinct; }

/* kmers: n*k bytes (no separators), counts: n entries, in A<C<G<T order. */
void oracle_result_get(const oracle_result* r, char* kmers, uint64_t* counts) {
  const Result* res = (const Result*)r;
  for (size_t i = 0; i < res->kmers.size(); ++i) {
    if (kmers) memcpy(kmers + i * res->kmers[i].size(), res->kmers[i].data(), res->kmers[i].size());
    if (counts) counts[i] = res->counts[i];
  }
}

void oracle_result_free(oracle_result* r) { delete (Result*)r; }

/* fnv1a(kmer) % mod == 0 — the sampling predicate, exposed for harnesses. */
int oracle_sample_keep(const char* kmer, uint32_t k, uint64_t mod) {
  return fnv1a(std::string(kmer, k)) % mod == 0;
}

void oracle_reverse_complement(const char* x, uint32_t n, char* out) {
  std::string r = reverse_complement(std::string(x, n));
  memcpy(out, r.data(), n);
}

void oracle_canonical(const char* x, uint32_t n, char* out) {
  std::string c = canonical(std::string(x, n));
  memcpy(out, c.data(), n);
}

/* One output record, App. C: "The counter of each occuring
 * k-mer is stored in binary form, followed by the corresponding byte-encoded
 * k-mer. Each four bases of a k-mer are encoded in one single byte. We encode A
 * with 00, C with 01, G with 10 and T with 11 ... only one byte for counters
 * less than 255. A counter greater than or equal to 255 is encoded in five
 * bytes. In the latter case, all bits of the first byte are set to 1. The
 * remaining four bytes contain the counter in a conventional 32-bit unsigned
 * integer." Byte order of the counter and bit order of the bases follow the
 * worked examples; the undefined pad bits X are written 0
 * (SPEC.md:54). Returns the record length; writes it to out if non-NULL. */
uint64_t oracle_encode_entry(const char* kmer, uint32_t k, uint64_t count, uint8_t* out) {
  std::vector<uint8_t> rec;
  if (count < 255) {
    rec.push_back((uint8_t)count);
  } else {
    rec.push_back(0xFF);
    for (int shift = 24; shift >= 0; shift -= 8) rec.push_back((uint8_t)((count >> shift) & 0xFF));
  }
  for (uint32_t i = 0; i < k; i += 4) {
    uint8_t byte = 0;
    for (uint32_t j = 0; j < 4; ++j) {
      uint8_t code = 0; /* pad bases beyond k: 00 */
      if (i + j < k) {
        switch (kmer[i + j]) {
          case 'A': code = 0; break;
          case 'C': code = 1; break;
          case 'G': code = 2; break;
          case 'T': code = 3; break;
        }
      }
      byte = (uint8_t)((byte << 2) | code);
    }
    rec.push_back(byte);
  }
  if (out) memcpy(out, rec.data(), rec.size());
  return rec.size();
}

/* Minimizer m-mer of one k-mer (ordering: see order_key_of; table = the DFP
 * key table for ordering 5, else NULL). */
void oracle_minimizer(const char* kmer, uint32_t k, uint32_t m, int ordering,
                      int symmetric, char* out) {
  std::string mm = minimizer_of(std::string(kmer, k), m, ordering, symmetric);
  memcpy(out, mm.data(), m);
}

void oracle_minimizer_t(const char* kmer, uint32_t k, uint32_t m, int ordering, int symmetric,
                        const uint32_t* table, char* out) {
  std::string mm = minimizer_of(std::string(kmer, k), m, ordering, symmetric, table);
  memcpy(out, mm.data(), m);
}

/* Ordering key of one m-mer (order_key_of). */
uint32_t oracle_order_key(const char* mmer, uint32_t m, int ordering, const uint32_t* table) {
  return order_key_of(std::string(mmer, m), ordering, table);
}

/* dfp(p) key table ("we initially sort the set of minimizers by
 * their frequency ... approximate them by taking samples during runtime ...
 * re-sort the minimizers by the absolute difference of their initial position
 * to the pivot position 4^m p"), reading Q23 in DESIGN.md:
 *  sample   = every m-mer occurrence that starts in a 1024-position tile
 *             t ≡ 0 (mod stride) of the batch (reads concatenated in input
 *             order, every sequence character one position) and lies inside
 *             one read with no undetermined base; each occurrence counts
 *             for f and for rc(f);
 *  position = rank in ascending (frequency, A<C<G<T number) order;
 *  key      = rank of the position in ascending (|position - 4^m p|,
 *             position) order: the pivot 4^m p is the real number the paper
 *             names, and equal distances go to the smaller initial position
 *             (SPEC.md:196, :176).
 * Writes 4^m keys (index = the A<C<G<T number); returns 0, or -1 on a parse error. */
int oracle_dfp_table(const char* text, uint64_t len, uint32_t m, double pivot, uint32_t stride,
                     uint32_t* out) {
  std::vector<std::string> reads;
  std::string e;
  if (!parse_reads(text, len, reads, e)) return -1;
  const uint64_t M = 1ull << (2 * m);
  std::vector<uint64_t> freq(M, 0);
  uint64_t base = 0;
  for (const std::string& r : reads) {
    std::string u = r;
    for (char& c : u)
      if (c >= 'a' && c <= 'z') c = (char)(c - 'a' + 'A');
    for (size_t j = 0; j + m <= u.size(); ++j) {
      if (((base + j) / 1024) % stride != 0) continue;
      const std::string f = u.substr(j, m);
      if (f.find_first_not_of("ACGT") != std::string::npos) continue;
      freq[number_in(f, "ACGT")]++;
      freq[number_in(reverse_complement(f), "ACGT")]++;
    }
    base += u.size();
  }
  std::vector<uint32_t> order(M);
  for (uint64_t v = 0; v < M; ++v) order[v] = (uint32_t)v;
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return freq[a] != freq[b] ? freq[a] < freq[b] : a < b;
  });
  const double x = pivot * (double)M; /* the pivot position 4^m p */
  std::vector<uint64_t> bypiv(M);
  for (uint64_t pos = 0; pos < M; ++pos) bypiv[pos] = pos;
  std::sort(bypiv.begin(), bypiv.end(), [&](uint64_t a, uint64_t b) {
    const double da = std::fabs((double)a - x), db = std::fabs((double)b - x);
    return da != db ? da < db : a < b;
  });
  for (uint64_t r = 0; r < M; ++r) out[order[bypiv[r]]] = (uint32_t)r;
  return 0;
}

/* Fig. Minimizer metric: number of distinct canonical
 * k-mers per (strand-symmetric) minimizer; returns the maximum and writes the
 * number of minimizers that own at least one k-mer. -1 on a parse error. */
int64_t oracle_minimizer_stats(const char* text, uint64_t len, uint32_t k, uint32_t m, int ordering,
                               const uint32_t* table, uint64_t* n_minimizers) {
  std::vector<std::string> reads;
  std::string e;
  if (!parse_reads(text, len, reads, e)) return -1;
  std::map<std::string, uint64_t> hist;
  uint64_t windows = 0;
  count_reads(reads, 0, reads.size(), k, 1, 1, hist, windows);
  std::map<std::string, uint64_t> per;
  for (auto& kv : hist) per[minimizer_of(kv.first, m, ordering, 1, table)]++;
  uint64_t mx = 0;
  for (auto& kv : per) mx = std::max(mx, kv.second);
  if (n_minimizers) *n_minimizers = per.size();
  return (int64_t)mx;
}

/* Super-mers of one ACGT-only fragment: maximal runs of consecutive k-mers
 * whose minimizers are equal (Fig. 1). Writes the super-mers
 * separated by '\n' into out (if large enough); returns the bytes needed. */
uint64_t oracle_supermers_t(const char* seq, uint32_t len, uint32_t k, uint32_t m, int ordering,
                            int symmetric, const uint32_t* table, char* out, uint64_t cap) {
  std::string s(seq, len), text;
  if (len >= k) {
    size_t nwin = len - k + 1;
    std::vector<std::string> mu(nwin);
    for (size_t p = 0; p < nwin; ++p) mu[p] = minimizer_of(s.substr(p, k), m, ordering, symmetric, table);
    size_t p0 = 0;
    for (size_t p = 1; p <= nwin; ++p) {
      if (p == nwin || mu[p] != mu[p0]) {
        /* windows p0..p-1 share one minimizer: bases [p0, p-1+k) */
        text += s.substr(p0, (p - 1 - p0) + k);
        text += '\n';
        p0 = p;
      }
    }
  }
  if (out && cap >= text.size()) memcpy(out, text.data(), text.size());
  return text.size();
}

uint64_t oracle_supermers(const char* seq, uint32_t len, uint32_t k, uint32_t m, int ordering,
                          int symmetric, char* out, uint64_t cap) {
  return oracle_supermers_t(seq, len, k, m, ordering, symmetric, nullptr, out, cap);
}

} /* extern "C" */
