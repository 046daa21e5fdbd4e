// reader.cpp — step (a): host reader, FASTA/FASTQ → 2-bit packed batch.
//
// PAPER.md:94-95 (§2.3.1 steps 1-2): reader threads load the reads, parser
// threads convert them "into an internal read bundle format"; App. B
// input formats; App. C 2-bit codes A=00 C=01
// G=10 T=11. Undetermined bases are kept in the batch as
// N-mask bits so that the device decides window validity (include/gerbil.h).
//
// Parsing rules (readings Q3/Q4): FASTA = '>' header then sequence
// lines concatenated; FASTQ = '@' header, one sequence line, '+' [header],
// quality line of the same length; otherwise one read per non-empty line.
// CR bytes are dropped; empty lines are skipped; lowercase bases are folded.
//
// Two passes: a sequential line scan (memchr) records each read's sequence
// lines; then threads pack disjoint read ranges (words shared at range
// edges are merged with atomic OR).
#include "reader.h"

#include <dlfcn.h>
#include <fcntl.h>
#include <zlib.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>

namespace gerbil {
namespace {

struct Seg {
  uint64_t off;     // byte offset of the line in the text
  uint64_t inread;  // bases of the same read before this line
  uint32_t len;     // line length without '\n'
  uint32_t read;    // read index
};

static inline uint32_t count_cr(const char* p, uint32_t n) {
  uint32_t c = 0;
  const char* e = p + n;
  while ((p = (const char*)memchr(p, '\r', e - p))) { ++c; ++p; }
  return c;
}

static bool scan(const char* text, uint64_t len, std::vector<Seg>& segs,
                 std::vector<uint64_t>& read_len, std::string& err, const char* name) {
  uint64_t i = 0, line_no = 0;
  int kind = -1;  // 0 fasta, 1 fastq, 2 raw
  int fq_state = 0;  // fastq: 0 expect header, 1 seq, 2 plus, 3 qual
  uint64_t fq_seq_bases = 0;
  while (i < len) {
    const char* nl = (const char*)memchr(text + i, '\n', len - i);
    uint64_t e = nl ? (uint64_t)(nl - text) : len;
    uint32_t L = (uint32_t)(e - i);
    ++line_no;
    const char* p = text + i;
    uint32_t cr = count_cr(p, L);
    uint32_t eff = L - cr;
    uint64_t start = i;
    i = e + 1;
    // empty lines are skipped, except inside a FASTQ record (empty read)
    if (eff == 0 && !(kind == 1 && fq_state != 0)) continue;
    char first = 0;
    for (uint32_t t = 0; t < L; ++t)
      if (p[t] != '\r') { first = p[t]; break; }
    if (kind < 0) kind = first == '>' ? 0 : first == '@' ? 1 : 2;
    if (kind == 0) {
      if (first == '>') {
        read_len.push_back(0);
      } else {
        segs.push_back({start, read_len.back(), L, (uint32_t)(read_len.size() - 1)});
        read_len.back() += eff;
      }
    } else if (kind == 1) {
      if (fq_state == 0) {
        if (first != '@') {
          err = std::string(name) + ":" + std::to_string(line_no) + ": FASTQ: expected '@'";
          return false;
        }
        fq_state = 1;
      } else if (fq_state == 1) {
        read_len.push_back(eff);
        segs.push_back({start, 0, L, (uint32_t)(read_len.size() - 1)});
        fq_seq_bases = eff;
        fq_state = 2;
      } else if (fq_state == 2) {
        if (first != '+') {
          err = std::string(name) + ":" + std::to_string(line_no) + ": FASTQ: expected '+'";
          return false;
        }
        fq_state = 3;
      } else {
        if (eff != fq_seq_bases) {
          err = std::string(name) + ":" + std::to_string(line_no) +
                ": FASTQ: quality length differs from sequence length";
          return false;
        }
        fq_state = 0;
      }
    } else {
      read_len.push_back(eff);
      segs.push_back({start, 0, L, (uint32_t)(read_len.size() - 1)});
    }
  }
  if (kind == 1 && fq_state != 0) {
    err = std::string(name) + ":" + std::to_string(line_no) + ": FASTQ: truncated record";
    return false;
  }
  return true;
}

struct Lut {
  uint8_t code[256];
  uint8_t is_n[256];
  uint8_t skip[256];
  Lut() {
    for (int c = 0; c < 256; ++c) { code[c] = 0; is_n[c] = 1; skip[c] = 0; }
    const char* u = "ACGT";
    const char* l = "acgt";
    for (int b = 0; b < 4; ++b) {
      code[(uint8_t)u[b]] = b; is_n[(uint8_t)u[b]] = 0;
      code[(uint8_t)l[b]] = b; is_n[(uint8_t)l[b]] = 0;
    }
    skip[(uint8_t)'\r'] = 1;
  }
};
static const Lut kLut;

// ---- compressed input (§2.3.1 step 1: reader threads decompress;
// App. B: "compressed files of these formats") -----------------------
// gzip (RFC 1952, any number of concatenated members, e.g. BGZF) through zlib; bzip2
// (any number of concatenated streams) through libbz2, loaded at run time (the image
// ships the library but no header: the few entry points and bz_stream are declared here).
bool inflate_gzip(const unsigned char* in, uint64_t len, std::string& out, std::string& err, const char* name) {
  constexpr uint64_t kPiece = 1u << 30;  // zlib counts in uInt
  z_stream z{};
  if (inflateInit2(&z, 15 + 32) != Z_OK) {
    err = std::string(name) + ": zlib init failed";
    return false;
  }
  out.assign(std::max<uint64_t>(len * 4, 1 << 16), '\0');
  uint64_t used = 0, fed = 0;  // fed: input bytes handed to zlib so far
  for (;;) {
    if (z.avail_in == 0 && fed < len) {
      const uint64_t n = std::min(len - fed, kPiece);
      z.next_in = const_cast<Bytef*>(in + fed);
      z.avail_in = (uInt)n;
      fed += n;
    }
    if (used == out.size()) out.resize(out.size() * 2);
    const uint64_t room = std::min<uint64_t>(out.size() - used, kPiece);
    z.next_out = reinterpret_cast<Bytef*>(&out[used]);
    z.avail_out = (uInt)room;
    const int r = inflate(&z, Z_NO_FLUSH);
    used += room - z.avail_out;
    if (r == Z_STREAM_END) {  // end of one member: another may follow (concatenated gzip / BGZF)
      uint64_t at = fed - z.avail_in;
      while (at < len && in[at] == 0) ++at;  // zero padding after the last member
      if (at >= len) break;
      inflateReset(&z);
      const uint64_t n = std::min(len - at, kPiece);
      z.next_in = const_cast<Bytef*>(in + at);
      z.avail_in = (uInt)n;
      fed = at + n;
      continue;
    }
    if (r == Z_BUF_ERROR && z.avail_in == 0 && fed >= len) {
      inflateEnd(&z);
      err = std::string(name) + ": truncated gzip stream";
      return false;
    }
    if (r != Z_OK && r != Z_BUF_ERROR) {
      inflateEnd(&z);
      err = std::string(name) + ": gzip data error (" + (z.msg ? z.msg : "inflate") + ")";
      return false;
    }
  }
  inflateEnd(&z);
  out.resize(used);
  return true;
}

struct BzStream {  // bzlib.h bz_stream (stable ABI since bzip2 1.0)
  char* next_in;
  unsigned int avail_in, total_in_lo32, total_in_hi32;
  char* next_out;
  unsigned int avail_out, total_out_lo32, total_out_hi32;
  void* state;
  void* (*bzalloc)(void*, int, int);
  void (*bzfree)(void*, void*);
  void* opaque;
};
struct Bz2Lib {
  int (*init)(BzStream*, int, int) = nullptr;
  int (*step)(BzStream*) = nullptr;
  int (*end)(BzStream*) = nullptr;
  bool ok = false;
  Bz2Lib() {
    void* h = dlopen("libbz2.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libbz2.so.1.0", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libbz2.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    init = reinterpret_cast<int (*)(BzStream*, int, int)>(dlsym(h, "BZ2_bzDecompressInit"));
    step = reinterpret_cast<int (*)(BzStream*)>(dlsym(h, "BZ2_bzDecompress"));
    end = reinterpret_cast<int (*)(BzStream*)>(dlsym(h, "BZ2_bzDecompressEnd"));
    ok = init && step && end;
  }
};
constexpr int kBzOk = 0, kBzStreamEnd = 4;

bool inflate_bzip2(const unsigned char* in, uint64_t len, std::string& out, std::string& err, const char* name) {
  static Bz2Lib lib;
  if (!lib.ok) {
    err = std::string(name) + ": bzip2 input needs libbz2.so.1";
    return false;
  }
  out.clear();
  out.resize(std::max<uint64_t>(len * 5, 1 << 16));
  uint64_t used = 0, pos = 0;
  while (pos < len) {  // one bzip2 stream per iteration (pbzip2 writes several)
    BzStream b{};
    if (lib.init(&b, 0, 0) != kBzOk) {
      err = std::string(name) + ": bzip2 init failed";
      return false;
    }
    int r = kBzOk;
    while (r == kBzOk) {
      if (used == out.size()) out.resize(out.size() * 2);
      const uint64_t in_chunk = std::min<uint64_t>(len - pos, 1u << 30);
      const uint64_t room = std::min<uint64_t>(out.size() - used, 1u << 30);
      b.next_in = const_cast<char*>(reinterpret_cast<const char*>(in + pos));
      b.avail_in = (unsigned)in_chunk;
      b.next_out = &out[used];
      b.avail_out = (unsigned)room;
      r = lib.step(&b);
      pos += in_chunk - b.avail_in;
      used += room - b.avail_out;
      if (r == kBzOk && in_chunk - b.avail_in == 0 && room - b.avail_out == 0 && pos >= len) r = -7;
    }
    lib.end(&b);
    if (r != kBzStreamEnd) {
      err = std::string(name) + ": bzip2 data error or truncated stream";
      return false;
    }
    while (pos < len && in[pos] == 0) ++pos;
  }
  out.resize(used);
  return true;
}

enum class Codec { kPlain, kGzip, kBzip2 };
Codec sniff(const unsigned char* b, uint64_t len) {
  if (len >= 2 && b[0] == 0x1f && b[1] == 0x8b) return Codec::kGzip;
  if (len >= 4 && b[0] == 'B' && b[1] == 'Z' && b[2] == 'h' && b[3] >= '1' && b[3] <= '9') return Codec::kBzip2;
  return Codec::kPlain;
}

// one input file as text: mapped when plain, decompressed into `owned` otherwise
struct FileText {
  const char* p = nullptr;
  uint64_t len = 0;
  void* map = nullptr;
  uint64_t map_len = 0;
  std::string owned;
  std::string err;
  bool ok = false;
  ~FileText() {
    if (map) munmap(map, map_len);
  }
};

void load_file(const char* path, FileText& f) {
  int fd = open(path, O_RDONLY);
  if (fd < 0) {
    f.err = std::string(path) + ": cannot open";
    return;
  }
  struct stat st;
  if (fstat(fd, &st) != 0) {
    close(fd);
    f.err = std::string(path) + ": cannot stat";
    return;
  }
  const uint64_t len = (uint64_t)st.st_size;
  if (len == 0) {
    close(fd);
    f.ok = true;
    return;
  }
  void* m = mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
  close(fd);
  if (m == MAP_FAILED) {
    f.err = std::string(path) + ": cannot map";
    return;
  }
  const unsigned char* b = (const unsigned char*)m;
  const Codec c = sniff(b, len);
  if (c == Codec::kPlain) {
    f.map = m;
    f.map_len = len;
    f.p = (const char*)m;
    f.len = len;
    f.ok = true;
    return;
  }
  f.ok = c == Codec::kGzip ? inflate_gzip(b, len, f.owned, f.err, path) : inflate_bzip2(b, len, f.owned, f.err, path);
  munmap(m, len);
  f.p = f.owned.data();
  f.len = f.owned.size();
}

}  // namespace

bool pack_text(const char* text, uint64_t len, int threads, PackedBatch& out,
               std::string& err, const char* name) {
  std::vector<Seg> segs;
  std::vector<uint64_t> read_len;
  if (!scan(text, len, segs, read_len, err, name)) return false;
  const uint64_t base_reads = out.n_reads;
  const uint64_t base_bases = out.n_bases;
  // read starts
  out.read_start.resize(base_reads + read_len.size() + 1);
  if (base_reads == 0) out.read_start[0] = 0;
  uint64_t acc = base_bases;
  for (size_t r = 0; r < read_len.size(); ++r) {
    out.read_start[base_reads + r] = acc;
    acc += read_len[r];
  }
  out.read_start[base_reads + read_len.size()] = acc;
  const uint64_t total = acc;
  out.codes.resize((total + 31) / 32, 0ull);
  out.nmask.resize((total + 63) / 64, 0ull);
  out.n_reads = base_reads + read_len.size();
  out.n_bases = total;
  if (segs.empty()) return true;

  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const size_t per = (segs.size() + threads - 1) / threads;
  uint64_t* codes = out.codes.data();
  uint64_t* nmask = out.nmask.data();
  const uint64_t* rstart = out.read_start.data();
  auto work = [&](size_t s0, size_t s1) {
    if (s0 >= s1) return;
    // base offset of the first segment: read start + bases of earlier segments of that read
    uint64_t pos = rstart[base_reads + segs[s0].read] + segs[s0].inread;
    uint64_t cw = 0, nw = 0;
    uint64_t cur_c = pos >> 5, cur_n = pos >> 6;
    auto flush_c = [&] { if (cw) std::atomic_ref<uint64_t>(codes[cur_c]).fetch_or(cw, std::memory_order_relaxed); cw = 0; };
    auto flush_n = [&] { if (nw) std::atomic_ref<uint64_t>(nmask[cur_n]).fetch_or(nw, std::memory_order_relaxed); nw = 0; };
    for (size_t s = s0; s < s1; ++s) {
      const unsigned char* p = (const unsigned char*)text + segs[s].off;
      for (uint32_t t = 0; t < segs[s].len; ++t) {
        const unsigned char ch = p[t];
        if (kLut.skip[ch]) continue;
        if ((pos >> 5) != cur_c) { flush_c(); cur_c = pos >> 5; }
        if ((pos >> 6) != cur_n) { flush_n(); cur_n = pos >> 6; }
        cw |= (uint64_t)kLut.code[ch] << (62 - 2 * (pos & 31));
        if (kLut.is_n[ch]) nw |= 1ull << (63 - (pos & 63));
        ++pos;
      }
    }
    flush_c();
    flush_n();
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) {
    size_t a = std::min(segs.size(), t * per), b = std::min(segs.size(), a + per);
    if (a >= b) break;
    ts.emplace_back(work, a, b);
  }
  for (auto& t : ts) t.join();
  return true;
}

bool pack_file(const char* path, int threads, PackedBatch& out, std::string& err) {
  return pack_files(&path, 1, threads, out, err);
}

// Files are loaded (mapped, or decompressed — one file per thread, in parallel) ahead of
// the packer, which appends them in order with all threads.
bool pack_files(const char* const* paths, uint32_t n, int threads, PackedBatch& out, std::string& err) {
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  std::vector<FileText> files(n);
  std::atomic<uint32_t> next{0};
  auto loader = [&] {
    for (uint32_t i; (i = next.fetch_add(1)) < n;) load_file(paths[i], files[i]);
  };
  std::vector<std::thread> ts;
  const uint32_t nl = std::min<uint32_t>(n, (uint32_t)threads);
  for (uint32_t t = 1; t < nl; ++t) ts.emplace_back(loader);
  loader();
  for (auto& t : ts) t.join();
  for (uint32_t i = 0; i < n; ++i) {
    if (!files[i].ok) {
      err = files[i].err;
      return false;
    }
    if (files[i].len && !pack_text(files[i].p, files[i].len, threads, out, err, paths[i])) return false;
  }
  return true;
}

}  // namespace gerbil
