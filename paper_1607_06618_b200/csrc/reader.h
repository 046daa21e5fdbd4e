// reader.h — step (a) host reader interface (internal).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

namespace gerbil {

// A packed read batch in the layout of include/gerbil.h.
struct PackedBatch {
  std::vector<uint64_t> codes, nmask, read_start;
  uint64_t n_bases = 0, n_reads = 0;
};

// Parses one FASTA/FASTQ/raw document and APPENDS its reads to out.
bool pack_text(const char* text, uint64_t len, int threads, PackedBatch& out,
               std::string& err, const char* name);
bool pack_file(const char* path, int threads, PackedBatch& out, std::string& err);
// Several files, in order; gzip (.gz, concatenated members) and bzip2 inputs are decompressed
// on host threads (one file per thread).
bool pack_files(const char* const* paths, uint32_t n, int threads, PackedBatch& out, std::string& err);

}  // namespace gerbil
