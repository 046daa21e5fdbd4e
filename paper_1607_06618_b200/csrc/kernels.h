// kernels.h — launch wrappers of the device steps (b)-(e); internal to the
// library (the public boundary is include/gerbil.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gerbil {

struct SupermerArgs {
  const uint64_t* codes;       // packed 2-bit stream
  const uint64_t* nmask;       // N bitmap or nullptr
  const uint64_t* read_start;  // n_reads + 1 base offsets
  uint64_t n_reads;
  uint64_t n_bases;            // read_start[n_reads]
  uint32_t k, m, n_bins, ordering;
  const uint32_t* order_rank;  // DFP ordering: key table [4^m] (ordering.cuh), else null
  uint32_t k_bits_for_words;   // k (payload words per super-mer = ceil((nwin+k-1)/32))
  // outputs
  uint64_t* desc;              // [cap] pos << 11 | (nwin - 1)
  uint32_t* bin;               // [cap]
  uint32_t* mu;                // [cap] minimizer key (debug) or nullptr
  uint64_t cap;
  unsigned long long* n_supermers;   // total produced (may exceed cap → caller regrows)
  unsigned long long* n_windows;     // Σ nwin (valid windows)
  unsigned long long* bin_windows;   // [n_bins]
  unsigned long long* bin_supermers; // [n_bins]
  unsigned long long* bin_words;     // [n_bins] payload words (multi-GPU) or nullptr
};
// Read-per-lane variant (supermer_reads.cu) for w = k-m+1 <= 64 and reads of
// <= 4096 bases on average; `work` is one device counter.
bool supermer_reads_applicable(uint32_t k, uint32_t m, uint64_t n_bases, uint64_t n_reads);
cudaError_t launch_supermer_reads(const SupermerArgs& a, unsigned long long* work, int sms, cudaStream_t s);
// rs_bits: scratch of supermer_scratch_words(n_bases) u64 (read-start bitmap).
cudaError_t launch_supermer(const SupermerArgs& a, uint64_t* rs_bits, int sms, cudaStream_t s);
uint64_t supermer_scratch_words(uint64_t n_bases);
// The same in pieces, for a batch that arrives in chunks: clear the bitmap,
// mark the starts of reads [r0, r1) (read_start[r1] must be resident), run
// tiles [t0, t1) (their bases [0, t1*1024 + supermer_tile_reach()) resident,
// and every read starting below that marked).
cudaError_t supermer_prepare(const SupermerArgs& a, uint64_t* rs_bits, cudaStream_t s);
cudaError_t supermer_mark_reads(const SupermerArgs& a, uint64_t* rs_bits, uint64_t r0, uint64_t r1, int sms,
                                cudaStream_t s);
cudaError_t supermer_run_tiles(const SupermerArgs& a, const uint64_t* rs_bits, uint64_t t0, uint64_t t1, int sms,
                               cudaStream_t s);
uint64_t supermer_tile_count(uint64_t n_bases);
uint64_t supermer_tile_reach();

// ordering.cu: dfp(p) m-mer frequency sample (freq[4^m], zeroed by the
// caller, accumulates) and the per-minimizer distinct-k-mer histogram of a
// result set (hist[hist_n] zeroed; out2[0] = max, out2[1] = non-empty, zeroed).
// parse.cu: step (a) on the device (FASTA/FASTQ/raw text → packed batch); api.cu
// gerbil_parse_text orchestrates. Error codes of classify (low 8 bits of *err,
// line index above): 1 expected '@', 2 expected '+', 3 quality length,
// 4 truncated record, 5 empty line between FASTQ records.
uint64_t parse_blocks(uint64_t len);
uint64_t scan_tmp_words(uint64_t n);
cudaError_t launch_parse_count(const uint8_t* t, uint64_t len, uint32_t* cnt_nl, uint32_t* cnt_cr, cudaStream_t s);
cudaError_t launch_widen(const uint32_t* a, uint64_t* b, uint64_t n, int sms, cudaStream_t s);
cudaError_t launch_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* tmp, uint64_t* total,
                            cudaStream_t s);
cudaError_t launch_parse_write(const uint8_t* t, uint64_t len, const uint64_t* off_nl, const uint64_t* off_cr,
                               uint64_t* line_start, uint64_t* cr_pos, cudaStream_t s);
cudaError_t launch_parse_lines(const uint8_t* t, const uint64_t* ls, uint64_t n_lines, const uint64_t* cr,
                               uint64_t n_cr, uint32_t* eff, uint8_t* first,
                               unsigned long long* first_nonempty /* [2]: min, max */, int sms, cudaStream_t s);
cudaError_t launch_parse_classify(const uint32_t* eff, const uint8_t* first, uint64_t n_lines, uint64_t f0,
                                  uint64_t n_eff, int kind, uint64_t* seq_len, uint64_t* rflag,
                                  unsigned long long* err, int sms, cudaStream_t s);
cudaError_t launch_parse_read_starts(const uint64_t* pos, const uint64_t* rflag, const uint64_t* ridx,
                                     uint64_t n_lines, uint64_t* read_start, int sms, cudaStream_t s);
cudaError_t launch_parse_pack(const uint8_t* t, const uint64_t* ls, const uint64_t* seq_len, const uint64_t* pos,
                              uint64_t n_lines, uint64_t* codes, uint64_t* nmask, int sms, cudaStream_t s);

cudaError_t launch_dfp_sample(const uint64_t* codes, const uint64_t* nmask, const uint64_t* rs_bits,
                              uint64_t n_bases, uint32_t m, uint32_t stride, uint32_t* freq, int sms,
                              cudaStream_t s);
cudaError_t launch_minimizer_hist(const uint64_t* keys, uint64_t n, uint32_t W, uint32_t k, uint32_t m,
                                  uint32_t ordering, const uint32_t* rank, uint32_t* hist, uint64_t hist_n,
                                  unsigned long long* out2, int sms, cudaStream_t s);

struct ScatterArgs {
  const uint64_t* desc_in;
  const uint32_t* bin_in;
  uint64_t n;
  uint32_t n_bins;
  unsigned long long* cursor;  // [n_bins], initialised to the bin offsets
  uint64_t* desc_out;
  uint32_t* bin_out;           // optional (nullptr)
  uint64_t pos_add;            // added to pos (rebasing received super-mers)
  const unsigned char* keep;   // optional per-bin filter (owned bins) or nullptr
  uint32_t bin_shift;          // group by bin_in >> bin_shift (bin_out keeps the full bin); 0 = by bin
  uint32_t pack_low_bits;      // > 0: no bin_out; the bin's low pack_low_bits bits go into descriptor bits
                               // 54.. (descriptors < 2^54, i.e. positions < 2^43)
};
constexpr int kDescPackShift = 54;
cudaError_t launch_scatter(const ScatterArgs& a, int sms, cudaStream_t s);
cudaError_t launch_rebase_desc(uint64_t* desc, uint64_t n, uint64_t pos_add, int sms, cudaStream_t s);
// Second level of a two-level scatter: descriptors already grouped by bin >> shift
// (group g = [off[g << shift], off[min((g + 1) << shift, n_bins)]) of desc_in/bin_in)
// are regrouped by bin inside each group with shared-memory cursors.
cudaError_t launch_regroup_fine(const uint64_t* desc_in, const uint32_t* bin_in, const unsigned long long* off,
                                uint32_t n_bins, uint32_t shift, uint64_t* desc_out, cudaStream_t s);
// the same with the bin's low `shift` bits packed in the descriptors (ScatterArgs.pack_low_bits)
cudaError_t launch_regroup_fine_packed(const uint64_t* desc_in, const unsigned long long* off, uint32_t n_bins,
                                       uint32_t shift, uint64_t* desc_out, cudaStream_t s);

// Group-major shuffle (shuffle.cu, single rank, n_bins <= 2^22, descriptors < 2^54): groups the
// step-(b) output by bin without any per-super-mer global atomic and derives every bin's offset
// and windows on the way (no step-(b) histogram needed). desc_alt may alias desc_in.
struct GroupShuffleArgs {
  const uint64_t* desc_in;      // [n] step (b) descriptors
  const uint32_t* bin_in;       // [n] their bins
  uint64_t n;
  uint32_t n_bins;
  uint64_t* tmp_desc;           // [n] scratch
  uint32_t* tmp_bin;            // [n] scratch
  uint64_t* desc_alt;           // [n] scratch (may be desc_in)
  uint64_t* desc_out;           // [n] bin-ordered descriptors
  unsigned long long* off;      // [n_bins + 1] first descriptor of each bin (out)
  unsigned long long* win;      // [n_bins] windows per bin (out)
  unsigned long long* scratch;  // group_shuffle_scratch_bytes(n_bins)
  uint64_t max_windows;         // bound on the windows of any one bin (picks 32-bit shared counters)
};
uint32_t group_shuffle_groups(uint32_t n_bins);
size_t group_shuffle_scratch_bytes(uint32_t n_bins);
cudaError_t launch_group_shuffle(const GroupShuffleArgs& a, int sms, cudaStream_t s);
// Multi-rank exchange of whole groups (shuffle.cu): per-group [3][G] windows / super-mers /
// relocated payload words of bin-ordered descriptors (off = bin offsets), and the pack of every
// group into the send buffers; base3 = [3][G]: first send descriptor, first send payload word,
// and the first payload word in the OWNER's receive buffer of each group.
cudaError_t launch_group_stats(const uint64_t* desc, const unsigned long long* off, uint32_t n_bins, uint32_t k,
                               unsigned long long* st, cudaStream_t s);
cudaError_t launch_group_pack(const uint64_t* desc, const unsigned long long* off, uint32_t n_bins,
                              const uint64_t* codes, uint32_t k, const unsigned long long* base3, uint64_t* send_desc,
                              uint32_t* send_bin, uint64_t* send_payload, cudaStream_t s);

// world > 1: copy every local super-mer (descriptor + word-aligned payload)
// into the send buffer, ordered by (destination rank, bin).
struct PackArgs {
  const uint64_t* desc_in;
  const uint32_t* bin_in;
  uint64_t n;
  const uint64_t* codes;
  uint32_t k;
  unsigned long long* cur_desc;              // [B] next send slot of the bin
  unsigned long long* cur_words;             // [B] next payload word of the bin
  const unsigned long long* seg_word_base;   // [B] first payload word of the bin's destination
  uint64_t* send_desc;
  uint32_t* send_bin;
  uint64_t* send_payload;
};
cudaError_t launch_pack(const PackArgs& a, int sms, cudaStream_t s);

struct TableArgs {
  unsigned char* table;  // nb buckets
  uint64_t nb;
  uint32_t max_probes;   // θ (buckets)
  uint64_t* ovf;         // overflow keys [ovf_cap * W]
  uint64_t ovf_cap;
  unsigned long long* ovf_n;
  unsigned long long* probe_hist;  // [4]: first-bucket hits, >1 bucket, max probes, unused
};

struct CountArgs {
  const uint64_t* codes;   // stream the descriptors point into
  const uint64_t* desc;    // bin-ordered descriptors
  uint64_t d0, d1;         // wave range
  uint32_t k;
  TableArgs t;
  unsigned long long* work;  // zeroed per launch: dynamic chunk counter
  uint32_t canonical;        // 1 = count min(x, rc x); 0 = `-d`
  uint32_t dpc;              // descriptors per warp work unit (1..32; 0 = 32): fewer for long super-mers
};
// descriptors per work unit for super-mers of `avg_windows` windows on average: ~512 windows
// per unit, at most 32 (one per lane)
inline uint32_t count_dpc(double avg_windows) {
  if (avg_windows <= 16.0) return 32;
  const double d = 512.0 / avg_windows;
  return d < 1.0 ? 1u : (uint32_t)d;
}
cudaError_t launch_count(const CountArgs& a, uint32_t W, int sms, cudaStream_t s);
cudaError_t launch_count_wide(const CountArgs& a, int sms, cudaStream_t s);  // W = 8..15 (count_wide.cu)

// count_smem.cu: steps (d)+(e) for bins whose distinct k-mers fit one warp's
// shared-memory table (one warp per bin, warp-synchronous inserts, in-place
// compaction). Abandoned bins (distinct > max_fill) are listed in `failed`.
constexpr int kSmemMaxWarps = 24;
constexpr int kRangeWinShift = 40;  // bin windows (clamped to 2^24 - 1) above the end descriptor index
constexpr unsigned long long kRangeEndMask = (1ull << kRangeWinShift) - 1;
struct SmemCountArgs {
  const uint64_t* codes;             // stream the descriptors point into
  const uint64_t* desc;              // bin-ordered descriptors
  const unsigned long long* range;   // [n_list][2]: first descriptor; end descriptor | windows << kRangeWinShift
  uint32_t n_list;
  uint32_t k, min_count, canonical;
  uint32_t cap;                      // table slots per warp (multiple of 32)
  uint32_t max_fill;                 // abandon a bin past this many distinct k-mers (<= cap - 64)
  uint64_t* out_keys;                // [out_cap * W]
  uint32_t* out_counts;              // [out_cap]
  uint64_t out_cap;
  unsigned long long* out_n;
  unsigned long long* sum_counts;
  unsigned long long* distinct;
  unsigned long long* failed;        // [n_list][2] range entries of abandoned bins
  unsigned long long* n_failed;
  uint32_t dbg;                      // diagnostics: 1 = no rc stage, 2 = no window map, 8 = full-size tables
  int32_t warps;                     // warps per CTA (0 = smem_count_warps(k)); cap must match; -1 = the
                                     // CTA-wide reference tables of count_ref.cu (any W)
  uint32_t parts, part;              // count_ref: only k-mers with (hash >> 32) % parts == part (0/1 = all)
};
// Table slots a bin of `win` windows gets (count_smem_kernel): windows * 1.25 + 32, rounded up to 32,
// capped at the warp's table (cap).
__host__ __device__ inline uint32_t smem_bin_slots(uint64_t win, uint32_t cap) {
  const uint64_t w = win < (1ull << 24) ? win : (1ull << 24) - 1;
  const uint64_t want = (w + (w >> 2) + 32u + 31u) & ~31ull;
  return want < cap ? (uint32_t)want : cap;
}
// Output bound of one bin in the shared-memory pass: a bin with a full-size table is abandoned
// past max_fill distinct k-mers (no output); a smaller table is never abandoned (distinct <= windows).
__host__ __device__ inline uint64_t smem_bin_out_bound(uint64_t win, uint32_t cap, uint32_t max_fill) {
  return smem_bin_slots(win, cap) < cap ? win : (win < max_fill ? win : max_fill);
}
int smem_count_warps(uint32_t k);                            // warps per CTA (GERBIL_SMEM_WARPS overrides)
uint32_t smem_slot_bytes(uint32_t k);
uint32_t smem_warp_bytes(uint32_t k, uint32_t cap);
uint32_t smem_table_slots(uint32_t k, size_t smem_per_block, int warps = 0);  // 0 = no room
cudaError_t launch_count_smem(const SmemCountArgs& a, int sms, cudaStream_t s);  // W >= 4: count_ref
// count_ref.cu (W >= 4): a.cap = slots of the CTA-wide table of occurrence references
size_t ref_table_bytes(uint32_t cap);
uint32_t ref_table_slots(size_t smem_per_block, int ctas_per_sm = 1);  // 2: two 256-thread CTAs per SM (a.warps = -2)
uint32_t ref_max_fill(uint32_t cap);
cudaError_t launch_count_ref(const SmemCountArgs& a, int sms, cudaStream_t s);
struct PlanBinsArgs {
  const unsigned long long* win;   // [n_bins] windows per bin (step b histogram)
  const unsigned long long* off;   // [n_bins + 1] first descriptor of each bin (exclusive scan)
  uint32_t n_bins;
  unsigned long long thr;          // shared-memory list iff windows <= thr
  uint32_t cap, max_fill;          // table slots per warp, abandonment threshold (output bound)
  unsigned long long* elig;        // [n_bins][2] shared-memory list (range entries, kRangeWinShift)
  unsigned long long* rest;        // [n_bins][3] first descriptor, end descriptor, windows
  unsigned long long* sums;        // [4]: n_elig, Σ elig windows, Σ smem_bin_out_bound, n_rest (zeroed)
  unsigned long long* max_win;     // (zeroed)
};
cudaError_t launch_plan_bins(const PlanBinsArgs& a, int sms, cudaStream_t s);
// dst[dst_off[i] + j] = src[ranges[2i] + j] for j < ranges[2i+1] - ranges[2i]
cudaError_t launch_gather_ranges(const uint64_t* src, const unsigned long long* ranges,
                                 const unsigned long long* dst_off, uint32_t n, uint64_t* dst, int sms,
                                 cudaStream_t s);

struct CountKeysArgs {      // emergency path: insert overflow keys
  const uint64_t* keys;     // [n * W]
  uint64_t n;
  uint32_t k;
  TableArgs t;
};
cudaError_t launch_count_keys(const CountKeysArgs& a, uint32_t W, int sms, cudaStream_t s);
cudaError_t launch_count_keys_wide(const CountKeysArgs& a, int sms, cudaStream_t s);

struct CompactArgs {
  unsigned char* table;
  uint64_t nb;
  uint32_t k, min_count;
  uint64_t* out_keys;      // [cap * W]
  uint32_t* out_counts;    // [cap]
  uint64_t cap;
  unsigned long long* out_n;
  unsigned long long* sum_counts;
  unsigned long long* distinct;
  unsigned long long* wave_distinct;  // per-wave slot or nullptr
  // optional App. C record stream: every kept k-mer is also
  // encoded into rec_out (page-locked host memory) at a byte range reserved on
  // *rec_n; nothing is written past rec_cap (rec_n still counts every byte)
  uint8_t* rec_out;
  uint64_t rec_cap;
  unsigned long long* rec_n;
};
cudaError_t launch_compact(const CompactArgs& a, int sms, cudaStream_t s);
cudaError_t launch_store_u64(unsigned long long* dst_mapped, const unsigned long long* src, cudaStream_t s);
cudaError_t launch_copy_words_mapped(unsigned long long* dst_mapped, const unsigned long long* src, uint64_t n,
                                     cudaStream_t s);
// App. C records of results [*lo, *hi) (device snapshots; at most max_n entries) appended to rec at a
// byte range reserved on *rec_n (nothing is written past rec_cap; *rec_n counts every byte)
cudaError_t launch_encode_records(const uint64_t* keys, const uint32_t* counts, const unsigned long long* lo,
                                  const unsigned long long* hi, uint64_t max_n, uint32_t k, uint8_t* rec,
                                  uint64_t rec_cap, unsigned long long* rec_n, int sms, cudaStream_t s);


cudaError_t launch_clear_table(unsigned char* table, uint64_t bytes, int sms, cudaStream_t s);

// sort.cu: LSD radix sort of n results (W-word keys of k bases, u32 counts) into A<C<G<T order
uint64_t sort_scratch_words(uint64_t n);
cudaError_t launch_sort_results(uint64_t* keys, uint32_t* cnt, uint64_t n, uint32_t W, uint32_t k, uint64_t* keys_tmp,
                                uint32_t* cnt_tmp, uint64_t* scratch, int sms, cudaStream_t s);

}  // namespace gerbil
